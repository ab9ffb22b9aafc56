// comm.cuh — internal view of ga_comm (multi-GPU plumbing).
#pragma once
#include <list>
#include <map>
#include <utility>
#include <vector>

#include "common.cuh"

// One symmetric allocation: the same size on every rank, each rank's copy mapped into every
// other rank's address space with CUDA IPC (peer loads over NVLink; same-device mappings
// when several ranks share a GPU).
struct GaSymAlloc {
    char *local = nullptr;
    size_t bytes = 0;
    std::vector<char *> peers;                          // [world]; peers[rank] == local
    std::map<size_t, const char **> dev_tables;         // offset -> DEVICE [world] of peers[q]+offset
};

struct ga_comm {
    int world = 1, rank = 0, device = -1;
    std::vector<int> fds;        // rank 0: fds[q] = socket to rank q (q >= 1); others: fds[0] = rank 0
    std::list<GaSymAlloc> allocs; // stable addresses
    // device barrier state: flags[q] (in the first symmetric allocation) is written by rank q
    GaSymAlloc *flag_alloc = nullptr;
    uint64_t gen = 0;
    // set to 1 by a device barrier that gave up waiting for a peer: pinned, device-mapped host
    // memory, so the host reads it without synchronising (ga_comm_status, and the entry check
    // of ga_attention_sharded)
    volatile int *timed_out_host = nullptr;
    int *timed_out_dev = nullptr;
    // CSR / BigBird all-gather scratch: full-length K and V (grown on demand)
    void *gather_k = nullptr, *gather_v = nullptr;
    size_t gather_bytes = 0;
    // ring exchange (GA_EXCHANGE_RING): two staging buffers for one shard of K and of V, the
    // fp32 carried state of the local rows, a copy stream and its events (grown on demand)
    void *ring_kv[2] = {nullptr, nullptr};
    size_t ring_bytes = 0; // per staging buffer (K and V of one shard)
    float *ring_state = nullptr;
    size_t ring_state_bytes = 0;
    cudaStream_t ring_stream = nullptr;
    cudaEvent_t ring_ready[2] = {nullptr, nullptr}, ring_done[2] = {nullptr, nullptr}, ring_start = nullptr,
                ring_end = nullptr;
};

namespace ga {
// symmetric allocation owning `p` (any address inside it), or nullptr
GaSymAlloc *comm_find(ga_comm *c, const void *p);
// DEVICE table of the peers' copies of `p` (same offset in every rank's allocation)
ga_status comm_peer_table(ga_comm *c, const void *p, const char *const **table);
ga_status comm_device_barrier(ga_comm *c, cudaStream_t s);
// after a sharded call: if any barrier of this comm timed out, overwrite `bytes` of `out` with
// 0xff (NaN in fp32 / bf16 / fp16) so a stalled peer cannot yield silently wrong rows
ga_status comm_poison_on_timeout(ga_comm *c, void *out, size_t bytes, cudaStream_t s);
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
} // namespace ga

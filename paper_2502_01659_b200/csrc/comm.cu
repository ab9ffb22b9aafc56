// comm.cu — multi-GPU plumbing of libga (SURVEY §8(b) comm entry points, §8(e)).
//
// The attention path shards by query ranges (the rows of Algorithm 1 are independent,
// PAPER.md:255).  What crosses GPUs is K/V rows: the window halo, LongNet's strided rows,
// and for explicit CSR the whole K/V.  Instead of a separate exchange step, every rank's
// K/V shard lives in a SYMMETRIC buffer mapped into all ranks with CUDA IPC, so the kernels
// of ga_attention_sharded load a neighbour's rows straight from its HBM over NVLink while
// computing (fused exchange + compute; kv_row in common.cuh).  CSR masks instead all-gather
// K/V with copy engines first (random gathers are HBM-bound and should stay local).
//
// Pieces:
//   bootstrap   a TCP star rooted at rank 0 on 127.0.0.1 (one node): ga_comm_get_unique_id
//               opens the listening socket, ga_comm_create connects the ranks; used only
//               for host all-gathers of small blobs (IPC handles) and host barriers.
//   symmetric   ga_comm_alloc: cudaMalloc + cudaIpcGetMemHandle, handles all-gathered,
//   buffers     peers opened with cudaIpcOpenMemHandle (lazy peer access).
//   barrier     a one-warp kernel: release-store our generation into every peer's flag
//               slot, acquire-spin until every peer's generation arrived (bounded by a
//               timeout so a dead peer cannot hang the GPU).
#include <arpa/inet.h>
#include <errno.h>
#include <fcntl.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <string.h>
#include <sys/socket.h>
#include <time.h>
#include <unistd.h>

#include <chrono>
#include <mutex>
#include <random>
#include <thread>

#include "comm.cuh"

namespace ga {

static constexpr uint32_t kIdMagic = 0x47414331u; // "GAC1"
static constexpr int kTimeoutMs = 120000;         // bootstrap socket timeout
static constexpr uint64_t kBarrierTimeoutNs = 60ull * 1000000000ull;

struct CommId {
    uint32_t magic;
    uint16_t port;
    uint16_t reserved;
    uint32_t addr; // IPv4, network order
    uint32_t reserved2;
    uint64_t nonce;
    uint8_t pad[104];
};
static_assert(sizeof(CommId) == 128, "ga comm id is 128 bytes");

struct Hello {
    uint32_t magic;
    int32_t rank;
    uint64_t nonce;
};

static std::mutex g_listen_mu;
static std::map<uint64_t, int> g_listen; // nonce -> listening socket (rank 0's process)

static bool send_all(int fd, const void *buf, size_t n)
{
    const char *p = static_cast<const char *>(buf);
    while (n > 0) {
        pollfd pf{fd, POLLOUT, 0};
        if (poll(&pf, 1, kTimeoutMs) <= 0) return false;
        const ssize_t k = send(fd, p, n, MSG_NOSIGNAL);
        if (k < 0 && (errno == EINTR || errno == EAGAIN)) continue;
        if (k <= 0) return false;
        p += k;
        n -= (size_t)k;
    }
    return true;
}

static bool recv_all(int fd, void *buf, size_t n)
{
    char *p = static_cast<char *>(buf);
    while (n > 0) {
        pollfd pf{fd, POLLIN, 0};
        if (poll(&pf, 1, kTimeoutMs) <= 0) return false;
        const ssize_t k = recv(fd, p, n, 0);
        if (k < 0 && (errno == EINTR || errno == EAGAIN)) continue;
        if (k <= 0) return false;
        p += k;
        n -= (size_t)k;
    }
    return true;
}

// host all-gather over the star: all = concat over ranks of `n` bytes each
static ga_status host_allgather(ga_comm *c, const void *mine, size_t n, void *all)
{
    char *out = static_cast<char *>(all);
    memcpy(out + (size_t)c->rank * n, mine, n);
    if (c->world == 1) return GA_OK;
    if (c->rank == 0) {
        for (int q = 1; q < c->world; ++q)
            if (!recv_all(c->fds[q], out + (size_t)q * n, n)) {
                set_error("comm: receive from rank %d failed", q);
                return GA_ERR_COMM;
            }
        for (int q = 1; q < c->world; ++q)
            if (!send_all(c->fds[q], out, n * c->world)) {
                set_error("comm: send to rank %d failed", q);
                return GA_ERR_COMM;
            }
        return GA_OK;
    }
    if (!send_all(c->fds[0], mine, n) || !recv_all(c->fds[0], out, n * c->world)) {
        set_error("comm: exchange with rank 0 failed");
        return GA_ERR_COMM;
    }
    return GA_OK;
}

static ga_status host_barrier(ga_comm *c)
{
    std::vector<char> all(c->world);
    const char one = 1;
    return host_allgather(c, &one, 1, all.data());
}

GaSymAlloc *comm_find(ga_comm *c, const void *p)
{
    const char *q = static_cast<const char *>(p);
    for (auto &a : c->allocs)
        if (q >= a.local && q < a.local + a.bytes) return &a;
    return nullptr;
}

ga_status comm_peer_table(ga_comm *c, const void *p, const char *const **table)
{
    GaSymAlloc *a = comm_find(c, p);
    if (!a) {
        set_error("buffer %p is not a ga_comm_alloc allocation of this comm", p);
        return GA_ERR_INVALID_ARG;
    }
    const size_t off = (size_t)(static_cast<const char *>(p) - a->local);
    auto it = a->dev_tables.find(off);
    if (it == a->dev_tables.end()) {
        std::vector<const char *> h(c->world);
        for (int q = 0; q < c->world; ++q) h[q] = a->peers[q] + off;
        const char **d = nullptr;
        cudaError_t e = cudaMalloc(&d, sizeof(char *) * c->world);
        if (e != cudaSuccess) return cuda_fail(e, "comm: peer table");
        e = cudaMemcpy(d, h.data(), sizeof(char *) * c->world, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { cudaFree(d); return cuda_fail(e, "comm: peer table copy"); }
        it = a->dev_tables.emplace(off, d).first;
    }
    *table = it->second;
    return GA_OK;
}

// flags layout in the barrier allocation: uint64 gen_from[world] | int timed_out
__global__ void comm_barrier_kernel(uint64_t *const *peer_flags, uint64_t *my_flags, int rank, int world, uint64_t gen,
                                    int *timed_out)
{
    const int q = threadIdx.x;
    if (q < world && q != rank) {
        __threadfence_system(); // the stream's earlier writes (K/V) before the flag
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flags[q] + rank), "l"(gen) : "memory");
    }
    if (q < world && q != rank) {
        uint64_t t0, t, v;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + q) : "memory");
            if (v >= gen) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > kBarrierTimeoutNs) { // mapped host flag: a plain system-scope store
                asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(timed_out), "r"(1) : "memory");
                break;
            }
            __nanosleep(200);
        }
    }
    __syncwarp();
}

ga_status comm_device_barrier(ga_comm *c, cudaStream_t s)
{
    if (c->world == 1) return GA_OK;
    if (!c->flag_alloc) { set_error("comm has no device (created with device = -1)"); return GA_ERR_INVALID_ARG; }
    if (c->world > 32) { set_error("device barrier supports up to 32 ranks"); return GA_ERR_UNSUPPORTED; }
    const char *const *tbl = nullptr;
    ga_status st = comm_peer_table(c, c->flag_alloc->local, &tbl);
    if (st != GA_OK) return st;
    ++c->gen;
    uint64_t *mine = reinterpret_cast<uint64_t *>(c->flag_alloc->local);
    comm_barrier_kernel<<<1, 32, 0, s>>>((uint64_t *const *)tbl, mine,
                                         c->rank, c->world, c->gen, c->timed_out_dev);
    GA_CHECK_LAUNCH("comm_barrier_kernel");
    return GA_OK;
}

__global__ void comm_poison_kernel(const int *timed_out, uint4 *out, size_t n16)
{
    if (*(const volatile int *)timed_out == 0) return; // the common case: one load per CTA
    const uint4 nan = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        out[i] = nan;
}

ga_status comm_poison_on_timeout(ga_comm *c, void *out, size_t bytes, cudaStream_t s)
{
    if (c->world == 1 || !c->timed_out_dev || !out || bytes < 16) return GA_OK;
    comm_poison_kernel<<<64, 256, 0, s>>>(c->timed_out_dev, reinterpret_cast<uint4 *>(out), bytes / 16);
    GA_CHECK_LAUNCH("comm_poison_kernel");
    return GA_OK;
}

static void close_fds(ga_comm *c)
{
    for (int fd : c->fds)
        if (fd >= 0) close(fd);
    c->fds.clear();
}

static ga_status sym_free(ga_comm *c, GaSymAlloc &a)
{
    for (auto &kv : a.dev_tables) cudaFree(kv.second);
    a.dev_tables.clear();
    for (int q = 0; q < c->world; ++q)
        if (q != c->rank && a.peers[q]) cudaIpcCloseMemHandle(a.peers[q]);
    // every rank has closed its mappings of our buffer before we free it
    ga_status st = host_barrier(c);
    if (a.local) cudaFree(a.local);
    a.local = nullptr;
    return st;
}

} // namespace ga

using namespace ga;

extern "C" {

ga_status ga_comm_get_unique_id(void *id128)
{
    if (!id128) { set_error("id is NULL"); return GA_ERR_INVALID_ARG; }
    const int fd = socket(AF_INET, SOCK_STREAM, 0);
    if (fd < 0) { set_error("comm: socket: %s", strerror(errno)); return GA_ERR_COMM; }
    const int yes = 1;
    setsockopt(fd, SOL_SOCKET, SO_REUSEADDR, &yes, sizeof(yes));
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_addr.s_addr = htonl(INADDR_LOOPBACK); // one node: ranks rendezvous on 127.0.0.1
    a.sin_port = 0;
    socklen_t al = sizeof(a);
    if (bind(fd, reinterpret_cast<sockaddr *>(&a), sizeof(a)) != 0 || listen(fd, 1024) != 0 ||
        getsockname(fd, reinterpret_cast<sockaddr *>(&a), &al) != 0) {
        set_error("comm: bind/listen: %s", strerror(errno));
        close(fd);
        return GA_ERR_COMM;
    }
    CommId id{};
    id.magic = kIdMagic;
    id.port = ntohs(a.sin_port);
    id.addr = a.sin_addr.s_addr;
    std::random_device rd;
    id.nonce = ((uint64_t)rd() << 32) ^ rd() ^ (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count() ^
               ((uint64_t)getpid() << 17);
    {
        std::lock_guard<std::mutex> g(g_listen_mu);
        g_listen[id.nonce] = fd;
    }
    memcpy(id128, &id, sizeof(id));
    return GA_OK;
}

ga_status ga_comm_create(int32_t world, int32_t rank, const void *id128, int32_t device, ga_comm **comm)
{
    if (!comm || !id128) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    *comm = nullptr;
    if (world < 1 || rank < 0 || rank >= world) { set_error("need 0 <= rank < world"); return GA_ERR_INVALID_ARG; }
    CommId id;
    memcpy(&id, id128, sizeof(id));
    if (id.magic != kIdMagic) { set_error("not a ga_comm_get_unique_id id"); return GA_ERR_INVALID_ARG; }
    ga_comm *c = new ga_comm;
    c->world = world;
    c->rank = rank;
    c->device = device;
    c->fds.assign(world, -1);
    int lfd = -1;
    if (rank == 0) {
        std::lock_guard<std::mutex> g(g_listen_mu);
        auto it = g_listen.find(id.nonce);
        if (it != g_listen.end()) { lfd = it->second; g_listen.erase(it); }
    }
    if (world > 1) {
        if (rank == 0) {
            if (lfd < 0) {
                set_error("rank 0 must create the id with ga_comm_get_unique_id in this process");
                delete c;
                return GA_ERR_INVALID_ARG;
            }
            for (int n = 1; n < world; ++n) {
                pollfd pf{lfd, POLLIN, 0};
                if (poll(&pf, 1, kTimeoutMs) <= 0) { set_error("comm: timed out waiting for ranks"); break; }
                const int fd = accept(lfd, nullptr, nullptr);
                if (fd < 0) { set_error("comm: accept: %s", strerror(errno)); break; }
                const int yes = 1;
                setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &yes, sizeof(yes));
                Hello h{};
                if (!recv_all(fd, &h, sizeof(h)) || h.magic != kIdMagic || h.nonce != id.nonce || h.rank <= 0 ||
                    h.rank >= world || c->fds[h.rank] >= 0) {
                    set_error("comm: bad hello");
                    close(fd);
                    break;
                }
                c->fds[h.rank] = fd;
            }
            close(lfd);
            lfd = -1;
            for (int q = 1; q < world; ++q)
                if (c->fds[q] < 0) { close_fds(c); delete c; return GA_ERR_COMM; }
        } else {
            const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(kTimeoutMs);
            int fd = -1;
            while (std::chrono::steady_clock::now() < deadline) {
                fd = socket(AF_INET, SOCK_STREAM, 0);
                sockaddr_in a{};
                a.sin_family = AF_INET;
                a.sin_addr.s_addr = id.addr;
                a.sin_port = htons(id.port);
                if (fd >= 0 && connect(fd, reinterpret_cast<sockaddr *>(&a), sizeof(a)) == 0) break;
                if (fd >= 0) close(fd);
                fd = -1;
                std::this_thread::sleep_for(std::chrono::milliseconds(10));
            }
            if (fd < 0) { set_error("comm: cannot reach rank 0"); delete c; return GA_ERR_COMM; }
            const int yes = 1;
            setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &yes, sizeof(yes));
            Hello h{kIdMagic, rank, id.nonce};
            if (!send_all(fd, &h, sizeof(h))) { set_error("comm: hello failed"); close(fd); delete c; return GA_ERR_COMM; }
            c->fds[0] = fd;
        }
    } else if (lfd >= 0) {
        close(lfd);
    }
    if (device >= 0) { // barrier flags: uint64 [world], zeroed before use; timeout flag in mapped host memory
        void *flags = nullptr;
        ga_status st = GA_OK;
        {
            DeviceGuard dg(device);
            // every pair of devices must reach each other's memory (the kernels load peer rows
            // over NVLink); ranks sharing one device need no peer access
            int ndev = 0;
            cudaGetDeviceCount(&ndev);
            std::vector<int> devs(world);
            st = host_allgather(c, &device, sizeof(int), devs.data());
            for (int q = 0; st == GA_OK && q < world; ++q) {
                if (devs[q] == device) continue;
                int can = 0;
                if (devs[q] < 0 || devs[q] >= ndev || cudaDeviceCanAccessPeer(&can, device, devs[q]) != cudaSuccess ||
                    !can) {
                    set_error("comm: device %d cannot access peer device %d (cudaDeviceCanAccessPeer)", device, devs[q]);
                    st = GA_ERR_COMM;
                }
            }
            int ok_all = st == GA_OK, all[64] = {};
            if (world <= 64 && host_allgather(c, &ok_all, sizeof(int), all) == GA_OK)
                for (int q = 0; q < world; ++q)
                    if (!all[q] && st == GA_OK) { set_error("comm: peer access missing on rank %d", q); st = GA_ERR_COMM; }
            void *h = nullptr;
            if (st == GA_OK) {
                cudaError_t e = cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable);
                if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->timed_out_dev), h, 0);
                if (e != cudaSuccess) st = cuda_fail(e, "comm: timeout flag");
                else {
                    c->timed_out_host = static_cast<volatile int *>(h);
                    *c->timed_out_host = 0;
                }
            }
        }
        if (st != GA_OK) { ga_comm_destroy(c); return st; }
        st = ga_comm_alloc(c, sizeof(uint64_t) * world + 64, &flags);
        if (st == GA_OK) {
            DeviceGuard dg(device);
            cudaError_t e = cudaMemset(flags, 0, sizeof(uint64_t) * world + 64);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) st = cuda_fail(e, "comm: zero flags");
        }
        if (st == GA_OK) st = host_barrier(c); // nobody signals before every flag block is zeroed
        if (st != GA_OK) { ga_comm_destroy(c); return st; }
        c->flag_alloc = comm_find(c, flags);
    }
    *comm = c;
    return GA_OK;
}

ga_status ga_comm_alloc(ga_comm *c, size_t bytes, void **local)
{
    if (!c || !local) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    *local = nullptr;
    if (c->device < 0) { set_error("comm has no device (created with device = -1)"); return GA_ERR_INVALID_ARG; }
    DeviceGuard dg(c->device);
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    // every rank must ask for the same size (symmetric)
    std::vector<uint64_t> sizes(c->world);
    const uint64_t mine = bytes;
    ga_status st = host_allgather(c, &mine, sizeof(mine), sizes.data());
    if (st != GA_OK) return st;
    for (int q = 0; q < c->world; ++q)
        if (sizes[q] != mine) { set_error("ga_comm_alloc: ranks asked for different sizes"); return GA_ERR_INVALID_ARG; }
    GaSymAlloc a;
    a.bytes = bytes;
    a.peers.assign(c->world, nullptr);
    cudaError_t e = cudaMalloc(&a.local, bytes);
    // the handle all-gather runs even after a local failure so the other ranks do not hang
    cudaIpcMemHandle_t h{};
    int ok = e == cudaSuccess;
    if (ok && c->world > 1) ok = cudaIpcGetMemHandle(&h, a.local) == cudaSuccess;
    struct Blob { cudaIpcMemHandle_t h; int ok; int pad; };
    Blob b{h, ok, 0};
    std::vector<Blob> all(c->world);
    st = host_allgather(c, &b, sizeof(b), all.data());
    if (st != GA_OK || !ok) {
        if (a.local) cudaFree(a.local);
        if (st == GA_OK) { set_error("ga_comm_alloc: cudaMalloc/IPC handle failed (%zu bytes)", bytes); st = GA_ERR_OOM; }
        return st;
    }
    for (int q = 0; q < c->world; ++q)
        if (!all[q].ok) { cudaFree(a.local); set_error("ga_comm_alloc failed on rank %d", q); return GA_ERR_OOM; }
    a.peers[c->rank] = a.local;
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        void *p = nullptr;
        e = cudaIpcOpenMemHandle(&p, all[q].h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int u = 0; u < q; ++u)
                if (u != c->rank && a.peers[u]) cudaIpcCloseMemHandle(a.peers[u]);
            cudaFree(a.local);
            return cuda_fail(e, "ga_comm_alloc: cudaIpcOpenMemHandle");
        }
        a.peers[q] = static_cast<char *>(p);
    }
    c->allocs.push_back(std::move(a));
    *local = c->allocs.back().local;
    return GA_OK;
}

ga_status ga_comm_free(ga_comm *c, void *local)
{
    if (!c || !local) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    for (auto it = c->allocs.begin(); it != c->allocs.end(); ++it) {
        if (it->local != local) continue;
        if (&*it == c->flag_alloc) { set_error("cannot free the comm's barrier flags"); return GA_ERR_INVALID_ARG; }
        DeviceGuard dg(c->device);
        cudaDeviceSynchronize(); // no kernel of ours still reads the mappings
        ga_status st = sym_free(c, *it);
        c->allocs.erase(it);
        return st;
    }
    set_error("ga_comm_free: %p was not allocated by this comm", local);
    return GA_ERR_INVALID_ARG;
}

ga_status ga_comm_barrier(ga_comm *c, void *stream)
{
    if (!c) { set_error("comm is NULL"); return GA_ERR_INVALID_ARG; }
    DeviceGuard dg(c->device);
    return comm_device_barrier(c, reinterpret_cast<cudaStream_t>(stream));
}

ga_status ga_comm_host_allgather(ga_comm *c, const void *mine, size_t bytes, void *all)
{
    if (!c || (!mine && bytes) || (!all && bytes)) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    return host_allgather(c, mine, bytes, all);
}

ga_status ga_comm_status(ga_comm *c, int *timed_out)
{
    if (!c || !timed_out) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    *timed_out = c->timed_out_host ? *c->timed_out_host : 0;
    return GA_OK;
}

ga_status ga_comm_destroy(ga_comm *c)
{
    if (!c) return GA_OK;
    ga_status st = GA_OK;
    if (c->device >= 0) {
        DeviceGuard dg(c->device);
        cudaDeviceSynchronize();
        for (auto &a : c->allocs) {
            ga_status s2 = sym_free(c, a);
            if (st == GA_OK) st = s2;
        }
        if (c->gather_k) cudaFree(c->gather_k);
        if (c->gather_v) cudaFree(c->gather_v);
        if (c->timed_out_host) cudaFreeHost(const_cast<int *>(c->timed_out_host));
        for (int b = 0; b < 2; ++b) {
            if (c->ring_kv[b]) cudaFree(c->ring_kv[b]);
            if (c->ring_ready[b]) cudaEventDestroy(c->ring_ready[b]);
            if (c->ring_done[b]) cudaEventDestroy(c->ring_done[b]);
        }
        if (c->ring_state) cudaFree(c->ring_state);
        if (c->ring_start) cudaEventDestroy(c->ring_start);
        if (c->ring_end) cudaEventDestroy(c->ring_end);
        if (c->ring_stream) cudaStreamDestroy(c->ring_stream);
    }
    c->allocs.clear();
    close_fds(c);
    delete c;
    return st;
}

} // extern "C"

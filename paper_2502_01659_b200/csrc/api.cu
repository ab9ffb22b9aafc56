// api.cu — the C ABI of libga.so (include/ga.h): validation, dispatch, errors.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "comm.cuh"

namespace ga {

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};

void note_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

void set_error(const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

ga_status cuda_fail(cudaError_t e, const char *where)
{
    set_error("%s: %s", where, cudaGetErrorString(e));
    return GA_ERR_CUDA;
}

static int64_t longnet_levels(int64_t w0, int64_t alpha, int64_t L)
{
    if (w0 > L) return 0;
    int64_t K = 0;
    __int128 seg = w0;
    while (seg * alpha <= L) { seg *= alpha; ++K; }
    return K;
}

// Validate a public ga_mask and convert it to the device descriptor.
static ga_status make_devmask(const ga_mask *m, int64_t L, DevMask &M)
{
    if (!m) { set_error("mask is NULL"); return GA_ERR_INVALID_ARG; }
    if (m->L != L || L <= 0) {
        set_error("mask->L (%lld) must equal L (%lld) > 0", (long long)m->L, (long long)L);
        return GA_ERR_INVALID_ARG;
    }
    if (L > INT32_MAX && (m->kind == GA_MASK_CSR || m->kind == GA_MASK_BIGBIRD)) {
        set_error("explicit CSR uses int32 column indices: L must be < 2^31");
        return GA_ERR_UNSUPPORTED;
    }
    M = DevMask{};
    M.kind = m->kind;
    M.L = L;
    switch (m->kind) {
    case GA_MASK_CSR:
        if (!m->row_ptr || (m->nnz > 0 && !m->col_idx) || m->nnz < 0) {
            set_error("CSR mask needs device row_ptr/col_idx and nnz >= 0");
            return GA_ERR_INVALID_ARG;
        }
        M.row_ptr = m->row_ptr;
        M.col_idx = m->col_idx;
        M.nnz = m->nnz;
        return GA_OK;
    case GA_MASK_WINDOW:
        if (m->w < 1 || m->r < 1) { set_error("window needs w >= 1 and r >= 1"); return GA_ERR_INVALID_ARG; }
        M.w = m->w;
        M.r = m->r;
        M.m = (m->w - 1) / m->r;
        return GA_OK;
    case GA_MASK_LONGNET:
        if (m->w0 < 1 || m->alpha < 2) { set_error("LongNet needs w0 >= 1 and alpha >= 2"); return GA_ERR_INVALID_ARG; }
        if (m->parts < 0 || m->parts > (GA_LONGNET_MULTISET | GA_LONGNET_HEAD_OFFSETS)) {
            set_error("LongNet parts: 0 (set union) or GA_LONGNET_MULTISET, optionally | GA_LONGNET_HEAD_OFFSETS");
            return GA_ERR_INVALID_ARG;
        }
        M.parts = m->parts;
        M.w0 = m->w0;
        M.alpha = m->alpha;
        M.K = longnet_levels(m->w0, m->alpha, L);
        return GA_OK;
    case GA_MASK_BLOCK_DILATED:
        if (m->seg < 1 || m->r < 1) { set_error("block dilation needs seg >= 1, r >= 1"); return GA_ERR_INVALID_ARG; }
        M.seg = m->seg;
        M.r = m->r;
        return GA_OK;
    case GA_MASK_BIGBIRD:
        if (m->w < 1 || m->n_global < 0 || m->n_random < 0 || m->n_global > L || m->r < 0 || m->parts < 0 ||
            m->parts > 7) {
            set_error("BigBird needs w >= 1, 0 <= n_global <= L, n_random >= 0, r >= 0, parts in [0, 7]");
            return GA_ERR_INVALID_ARG;
        }
        M.w = m->w;
        M.r = m->r > 0 ? m->r : 1; // dilated window (0 = 1)
        M.parts = m->parts;
        M.gidx = m->global_idx;
        M.ng = m->n_global;
        M.nrand = m->n_random;
        M.seed = m->seed;
        return GA_OK;
    }
    set_error("unknown mask kind %d", m->kind);
    return GA_ERR_INVALID_ARG;
}

static size_t dtype_bytes(ga_dtype dt) { return dt == GA_F32 ? 4 : 2; }

// Stream-ordered scratch comes from a libga-private memory pool per device (cudaMemPoolCreate),
// whose release threshold is raised so freed blocks stay cached between calls (no re-mapping
// on every synchronisation).  The device's DEFAULT pool is left untouched, so other
// allocators in the process (PyTorch's caching allocator, libraries using cudaMallocAsync)
// see the usual behaviour; ga_scratch_trim() hands the cached blocks back.
static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[64] = {};

static cudaMemPool_t scratch_pool(int dev)
{
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        g_pool[dev] = pool;
    }
    return g_pool[dev];
}

cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t s)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = scratch_pool(dev);
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

cudaError_t scratch_free(void *p, cudaStream_t s) { return p ? cudaFreeAsync(p, s) : cudaSuccess; }

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static const int64_t kDefaultHeavy = 4096;

struct Resolved {
    AttnParams p;
    int64_t heavy;
};

static ga_status resolve(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out, int64_t L,
                         int32_t d, int32_t heads, ga_dtype dtype, const ga_opts *opts, Resolved &R)
{
    if (dtype != GA_F32 && dtype != GA_BF16 && dtype != GA_F16) {
        set_error("dtype %d invalid", (int)dtype);
        return GA_ERR_INVALID_ARG;
    }
    if (d != 32 && d != 64 && d != 128) { set_error("d=%d unsupported (32, 64, 128)", d); return GA_ERR_UNSUPPORTED; }
    if (heads < 1) { set_error("heads must be >= 1"); return GA_ERR_INVALID_ARG; }
    const bool with_state = opts && opts->state.m;
    if (with_state) {
        const ga_state &st = opts->state;
        if (!st.l || !st.o || !aligned16(st.o) || (reinterpret_cast<uintptr_t>(st.m) & 3u) ||
            (reinterpret_cast<uintptr_t>(st.l) & 3u)) {
            set_error("state needs m, l (4-byte aligned) and o (16-byte aligned) device buffers");
            return GA_ERR_INVALID_ARG;
        }
        if (opts->state_mode != GA_STATE_WRITE && opts->state_mode != GA_STATE_ACCUMULATE) {
            set_error("state_mode must be GA_STATE_WRITE or GA_STATE_ACCUMULATE");
            return GA_ERR_INVALID_ARG;
        }
    }
    if (!Q || !K || !V || (!out && !with_state)) {
        set_error("Q, K, V and out (unless a state is requested) must be non-NULL");
        return GA_ERR_INVALID_ARG;
    }
    if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || (out && !aligned16(out))) {
        set_error("Q, K, V, out must be 16-byte aligned");
        return GA_ERR_INVALID_ARG;
    }
    DevMask M;
    ga_status st = make_devmask(mask, L, M);
    if (st != GA_OK) return st;
    ga_opts o{};
    if (opts) o = *opts;
    if (o.q_begin < 0 || o.q_begin > L || o.q_rows < 0 || o.q_begin + o.q_rows > L) {
        set_error("query range [%lld, +%lld) outside [0, L)", (long long)o.q_begin, (long long)o.q_rows);
        return GA_ERR_INVALID_ARG;
    }
    if (o.q_rows == 0) o.q_rows = L - o.q_begin;
    if (o.kv_begin < 0 || o.kv_rows < 0 || o.kv_begin + o.kv_rows > L) {
        set_error("key/value range outside [0, L)");
        return GA_ERR_INVALID_ARG;
    }
    if (o.kv_rows == 0) o.kv_rows = L - o.kv_begin;
    const size_t row_bytes = (size_t)heads * d * dtype_bytes(dtype);
    if (out) { // out must not overlap K or V (it is written while they are read)
        const char *ob = (const char *)out, *oe = ob + (size_t)o.q_rows * row_bytes;
        const char *kb = (const char *)K, *ke = kb + (size_t)o.kv_rows * row_bytes;
        const char *vb = (const char *)V, *ve = vb + (size_t)o.kv_rows * row_bytes;
        if ((ob < ke && kb < oe) || (ob < ve && vb < oe)) {
            set_error("out must not alias K or V");
            return GA_ERR_INVALID_ARG;
        }
        // out may BE Q (every launch sequence reads a row's Q before any launch writes that
        // row's O: tests/test_gpu_contracts.py), but a shifted overlap would overwrite other
        // rows' queries before they are read
        const char *qb = (const char *)Q, *qe = qb + (size_t)o.q_rows * row_bytes;
        if (ob != qb && ob < qe && qb < oe) {
            set_error("out overlaps Q at a different offset (only out == Q is allowed)");
            return GA_ERR_INVALID_ARG;
        }
    }
    AttnParams &p = R.p;
    p = AttnParams{};
    p.Q = Q;
    p.K = K;
    p.V = V;
    p.out = out;
    p.mask = M;
    p.q_begin = o.q_begin;
    p.q_rows = o.q_rows;
    p.kv_begin = o.kv_begin;
    p.kv_rows = o.kv_rows;
    p.H = heads;
    p.d = d;
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
    p.nnz = M.kind == GA_MASK_CSR ? mask->nnz : 0;
    p.edge_counter = o.edge_counter;
    p.row_fingerprint = o.row_fingerprint;
    p.tensor_counter = o.tensor_counter;
    if (with_state) {
        p.state = o.state;
        p.state_mode = o.state_mode;
    }
    R.heavy = o.heavy_threshold > 0 ? o.heavy_threshold : kDefaultHeavy;
    if (M.kind == GA_MASK_BIGBIRD) return bigbird_check(p);
    return GA_OK;
}

// Kernel choice for resolved parameters (shared by ga_attention_ex and the sharded path).
static ga_status dispatch(AttnParams &p, ga_dtype dtype, const ga_opts *opts, int64_t heavy, cudaStream_t s)
{
    const int kernel = opts ? opts->kernel : GA_KERNEL_AUTO;
    const bool probe = p.edge_counter || p.row_fingerprint;
    if (opts && opts->workspace && opts->workspace_bytes > 0) {
        p.workspace = opts->workspace;
        p.workspace_bytes = opts->workspace_bytes;
    }
    ga_status st;
    if (p.mask.kind == GA_MASK_BIGBIRD) { // implicit BigBird / Longformer (bigbird.cu)
        if (probe) { set_error("probes are not supported for implicit BIGBIRD masks (run its CSR)"); return GA_ERR_UNSUPPORTED; }
        if (kernel == GA_KERNEL_TILED) { set_error("no mma.sync band kernel for implicit BIGBIRD masks"); return GA_ERR_UNSUPPORTED; }
        return launch_bigbird(p, dtype, s);
    }
    if (p.state.m) { // carried state: (m, l, o) per (row, head) from the tcgen05 window kernel or the edge kernel
        if (kernel != GA_KERNEL_AUTO && kernel != GA_KERNEL_EDGE && kernel != GA_KERNEL_TC) {
            set_error("a carried state runs on the tcgen05 window kernel or the edge kernel (kernel AUTO, TC or EDGE)");
            return GA_ERR_UNSUPPORTED;
        }
        if (kernel != GA_KERNEL_EDGE && !probe && window_tc_supported(p, dtype)) return launch_window_tc(p, dtype, s);
        // explicit CSR on the mma.sync edge-block kernels (their epilogue merges the state);
        // not with the heavy-row split (whose merge kernels write the output only)
        if (kernel == GA_KERNEL_AUTO && !probe && p.mask.kind == GA_MASK_CSR && !p.kv_clip &&
            csr_mma_supported(p, dtype) && !(opts && opts->workspace && opts->workspace_bytes > 0))
            return launch_csr_mma(p, dtype, s);
        if (kernel == GA_KERNEL_TC) { set_error("tcgen05 path does not support this (mask, dtype, d) with a state"); return GA_ERR_UNSUPPORTED; }
        return launch_edge(p, dtype, s);
    }
    if (p.mask.kind == GA_MASK_CSR) {
        const bool split = opts && opts->workspace && opts->workspace_bytes > 0;
        // bf16/fp16: per-edge products on mma.sync (csr_mma.cu); fp32 and probes: edge kernel
        const bool mma = !probe && (kernel == GA_KERNEL_AUTO || kernel == GA_KERNEL_TILED) && csr_mma_supported(p, dtype);
        if (kernel == GA_KERNEL_TC) { set_error("no tcgen05 kernel for explicit CSR masks"); return GA_ERR_UNSUPPORTED; }
        if (split) {
            if (probe) { set_error("probes are not supported with the heavy-row split"); return GA_ERR_UNSUPPORTED; }
            p.heavy_threshold = heavy;
            st = mma ? launch_csr_mma(p, dtype, s) : launch_edge(p, dtype, s); // light rows
            if (st != GA_OK) return st;
            return launch_csr_heavy(p, dtype, opts->workspace, opts->workspace_bytes, s);
        }
        return mma ? launch_csr_mma(p, dtype, s) : launch_edge(p, dtype, s);
    }
    // the tcgen05 window kernel probes itself for edge_counter (weighted pairs) and
    // tensor_counter (MMA tile products); a row fingerprint needs the instrumented edge kernel
    const bool wtc_probe = p.edge_counter && !p.row_fingerprint;
    if ((!probe || wtc_probe) && (kernel == GA_KERNEL_TC || kernel == GA_KERNEL_AUTO) && window_tc_supported(p, dtype))
        return launch_window_tc(p, dtype, s);
    if (!probe && (kernel == GA_KERNEL_TC || kernel == GA_KERNEL_AUTO) && longnet_tc_supported(p, dtype))
        return launch_longnet_tc(p, dtype, s, /*use_umma=*/true); // tcgen05 groups + mma.sync rest
    if (kernel == GA_KERNEL_TC) { set_error("tcgen05 path does not support this (mask, dtype, d)"); return GA_ERR_UNSUPPORTED; }
    if (!probe && (kernel == GA_KERNEL_TILED || kernel == GA_KERNEL_AUTO)) {
        if (window_tiled_supported(p, dtype)) return launch_window_tiled(p, dtype, s);
        if (longnet_tc_supported(p, dtype)) return launch_longnet_tc(p, dtype, s, /*use_umma=*/false);
    }
    if (kernel == GA_KERNEL_TILED) { set_error("no tiled tensor-core kernel for this (mask, dtype, d)"); return GA_ERR_UNSUPPORTED; }
    return launch_edge(p, dtype, s);
}

} // namespace ga

using namespace ga;

extern "C" {

const char *ga_last_error(void) { return g_err.c_str(); }

unsigned long long ga_launch_count(void) { return g_launches.load(); }

const char *ga_version(void) { return "libga 0.1 (sm_100a; graph-view masked attention, arXiv 2502.01659)"; }

ga_status ga_workspace_size(const ga_mask *mask, int64_t L, int32_t d, int32_t heads, ga_dtype dtype,
                            const ga_opts *opts, size_t *bytes)
{
    if (!bytes) { set_error("bytes is NULL"); return GA_ERR_INVALID_ARG; }
    *bytes = 0;
    DevMask M;
    ga_status st = make_devmask(mask, L, M);
    if (st != GA_OK) return st;
    int64_t q_rows = opts && opts->q_rows > 0 ? opts->q_rows : L - (opts ? opts->q_begin : 0);
    if (M.kind == GA_MASK_LONGNET) { // tcgen05 block-mode partial states (optional: else stream-ordered)
        AttnParams p{};
        p.mask = M;
        p.d = d;
        p.H = heads;
        p.q_begin = opts ? opts->q_begin : 0;
        p.q_rows = q_rows;
        const int s_umma = longnet_umma_levels(p, dtype);
        if (s_umma >= 0 && s_umma < (int)M.K) *bytes = longnet_umma_workspace(p, s_umma + 1);
        return GA_OK;
    }
    if (M.kind == GA_MASK_BIGBIRD) { // window-part state + full-row partials (bigbird.cu)
        AttnParams p{};
        p.mask = M;
        p.d = d;
        p.H = heads;
        p.q_rows = q_rows;
        *bytes = bigbird_workspace(p, dtype);
        return GA_OK;
    }
    if (M.kind != GA_MASK_CSR) return GA_OK;
    int64_t C = opts && opts->heavy_threshold > 0 ? opts->heavy_threshold : kDefaultHeavy;
    *bytes = csr_heavy_workspace(q_rows, L, mask->nnz, heads, d, C);
    return GA_OK;
}

ga_status ga_attention_ex(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out, int64_t L,
                          int32_t d, int32_t heads, ga_dtype dtype, const ga_opts *opts, void *stream)
{
    Resolved R;
    ga_status st = resolve(Q, K, V, mask, out, L, d, heads, dtype, opts, R);
    if (st != GA_OK) return st;
    return dispatch(R.p, dtype, opts, R.heavy, reinterpret_cast<cudaStream_t>(stream));
}

// Ring exchange of K/V for explicit CSR (GA_EXCHANGE_RING): the key
// dimension is cut into the ranks' shards; step s computes this rank's rows against shard
// q = (rank + s) mod world only (edge kernel, kv_clip: each row's slice of sorted columns in
// that range) into a carried state, while the copy stream brings shard q + 1 from its owner
// into the other staging buffer.  Memory per rank: 2 staging buffers of one K + V shard and
// the fp32 state of the local rows, instead of the full-length K and V.
static ga_status sharded_ring(ga_comm *c, const void *Q, const void *K, const void *V, const ga_mask *mask, void *out,
                              int64_t L, int64_t b, int64_t rows, int64_t S, int32_t d, int32_t heads, ga_dtype dtype,
                              const GaSymAlloc *ak, const GaSymAlloc *av, cudaStream_t s)
{
    const size_t rb = (size_t)heads * d * dtype_bytes(dtype);
    const size_t blk = (size_t)S * rb; // K (or V) of one shard
    cudaError_t e = cudaSuccess;
    if (c->ring_bytes < 2 * blk) {
        for (int i = 0; i < 2; ++i) {
            if (c->ring_kv[i]) cudaFree(c->ring_kv[i]);
            c->ring_kv[i] = nullptr;
        }
        c->ring_bytes = 0;
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&c->ring_kv[i], 2 * blk);
        if (e != cudaSuccess) { set_error("ring staging buffers (%zu B): %s", 4 * blk, cudaGetErrorString(e)); return GA_ERR_OOM; }
        c->ring_bytes = 2 * blk;
    }
    const size_t rh = (size_t)rows * heads, a256 = (sizeof(float) * rh + 255) & ~size_t(255);
    const size_t st_bytes = 2 * a256 + sizeof(float) * rh * d;
    if (c->ring_state_bytes < st_bytes) {
        if (c->ring_state) cudaFree(c->ring_state);
        c->ring_state = nullptr;
        c->ring_state_bytes = 0;
        if ((e = cudaMalloc(&c->ring_state, st_bytes)) != cudaSuccess) { set_error("ring state (%zu B): %s", st_bytes, cudaGetErrorString(e)); return GA_ERR_OOM; }
        c->ring_state_bytes = st_bytes;
    }
    if (!c->ring_stream) {
        e = cudaStreamCreateWithFlags(&c->ring_stream, cudaStreamNonBlocking);
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&c->ring_ready[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ring_done[i], cudaEventDisableTiming);
        }
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ring_start, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ring_end, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "ring stream / events");
    }
    char *sb = reinterpret_cast<char *>(c->ring_state);
    ga_state stt{reinterpret_cast<float *>(sb), reinterpret_cast<float *>(sb + a256), reinterpret_cast<float *>(sb + 2 * a256)};
    const size_t koff = (size_t)((const char *)K - ak->local), voff = (size_t)((const char *)V - av->local);
    // the copy stream starts after the entry barrier (every shard complete)
    cudaEventRecord(c->ring_start, s);
    cudaStreamWaitEvent(c->ring_stream, c->ring_start, 0);
    auto shard = [&](int step, int64_t &qb, int64_t &qn) {
        const int q = (c->rank + step) % c->world;
        qb = imin(L, (int64_t)q * S);
        qn = imin(L, qb + S) - qb;
        return q;
    };
    auto prefetch = [&](int step) -> cudaError_t {
        int64_t qb, qn;
        const int q = shard(step, qb, qn);
        if (qn <= 0) return cudaSuccess;
        const int bi = step & 1;
        cudaStreamWaitEvent(c->ring_stream, c->ring_done[bi], 0); // step - 2 finished reading this buffer
        char *dk = static_cast<char *>(c->ring_kv[bi]), *dv = dk + blk;
        cudaError_t ce = cudaMemcpyAsync(dk, ak->peers[q] + koff, (size_t)qn * rb, cudaMemcpyDefault, c->ring_stream);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(dv, av->peers[q] + voff, (size_t)qn * rb, cudaMemcpyDefault, c->ring_stream);
        if (ce == cudaSuccess) ce = cudaEventRecord(c->ring_ready[bi], c->ring_stream);
        return ce;
    };
    ga_status st = GA_OK;
    for (int step = 0; step < c->world && st == GA_OK; ++step) {
        if (step + 1 < c->world && (e = prefetch(step + 1)) != cudaSuccess) { st = cuda_fail(e, "ring copy"); break; }
        int64_t qb, qn;
        shard(step, qb, qn);
        if (qn <= 0) continue;
        const char *kb = (const char *)K, *vb = (const char *)V;
        if (step > 0) {
            kb = static_cast<const char *>(c->ring_kv[step & 1]);
            vb = kb + blk;
            cudaStreamWaitEvent(s, c->ring_ready[step & 1], 0);
        }
        ga_opts oo{};
        oo.q_begin = b;
        oo.q_rows = rows;
        oo.kv_begin = qb;
        oo.kv_rows = qn;
        oo.state = stt;
        oo.state_mode = step == 0 ? GA_STATE_WRITE : GA_STATE_ACCUMULATE;
        Resolved R;
        st = resolve(Q, kb, vb, mask, nullptr, L, d, heads, dtype, &oo, R);
        if (st != GA_OK) break;
        R.p.kv_clip = 1;
        st = launch_edge(R.p, dtype, s);
        cudaEventRecord(c->ring_done[step & 1], s);
    }
    // join the copy stream (its reads of the peers' shards precede the exit barrier)
    cudaEventRecord(c->ring_end, c->ring_stream);
    cudaStreamWaitEvent(s, c->ring_end, 0);
    if (st == GA_OK) st = state_finalize(stt, rows, heads, d, dtype, out, s);
    return st;
}

ga_status ga_attention_sharded(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out, int64_t L,
                               int64_t row_begin, int64_t row_end, int32_t d, int32_t heads, ga_dtype dtype,
                               const ga_opts *opts, ga_comm *comm, void *stream)
{
    if (!comm || !mask) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    if (comm->device < 0) { set_error("comm has no device (created with device = -1)"); return GA_ERR_INVALID_ARG; }
    if (L <= 0) { set_error("L must be > 0"); return GA_ERR_INVALID_ARG; }
    const int64_t S = (L + comm->world - 1) / comm->world;
    const int64_t b = imin(L, (int64_t)comm->rank * S), e = imin(L, b + S);
    if (row_begin != b || row_end != e) {
        set_error("rank %d of %d owns rows [%lld, %lld) of L=%lld (got [%lld, %lld))", comm->rank, comm->world,
                  (long long)b, (long long)e, (long long)L, (long long)row_begin, (long long)row_end);
        return GA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(comm->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t rows = e - b;
    const size_t row_bytes = (size_t)heads * d * dtype_bytes(dtype);
    GaSymAlloc *ak = comm_find(comm, K), *av = comm_find(comm, V);
    if (!ak || !av) { set_error("K and V must live in ga_comm_alloc buffers of this comm"); return GA_ERR_INVALID_ARG; }
    if ((const char *)K + rows * row_bytes > ak->local + ak->bytes ||
        (const char *)V + rows * row_bytes > av->local + av->bytes) {
        set_error("K/V shard overruns its ga_comm_alloc buffer");
        return GA_ERR_INVALID_ARG;
    }
    if (comm->timed_out_host && *comm->timed_out_host) {
        set_error("a device barrier of this comm timed out earlier (a peer stalled): the comm is unusable");
        return GA_ERR_COMM;
    }
    ga_opts o{};
    if (opts) o = *opts;
    ga_status st = comm_device_barrier(comm, s); // every rank's K/V shard is complete
    if (st != GA_OK) return st;
    if (rows > 0) {
        if (mask->kind == GA_MASK_CSR && o.exchange == GA_EXCHANGE_RING && comm->world > 1) {
            if (!out) { set_error("ring exchange needs out"); return GA_ERR_INVALID_ARG; }
            st = sharded_ring(comm, Q, K, V, mask, out, L, b, rows, S, d, heads, dtype, ak, av, s);
        } else if (mask->kind == GA_MASK_CSR || mask->kind == GA_MASK_BIGBIRD) {
            // unstructured columns (explicit CSR, BigBird's random columns): all-gather K and V (copy engines, peer -> local), then a
            // local launch over the full-length buffers
            const size_t full = (size_t)L * row_bytes;
            if (comm->gather_bytes < full) {
                if (comm->gather_k) cudaFree(comm->gather_k);
                if (comm->gather_v) cudaFree(comm->gather_v);
                comm->gather_k = comm->gather_v = nullptr;
                comm->gather_bytes = 0;
                cudaError_t ce = cudaMalloc(&comm->gather_k, full);
                if (ce == cudaSuccess) ce = cudaMalloc(&comm->gather_v, full);
                if (ce != cudaSuccess) { set_error("CSR all-gather buffers (%zu B): %s", 2 * full, cudaGetErrorString(ce)); return GA_ERR_OOM; }
                comm->gather_bytes = full;
            }
            const size_t koff = (size_t)((const char *)K - ak->local), voff = (size_t)((const char *)V - av->local);
            for (int q = 0; q < comm->world; ++q) {
                const int64_t qb = imin(L, (int64_t)q * S), qn = imin(L, qb + S) - qb;
                if (qn <= 0) continue;
                cudaError_t ce = cudaMemcpyAsync((char *)comm->gather_k + qb * row_bytes, ak->peers[q] + koff,
                                                 qn * row_bytes, cudaMemcpyDefault, s);
                if (ce == cudaSuccess)
                    ce = cudaMemcpyAsync((char *)comm->gather_v + qb * row_bytes, av->peers[q] + voff, qn * row_bytes,
                                         cudaMemcpyDefault, s);
                if (ce != cudaSuccess) return cuda_fail(ce, "CSR K/V all-gather");
            }
            o.q_begin = b;
            o.q_rows = rows;
            o.kv_begin = 0;
            o.kv_rows = L;
            st = ga_attention_ex(Q, comm->gather_k, comm->gather_v, mask, out, L, d, heads, dtype, &o, stream);
        } else {
            const char *const *tk = nullptr, *const *tv = nullptr;
            st = comm_peer_table(comm, K, &tk);
            if (st == GA_OK) st = comm_peer_table(comm, V, &tv);
            if (st != GA_OK) return st;
            o.q_begin = b;
            o.q_rows = rows;
            o.kv_begin = b;
            o.kv_rows = rows;
            Resolved R;
            st = resolve(Q, K, V, mask, out, L, d, heads, dtype, &o, R);
            if (st != GA_OK) return st;
            R.p.k_peer = tk;
            R.p.v_peer = tv;
            R.p.shard_rows = S;
            st = dispatch(R.p, dtype, &o, R.heavy, s);
        }
        if (st != GA_OK) return st;
    }
    st = comm_device_barrier(comm, s); // no rank changes its K/V while others still read it
    // a peer that missed either barrier may have left its K/V rows unwritten: poison this
    // rank's output (NaN) instead of returning silently wrong rows
    if (st == GA_OK && out) st = comm_poison_on_timeout(comm, out, (size_t)rows * row_bytes, s);
    return st;
}

ga_status ga_attention_backward(const void *Q, const void *K, const void *V, const void *O, const void *dO,
                                const ga_mask *mask, const float *lse, float *dQ, float *dK, float *dV, int64_t L,
                                int32_t d, int32_t heads, ga_dtype dtype, void *stream)
{
    if (dtype != GA_F32 && dtype != GA_BF16 && dtype != GA_F16) { set_error("dtype %d invalid", (int)dtype); return GA_ERR_INVALID_ARG; }
    if (d != 32 && d != 64 && d != 128) { set_error("d=%d unsupported (32, 64, 128)", d); return GA_ERR_UNSUPPORTED; }
    if (heads < 1) { set_error("heads must be >= 1"); return GA_ERR_INVALID_ARG; }
    if (!Q || !K || !V || !O || !dO || !dQ || !dK || !dV) { set_error("Q, K, V, O, dO, dQ, dK, dV must be non-NULL"); return GA_ERR_INVALID_ARG; }
    for (const void *x : {Q, K, V, O, dO, (const void *)dQ, (const void *)dK, (const void *)dV})
        if (!aligned16(x)) { set_error("all tensors must be 16-byte aligned"); return GA_ERR_INVALID_ARG; }
    if (lse && (reinterpret_cast<uintptr_t>(lse) & 3u)) { set_error("lse must be 4-byte aligned"); return GA_ERR_INVALID_ARG; }
    DevMask M;
    ga_status st = make_devmask(mask, L, M);
    if (st != GA_OK) return st;
    if (M.kind == GA_MASK_BIGBIRD) {
        set_error("backward of an implicit BIGBIRD mask: materialise it with ga_mask_to_csr");
        return GA_ERR_UNSUPPORTED;
    }
    const size_t bytes = (size_t)L * heads * d;
    const char *gb[3] = {(const char *)dQ, (const char *)dK, (const char *)dV};
    for (int a = 0; a < 3; ++a) // the gradients are written while every input is still read
        for (const void *x : {Q, K, V, O, dO}) {
            const char *xb = (const char *)x, *xe = xb + bytes * dtype_bytes(dtype);
            if (gb[a] < xe && xb < gb[a] + bytes * 4) { set_error("dQ, dK, dV must not overlap the inputs"); return GA_ERR_INVALID_ARG; }
        }
    AttnParams p{};
    p.Q = Q;
    p.K = K;
    p.V = V;
    p.mask = M;
    p.q_rows = p.kv_rows = L;
    p.H = heads;
    p.d = d;
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
    p.nnz = M.kind == GA_MASK_CSR ? mask->nnz : 0;
    return attention_backward(p, dtype, O, dO, lse, dQ, dK, dV, reinterpret_cast<cudaStream_t>(stream));
}

ga_status ga_state_finalize(const ga_state *state, int64_t rows, int32_t heads, int32_t d, ga_dtype dtype, void *out,
                            void *stream)
{
    if (!state || !state->l || !state->o || !out) { set_error("state (l, o) and out must be non-NULL"); return GA_ERR_INVALID_ARG; }
    if (rows < 0 || heads < 1 || d < 1) { set_error("rows >= 0, heads >= 1, d >= 1"); return GA_ERR_INVALID_ARG; }
    if (dtype != GA_F32 && dtype != GA_BF16 && dtype != GA_F16) { set_error("dtype invalid"); return GA_ERR_INVALID_ARG; }
    return state_finalize(*state, rows, heads, d, dtype, out, reinterpret_cast<cudaStream_t>(stream));
}

ga_status ga_attention(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out, int64_t L,
                       int32_t d, int32_t heads, ga_dtype dtype, void *stream)
{
    return ga_attention_ex(Q, K, V, mask, out, L, d, heads, dtype, nullptr, stream);
}

// Host-buffer path for Window and CSR masks: the query range is cut into kHostPipeChunks
// aligned chunks (ga_query_alignment, so every row is computed exactly as by one launch).
// Chunk c needs Q rows [b, e) and K/V rows up to e + w (Window: |i - j| < w; CSR: all of
// K/V, copied with chunk 0), so its launch starts as soon as those rows are in; H2D of the
// next chunk, the launch and D2H of the previous output overlap on two copy streams forked
// from and joined back to the caller's stream.
static const int kHostPipeChunks = 8;
static const int64_t kHostPipeMinRows = 4096;

static ga_status host_copy_streams(cudaStream_t *h2d, cudaStream_t *d2h)
{
    static std::mutex mu;
    static cudaStream_t tab[64][2] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess || dev < 0 || dev >= 64) return cuda_fail(e, "ga_attention_host: cudaGetDevice");
    std::lock_guard<std::mutex> g(mu);
    for (int k = 0; k < 2; ++k)
        if (!tab[dev][k] && (e = cudaStreamCreateWithFlags(&tab[dev][k], cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "ga_attention_host: copy stream");
    *h2d = tab[dev][0];
    *d2h = tab[dev][1];
    return GA_OK;
}

static ga_status host_window_pipeline(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out,
                                      int64_t L, int32_t d, int32_t heads, ga_dtype dtype, cudaStream_t s, char *dq,
                                      char *dk, char *dv, char *dout)
{
    cudaStream_t sh, so;
    ga_status st = host_copy_streams(&sh, &so);
    if (st != GA_OK) return st;
    int64_t align = 1;
    if ((st = ga_query_alignment(mask, d, dtype, &align)) != GA_OK) return st;
    if (align < 1) align = 1;
    const size_t rb = (size_t)heads * d * dtype_bytes(dtype);
    int64_t per = (L + kHostPipeChunks - 1) / kHostPipeChunks;
    per = (per + align - 1) / align * align;
    const int nc = (int)((L + per - 1) / per);
    std::vector<cudaEvent_t> ev(2 * nc + 2, nullptr);
    cudaError_t e = cudaSuccess;
    for (auto &x : ev)
        if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) break;
    if (e != cudaSuccess) {
        for (auto x : ev)
            if (x) cudaEventDestroy(x);
        return cuda_fail(e, "ga_attention_host: events");
    }
    cudaEvent_t fork = ev[2 * nc], join = ev[2 * nc + 1];
    // fork: the copy streams start after the caller's prior work and the allocations
    cudaEventRecord(fork, s);
    cudaStreamWaitEvent(sh, fork, 0);
    cudaStreamWaitEvent(so, fork, 0);
    const char *hq = (const char *)Q, *hk = (const char *)K, *hv = (const char *)V;
    int64_t kv_done = 0;
    for (int c = 0; c < nc && st == GA_OK; ++c) {
        const int64_t b = (int64_t)c * per, n = imin(L, b + per) - b;
        // K/V rows [0, need) are on the device once this chunk's copies land (saturating:
        // a huge w must not overflow b + n + w)
        const int64_t need = mask->kind == GA_MASK_CSR || mask->w >= L - (b + n) ? L : b + n + mask->w;
        if ((e = cudaMemcpyAsync(dq + b * rb, hq + b * rb, n * rb, cudaMemcpyHostToDevice, sh)) != cudaSuccess ||
            (need > kv_done &&
             ((e = cudaMemcpyAsync(dk + kv_done * rb, hk + kv_done * rb, (need - kv_done) * rb,
                                   cudaMemcpyHostToDevice, sh)) != cudaSuccess ||
              (e = cudaMemcpyAsync(dv + kv_done * rb, hv + kv_done * rb, (need - kv_done) * rb,
                                   cudaMemcpyHostToDevice, sh)) != cudaSuccess))) {
            st = cuda_fail(e, "ga_attention_host: H2D");
            break;
        }
        kv_done = need;
        cudaEventRecord(ev[2 * c], sh);
        cudaStreamWaitEvent(s, ev[2 * c], 0);
        ga_opts o{};
        o.q_begin = b;
        o.q_rows = n;
        // the launch sees only the rows copied so far: tile loads past `need` (whole 64-key
        // chunks) are zero-filled by TMA instead of reading rows still in flight on the copy
        // stream or uninitialised pool memory (NaN x 0 = NaN)
        o.kv_begin = 0;
        o.kv_rows = need;
        st = ga_attention_ex(dq + b * rb, dk, dv, mask, dout + b * rb, L, d, heads, dtype, &o, s);
        if (st != GA_OK) break;
        cudaEventRecord(ev[2 * c + 1], s);
        cudaStreamWaitEvent(so, ev[2 * c + 1], 0);
        if ((e = cudaMemcpyAsync((char *)out + b * rb, dout + b * rb, n * rb, cudaMemcpyDeviceToHost, so)) !=
            cudaSuccess)
            st = cuda_fail(e, "ga_attention_host: D2H");
    }
    // join: the caller's stream (and the frees enqueued on it) wait for both copy streams
    cudaEventRecord(join, so);
    cudaStreamWaitEvent(s, join, 0);
    cudaEventRecord(ev[2 * nc - 2], sh); // reuse: H2D tail (covers an early break)
    cudaStreamWaitEvent(s, ev[2 * nc - 2], 0);
    for (auto x : ev) cudaEventDestroy(x);
    return st;
}

ga_status ga_attention_host(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out, int64_t L,
                            int32_t d, int32_t heads, ga_dtype dtype, void *stream)
{
    if (!Q || !K || !V || !out) { set_error("host buffers must be non-NULL"); return GA_ERR_INVALID_ARG; }
    if (dtype != GA_F32 && dtype != GA_BF16 && dtype != GA_F16) { set_error("dtype invalid"); return GA_ERR_INVALID_ARG; }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)L * heads * d * dtype_bytes(dtype);
    void *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr;
    cudaError_t e;
    if ((e = scratch_alloc(&dq, bytes, s)) != cudaSuccess || (e = scratch_alloc(&dk, bytes, s)) != cudaSuccess ||
        (e = scratch_alloc(&dv, bytes, s)) != cudaSuccess || (e = scratch_alloc(&dout, bytes, s)) != cudaSuccess) {
        if (dq) cudaFreeAsync(dq, s);
        if (dk) cudaFreeAsync(dk, s);
        if (dv) cudaFreeAsync(dv, s);
        set_error("ga_attention_host: scratch allocation: %s", cudaGetErrorString(e));
        return GA_ERR_OOM;
    }
    ga_status st = GA_OK;
    if (mask && ((mask->kind == GA_MASK_WINDOW && mask->w >= 1) || mask->kind == GA_MASK_CSR) &&
        L >= 2 * kHostPipeMinRows) {
        st = host_window_pipeline(Q, K, V, mask, out, L, d, heads, dtype, s, (char *)dq, (char *)dk, (char *)dv,
                                  (char *)dout);
        cudaFreeAsync(dq, s);
        cudaFreeAsync(dk, s);
        cudaFreeAsync(dv, s);
        cudaFreeAsync(dout, s);
        return st;
    }
    if ((e = cudaMemcpyAsync(dq, Q, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dk, K, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dv, V, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
        st = cuda_fail(e, "ga_attention_host: H2D");
    }
    if (st == GA_OK) st = ga_attention_ex(dq, dk, dv, mask, dout, L, d, heads, dtype, nullptr, stream);
    if (st == GA_OK && (e = cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        st = cuda_fail(e, "ga_attention_host: D2H");
    cudaFreeAsync(dq, s);
    cudaFreeAsync(dk, s);
    cudaFreeAsync(dv, s);
    cudaFreeAsync(dout, s);
    return st;
}

ga_status ga_query_alignment(const ga_mask *mask, int32_t d, ga_dtype dtype, int64_t *tokens)
{
    if (!mask || !tokens) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    DevMask M;
    ga_status st = make_devmask(mask, mask->L, M);
    if (st != GA_OK) return st;
    AttnParams p{};
    p.mask = M;
    p.d = d;
    *tokens = 1;
    p.q_rows = M.L;
    p.kv_rows = M.L;
    if (M.kind == GA_MASK_BIGBIRD) { // its window part runs on the window kernels
        p.mask.kind = GA_MASK_WINDOW;
        p.mask.m = (M.w - 1) / M.r;
    }
    if (window_tc_supported(p, dtype)) *tokens = window_tc_tile_rows() * M.r;
    else if (window_tiled_supported(p, dtype)) *tokens = band_tile_rows() * M.r;
    else if (longnet_tc_supported(p, dtype)) *tokens = M.w0;
    return GA_OK;
}

ga_status ga_mask_count(const ga_mask *pattern, int64_t *nnz_out)
{
    if (!pattern || !nnz_out) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    const int64_t L = pattern->L;
    DevMask M;
    ga_status st = make_devmask(pattern, L, M);
    if (st != GA_OK) return st;
    switch (M.kind) {
    case GA_MASK_CSR: *nnz_out = pattern->nnz; return GA_OK;
    case GA_MASK_WINDOW: { // L + 2 sum_{t=1}^{m'} (L - t r)
        const int64_t mp = imin(M.m, (L - 1) / M.r);
        *nnz_out = L + 2 * (mp * L - M.r * (mp * (mp + 1) / 2));
        return GA_OK;
    }
    case GA_MASK_BLOCK_DILATED: { // sum over segments of ceil(len/r)^2
        int64_t n = 0;
        for (int64_t s0 = 0; s0 < L; s0 += M.seg) {
            const int64_t c = ceil_div(imin(M.seg, L - s0), M.r);
            n += c * c;
        }
        *nnz_out = n;
        return GA_OK;
    }
    case GA_MASK_LONGNET: {
        if (M.parts & GA_LONGNET_HEAD_OFFSETS) {
            set_error("LongNet with per-head offsets has one edge set per head: no single count");
            return GA_ERR_UNSUPPORTED;
        }
        // Per level t and level-t segment [s0,s1): rows with s = min(nu(i),K) == t contribute
        // all U multiples of alpha^t in the segment; rows with s > t contribute the U -
        // ceil(U/alpha) of them whose valuation is exactly t (masks.cuh decomposition).
        auto multiples = [](int64_t a, int64_t b, int64_t q) { // multiples of q in [a, b)
            return (b - 1) / q - (a > 0 ? (a - 1) / q : -1);
        };
        int64_t n = 0, stp = 1;
        for (int64_t t = 0; t <= M.K; ++t) {
            const int64_t segw = M.w0 * stp;
            for (int64_t s0 = 0; s0 < L; s0 += segw) {
                const int64_t s1 = imin(L, s0 + segw);
                const int64_t U = multiples(s0, s1, stp);
                if (M.parts == GA_LONGNET_MULTISET) { // every level's block counted: U x U
                    n += U * U;
                    continue;
                }
                const int64_t gt = t < M.K ? multiples(s0, s1, stp * M.alpha) : 0;
                const int64_t rx = (M.alpha - (s0 / stp) % M.alpha) % M.alpha; // excluded residue
                const int64_t keep = U - (U > rx ? (U - 1 - rx) / M.alpha + 1 : 0);
                n += gt * keep + (U - gt) * U;
            }
            stp *= M.alpha;
        }
        *nnz_out = n;
        return GA_OK;
    }
    case GA_MASK_BIGBIRD: {
        std::vector<int64_t> g;
        if (M.gidx && M.ng > 0) {
            g.resize(M.ng);
            cudaError_t e = cudaMemcpy(g.data(), M.gidx, sizeof(int64_t) * M.ng, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return cuda_fail(e, "ga_mask_count: copy global_idx");
            M.gidx = g.data();
        }
        int64_t n = 0;
        for (int64_t i = 0; i < L; ++i) n += bb_degree(M, i);
        *nnz_out = n;
        return GA_OK;
    }
    }
    set_error("unknown mask kind");
    return GA_ERR_INVALID_ARG;
}

ga_status ga_mask_to_csr(const ga_mask *pattern, int64_t *row_ptr, int32_t *col_idx, void *stream)
{
    if (!pattern || !row_ptr) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    DevMask M;
    ga_status st = make_devmask(pattern, pattern->L, M);
    if (st != GA_OK) return st;
    if (M.kind == GA_MASK_CSR) { set_error("mask is already CSR"); return GA_ERR_INVALID_ARG; }
    if (M.L > INT32_MAX) { set_error("CSR columns are int32: L must be < 2^31"); return GA_ERR_UNSUPPORTED; }
    if (M.kind == GA_MASK_LONGNET && (M.parts & GA_LONGNET_HEAD_OFFSETS)) {
        set_error("LongNet with per-head offsets has one edge set per head: no single CSR");
        return GA_ERR_UNSUPPORTED;
    }
    return maskgen_to_csr(M, row_ptr, col_idx, reinterpret_cast<cudaStream_t>(stream));
}

ga_status ga_mask_validate(const ga_mask *csr, void *stream, int *ok)
{
    if (!csr || !ok) { set_error("NULL argument"); return GA_ERR_INVALID_ARG; }
    *ok = 0;
    if (csr->kind != GA_MASK_CSR) { set_error("not a CSR mask"); return GA_ERR_INVALID_ARG; }
    DevMask M;
    ga_status st = make_devmask(csr, csr->L, M);
    if (st != GA_OK) return st;
    return mask_validate(M, reinterpret_cast<cudaStream_t>(stream), ok);
}

ga_status ga_fill_inputs(void *dst, ga_dtype dtype, int64_t n, uint64_t seed, int32_t tensor, int64_t e0, float shift,
                         void *stream)
{
    if (!dst && n > 0) { set_error("dst is NULL"); return GA_ERR_INVALID_ARG; }
    if (n < 0 || e0 < 0) { set_error("n and e0 must be >= 0"); return GA_ERR_INVALID_ARG; }
    return fill_inputs(dst, dtype, n, seed, tensor, e0, shift, reinterpret_cast<cudaStream_t>(stream));
}

} // extern "C"

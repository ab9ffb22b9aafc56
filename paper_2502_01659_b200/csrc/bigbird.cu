// bigbird.cu — BigBird / Longformer masks as an IMPLICIT descriptor (no materialised CSR):
// window ∪ global rows and columns ∪ random columns (
// readings R8-R10).
//
// The paper runs such a mask either as one CSR call or as "a sequential combination of our
// local, global, and CSR (for random attention) algorithms", the global kernel being
// "global minus local".  Here the composition is one ga_attention call whose three
// launches split the edge set disjointly and merge through the carried online-softmax state
// (the associative (+) of a7):
//
//   1. window part W_i of every row: the tcgen05 window kernel (window_tc.cu) — or the edge
//      kernel when the (w, r, dtype, d) is outside its range — writes the fp32 state
//      (m, l, o~) of each row's window edges into scratch (or the caller's workspace);
//   2. bb_extras_kernel, warp per (row, head) of the non-global rows: the row's extra columns
//      (G \ W_i) ∪ R_i are enumerated on the fly into shared memory — the globals by index
//      arithmetic, the random columns by R10's counter-hash rejection rule evaluated 32
//      candidates per step (first occurrences of valid candidates, in candidate order, so the
//      set equals the sequential rule's and the CSR generator's bit for bit) — then gathered
//      (16-byte K/V row slices, several edges in flight per warp, edge_core.cuh), merged with
//      the row's window state and normalised;
//   3. global rows (degree L: every column) as dense full-row tiles on mma.sync with the key
//      range split across CTAs and (+)-merged (csr_heavy.cu), bf16/fp16 with L % 16 == 0;
//      otherwise the extras kernel walks all L columns of those rows itself.
//
// Every edge of the union is computed exactly once, except the window edges of the g global
// rows (g * |W_i| products, computed by step 1 and superseded by step 3).
#include "edge_core.cuh"

namespace ga {
namespace bb {

constexpr int WARPS = 8;
constexpr int CAP = 1024; // extra columns per row held in shared memory (n_global + n_random)

struct Args {
    ga_state win;    // window-part state from step 1 ([q_rows, H] / [q_rows, H, d] fp32)
    int full_rows;   // global rows are handled by the full-row tiles (skip them here)
};

__device__ __forceinline__ unsigned lanemask_lt(int lane) { return (1u << lane) - 1u; }

// The mask's geometry in 32-bit arithmetic (L < 2^31 for BIGBIRD) with the sorted global list
// staged in shared memory once per CTA: membership tests are a binary search over shared
// memory instead of 64-bit divisions (the evenly spaced default G = {floor(k L / g)}).
struct View {
    const int32_t *G; // shared, ascending
    int32_t ng, L, w, r;
    __device__ __forceinline__ bool in_window(int32_t i, int32_t j) const
    {
        const int32_t d = i > j ? i - j : j - i;
        return d < w && (r == 1 || d % r == 0);
    }
    __device__ __forceinline__ int32_t count_below(int32_t x) const // globals < x
    {
        int32_t lo = 0, hi = ng;
        while (lo < hi) {
            const int32_t mid = (lo + hi) >> 1;
            if (G[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    }
    __device__ __forceinline__ bool is_global(int32_t j) const
    {
        const int32_t k = count_below(j);
        return k < ng && G[k] == j;
    }
    // |W_i U G| (reading R10's exclusion set)
    __device__ __forceinline__ int32_t wg(int32_t i) const
    {
        const int32_t wlo = i - min(i, w - 1), whi = i + min(L - 1 - i, w - 1);
        const int32_t nw = 1 + min(i, w - 1) / r + min(L - 1 - i, w - 1) / r;
        const int32_t a = count_below(wlo), b = count_below(whi + 1);
        int32_t in = b - a;
        if (r > 1) {
            in = 0;
            for (int32_t k = a; k < b; ++k) in += in_window(i, G[k]) ? 1 : 0;
        }
        return nw + (ng - in);
    }
};

// Extra columns of non-global row i — (G \ W_i) if parts has GA_BB_GLOBAL, R_i if it has
// GA_BB_RANDOM — into buf (warp-collective; returns the warp-uniform count).
__device__ int extras(const DevMask &M, const View &V, int parts, int32_t i, int32_t *buf, int lane)
{
    int n = 0;
    if (parts & 2) {
        for (int32_t k0 = 0; k0 < V.ng; k0 += 32) {
            const int32_t k = k0 + lane;
            const int32_t gv = k < V.ng ? V.G[k] : 0;
            const bool keep = k < V.ng && !V.in_window(i, gv);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) buf[n + __popc(bal & lanemask_lt(lane))] = gv;
            n += __popc(bal);
        }
    }
    if ((parts & 4) && M.nrand > 0) {
        const int32_t comp = V.L - V.wg(i); // |complement of W_i U G|
        if (comp <= M.nrand) {              // exhausted: all of the complement (R10)
            for (int32_t j0 = 0; j0 < V.L; j0 += 32) {
                const int32_t j = j0 + lane;
                const bool keep = j < V.L && !V.in_window(i, j) && !V.is_global(j);
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (keep) buf[n + __popc(bal & lanemask_lt(lane))] = j;
                n += __popc(bal);
            }
        } else {
            // R10: candidates c_t, t = 0, 1, ...; c_t is taken iff it lies outside W_i U G and
            // is not already taken — i.e. iff it is the FIRST occurrence of a valid value —
            // until n_random are taken.  32 candidates per step: a lane's candidate is new if
            // it differs from every column taken in earlier steps and from every valid
            // candidate of a lower lane (match_any), and the step's new columns are taken in
            // lane (= candidate) order up to the target.
            const int target = (int)M.nrand;
            const uint64_t base = splitmix64(M.seed);
            int32_t *R = buf + n;
            int got = 0;
            for (uint64_t t0 = 0; got < target; t0 += 32) {
                const int32_t c = (int32_t)bb_candidate(M, base, i, t0 + (uint64_t)lane);
                bool valid = !V.in_window(i, c) && !V.is_global(c);
                for (int q = 0; valid && q < got; ++q)
                    if (R[q] == c) valid = false;
                const unsigned vm = __ballot_sync(0xffffffffu, valid);
                bool first = false;
                if (valid) {
                    const unsigned same = __match_any_sync(vm, c);
                    first = (same & lanemask_lt(lane)) == 0u;
                }
                const unsigned fm = __ballot_sync(0xffffffffu, first);
                const int rank = __popc(fm & lanemask_lt(lane));
                if (first && got + rank < target) R[got + rank] = c;
                __syncwarp();
                got = min(target, got + __popc(fm));
            }
            n += target;
        }
    }
    __syncwarp();
    return n;
}

template <typename T, int D>
__global__ void __launch_bounds__(WARPS * 32) extras_kernel(const __grid_constant__ AttnParams p, const Args a)
{
    __shared__ int32_t cols[WARPS][CAP];
    __shared__ int32_t sG[CAP];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const DevMask &M = p.mask;
    for (int k = threadIdx.x; k < M.ng; k += WARPS * 32) sG[k] = (int32_t)bb_global_at(M, k);
    __syncthreads();
    // |i - j| < L always, so w and r above L act as L (keeps them in 32 bits)
    const View V{sG, (int32_t)M.ng, (int32_t)M.L, (int32_t)imin(M.w, M.L), (int32_t)imin(M.r, M.L)};
    const int64_t gw = (int64_t)blockIdx.x * WARPS + wib;
    const int H = p.H;
    if (gw >= p.q_rows * H) return;
    const int64_t t = gw / H;
    const int h = (int)(gw - t * H);
    const int32_t i = (int32_t)(p.q_begin + t);
    const int parts = M.parts ? M.parts : 7;
    const bool glob = M.ng > 0 && V.is_global(i);
    if (glob && a.full_rows) return;

    EdgeAcc<T, D, false> acc;
    acc.init(p, t, h, lane);
    bool with_window = true;
    if (glob) {
        if (parts & 2) { // a global row attends to every column: W_i U (all \ W_i)
            Piece P;
            P.mode = P_AFFINE;
            P.base = 0;
            P.step = 1;
            P.count = M.L;
            P.alpha = P.rexcl = P.pad = 0;
            P.cols = nullptr;
            acc.run(P, 0, M.L);
            with_window = false;
        } // else: window only (random columns are drawn for non-global rows, R10)
    } else {
        const int n = extras(M, V, parts, i, cols[wib], lane);
        acc.template run_csr<csr_depth<T, D>()>(cols[wib], 0, n);
    }
    acc.merge_groups();
    if (with_window && acc.g == 0) { // (+) the window part's state of this row
        const size_t rh = (size_t)t * H + h;
        const float l2 = a.win.l[rh];
        if (l2 > 0.f) {
            const float m2 = a.win.m[rh];
            const float mn = acc.l > 0.f ? fmaxf(acc.m, m2) : m2;
            const float x = acc.l > 0.f ? ex2(acc.m - mn) : 0.f, y = ex2(m2 - mn);
            const float *so = a.win.o + rh * D + acc.sub * acc.PER;
            acc.l = acc.l * x + l2 * y;
#pragma unroll
            for (int e = 0; e < acc.PER; ++e) acc.o[e] = acc.o[e] * x + so[e] * y;
            acc.m = mn;
        }
    }
    acc.store(p, t, h);
}

// the global rows inside the query range, as local rows (G is sorted): full_row[] and the
// packed count (bits 40-63) the full-row kernels read
__global__ void full_prep_kernel(DevMask M, int64_t q_begin, int64_t q_rows, int64_t *full_row, int64_t *nfull)
{
    const int lane = threadIdx.x;
    int64_t n = 0;
    for (int64_t k0 = 0; k0 < M.ng; k0 += 32) {
        const int64_t k = k0 + lane;
        const int64_t gv = k < M.ng ? bb_global_at(M, k) : -1;
        const bool in = gv >= q_begin && gv < q_begin + q_rows;
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) full_row[n + __popc(bal & lanemask_lt(lane))] = gv - q_begin;
        n += __popc(bal);
    }
    if (lane == 0) *nfull = n << 40;
}

template <typename T> static ga_status launch_extras_d(const AttnParams &p, const Args &a, cudaStream_t s)
{
    const int64_t blocks = (p.q_rows * p.H + WARPS - 1) / WARPS;
    switch (p.d) {
    case 32: extras_kernel<T, 32><<<(unsigned)blocks, WARPS * 32, 0, s>>>(p, a); break;
    case 64: extras_kernel<T, 64><<<(unsigned)blocks, WARPS * 32, 0, s>>>(p, a); break;
    case 128: extras_kernel<T, 128><<<(unsigned)blocks, WARPS * 32, 0, s>>>(p, a); break;
    default: set_error("d=%d unsupported", p.d); return GA_ERR_UNSUPPORTED;
    }
    GA_CHECK_LAUNCH("bb::extras_kernel");
    return GA_OK;
}

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
    size_t m, l, o, full_row, nfull, fpart, total;
    int64_t F;
    bool full_rows;
};

static Layout layout(const AttnParams &p, ga_dtype dt)
{
    Layout y{};
    const size_t rh = (size_t)p.q_rows * p.H;
    const int parts = p.mask.parts ? p.mask.parts : 7;
    y.F = imin(p.mask.ng, p.q_rows);
    y.full_rows = (parts & 2) && y.F > 0 && dt != GA_F32 && p.mask.L % 16 == 0;
    size_t off = 0;
    y.m = off;
    off += align256(sizeof(float) * rh);
    y.l = off;
    off += align256(sizeof(float) * rh);
    y.o = off;
    off += align256(sizeof(float) * rh * p.d);
    y.full_row = off;
    y.nfull = off + align256(sizeof(int64_t) * (size_t)y.F);
    y.fpart = y.nfull + 256;
    if (y.full_rows) off = y.fpart + align256(full_rows_partials_bytes(y.F, p.mask.L, p.H, p.d));
    y.total = off;
    return y;
}

} // namespace bb

ga_status bigbird_check(const AttnParams &p)
{
    const int parts = p.mask.parts ? p.mask.parts : 7;
    if (!(parts & 1)) {
        set_error("implicit BIGBIRD needs the window component in parts (materialise other part sets with ga_mask_to_csr)");
        return GA_ERR_UNSUPPORTED;
    }
    if (((parts & 2) ? p.mask.ng : 0) + ((parts & 4) ? p.mask.nrand : 0) > bb::CAP) {
        set_error("implicit BIGBIRD supports n_global + n_random <= %d per row (use ga_mask_to_csr)", bb::CAP);
        return GA_ERR_UNSUPPORTED;
    }
    if (p.state.m) {
        set_error("implicit BIGBIRD with a carried state: compose its components (parts) instead");
        return GA_ERR_UNSUPPORTED;
    }
    return GA_OK;
}

size_t bigbird_workspace(const AttnParams &p, ga_dtype dt) { return bb::layout(p, dt).total; }

ga_status launch_bigbird(const AttnParams &p, ga_dtype dt, cudaStream_t s)
{
    ga_status st = bigbird_check(p);
    if (st != GA_OK) return st;
    if (p.q_rows == 0) return GA_OK;
    const bb::Layout y = bb::layout(p, dt);
    char *w = nullptr;
    bool owned = false;
    if (p.workspace && p.workspace_bytes >= y.total) {
        w = reinterpret_cast<char *>(p.workspace);
    } else {
        cudaError_t e = scratch_alloc(reinterpret_cast<void **>(&w), y.total, s);
        if (e != cudaSuccess) return cuda_fail(e, "BigBird scratch allocation");
        owned = true;
    }
    bb::Args a{};
    a.win.m = reinterpret_cast<float *>(w + y.m);
    a.win.l = reinterpret_cast<float *>(w + y.l);
    a.win.o = reinterpret_cast<float *>(w + y.o);
    a.full_rows = y.full_rows ? 1 : 0;

    // 1. window part -> state (tcgen05 window kernel when it covers (w, r, dtype, d))
    AttnParams pw = p;
    pw.mask = DevMask{};
    pw.mask.kind = K_WINDOW;
    pw.mask.L = p.mask.L;
    pw.mask.w = p.mask.w;
    pw.mask.r = p.mask.r;
    pw.mask.m = (p.mask.w - 1) / p.mask.r;
    pw.out = nullptr;
    pw.state = a.win;
    pw.state_mode = GA_STATE_WRITE;
    st = window_tc_supported(pw, dt) ? launch_window_tc(pw, dt, s) : launch_edge(pw, dt, s);
    // 2. extra columns of the non-global rows, merged with their window state
    if (st == GA_OK) {
        switch (dt) {
        case GA_F32: st = bb::launch_extras_d<float>(p, a, s); break;
        case GA_BF16: st = bb::launch_extras_d<__nv_bfloat16>(p, a, s); break;
        case GA_F16: st = bb::launch_extras_d<__half>(p, a, s); break;
        }
    }
    // 3. global rows: dense full-row tiles over every column
    if (st == GA_OK && y.full_rows) {
        int64_t *full_row = reinterpret_cast<int64_t *>(w + y.full_row), *nfull = reinterpret_cast<int64_t *>(w + y.nfull);
        bb::full_prep_kernel<<<1, 32, 0, s>>>(p.mask, p.q_begin, p.q_rows, full_row, nfull);
        GA_CHECK_LAUNCH("bb::full_prep_kernel");
        st = launch_full_rows(p, dt, nfull, full_row, reinterpret_cast<float *>(w + y.fpart), y.F, s);
    }
    if (owned) scratch_free(w, s);
    return st;
}

} // namespace ga

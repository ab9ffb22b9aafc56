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
#include "tc_common.cuh"

namespace ga {
namespace bb {

#ifndef GA_BB_DEPTH
#define GA_BB_DEPTH 2
#endif
constexpr int WARPS = 8;
constexpr int CAP = 1024; // extra columns per row held in shared memory (n_global + n_random)
constexpr int BITS = 4096; // per-warp bitmap of the taken random columns (mod BITS)

struct Args {
    ga_state win;    // window-part state from step 1 ([q_rows, H] / [q_rows, H, d] fp32)
    int full_rows;   // global rows are handled by the full-row tiles (skip them here)
    int globals_done; // the global columns were merged into `win` by globals_kernel
};

constexpr int GT_ROWS = 64, GT_THREADS = 128, GT_MAXG = 256; // globals kernel: row tile, threads, max |G|

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
__device__ int extras(const DevMask &M, const View &V, int parts, int32_t i, int32_t *buf, int lane, bool skip_globals,
                      uint32_t *bits)
{
    int n = 0;
    if (parts & 2 && !skip_globals) {
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
            // taken columns also set bit (c mod BITS) of a per-warp bitmap: a candidate whose bit
            // is clear is certainly new (one shared load instead of a scan of the taken list;
            // the scan runs only on a bit collision, ~got / BITS of the candidates)
            for (int k = lane; k < BITS / 32; k += 32) bits[k] = 0u;
            __syncwarp();
            for (uint64_t t0 = 0; got < target; t0 += 32) {
                const int32_t c = (int32_t)bb_candidate(M, base, i, t0 + (uint64_t)lane);
                bool valid = !V.in_window(i, c) && !V.is_global(c);
                if (valid && ((bits[(c & (BITS - 1)) >> 5] >> (c & 31)) & 1u))
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
                if (first && got + rank < target) {
                    R[got + rank] = c;
                    atomicOr(&bits[(c & (BITS - 1)) >> 5], 1u << (c & 31));
                }
                __syncwarp();
                got = min(target, got + __popc(fm));
            }
            n += target;
        }
    }
    __syncwarp();
    return n;
}

#ifndef GA_BB_MINB
#define GA_BB_MINB 4 // CTAs per SM the register allocation targets: 4 -> 64 registers (36 B of spills
                      // in cold paths) 4.44 ms at cfg3i; 3 -> 76, spill-free, 5.32; 5 -> 48, 4.50-4.60;
                      // 6 -> 40, 6.5 (the gathers want warps in flight more than registers)
#endif
template <typename T, int D>
__global__ void __launch_bounds__(WARPS * 32, GA_BB_MINB) extras_kernel(const __grid_constant__ AttnParams p, const Args a)
{
    __shared__ int32_t cols[WARPS][CAP];
    __shared__ int32_t sG[CAP];
    __shared__ uint32_t sbits[WARPS][BITS / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const DevMask &M = p.mask;
    for (int k = threadIdx.x; k < M.ng; k += WARPS * 32) sG[k] = (int32_t)bb_global_at(M, k);
    __syncthreads();
    // |i - j| < L always, so w and r above L act as L (keeps them in 32 bits)
    const View V{sG, (int32_t)M.ng, (int32_t)M.L, (int32_t)imin(M.w, M.L), (int32_t)imin(M.r, M.L)};
    const int64_t gw = (int64_t)blockIdx.x * WARPS + wib;
    const int H = p.H;
    if (gw >= p.q_rows * H) return;
    const int64_t t = div_heads(gw, H);
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
        const int n = extras(M, V, parts, i, cols[wib], lane, a.globals_done != 0, sbits[wib]);
        // edge steps in flight per warp: 2 measured best at cfg3i (4 / 8 cost occupancy)
        acc.template run_csr<GA_BB_DEPTH>(cols[wib], 0, n);
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

// Step 2a (bf16/fp16, |G| <= GT_MAXG): the global COLUMNS of every non-global row on the tensor
// cores.  All rows share the same <= 256 global keys, so (row tile) x (global keys) is a dense
// block, minus the globals inside a row's window (masked to weight 0: those edges belong to
// the window part) and minus the global rows themselves (theirs run as full rows).  CTA = 4
// warps x 16 rows on mma.sync with K_G, V_G staged once in shared memory; each row's partial
// state is (+)-merged into the window state in place.  The extras kernel then gathers only the
// random columns.
template <typename T, int D>
__device__ __forceinline__ void gblock(tc::MmaRows<T, D> &st, const uint32_t *kaddr, const uint32_t *vaddr,
                                       uint32_t off, float sl2, const bool (*valid)[4])
{
    using G = tc::Geo<D>;
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < G::KS; ++kk) {
        uint32_t b0, b1, b2, b3;
        tc::ldsm_x4(kaddr[kk] + off, b0, b1, b2, b3);
        tc::mma16816<T>(sc[0], st.qa[kk], b0, b1);
        tc::mma16816<T>(sc[1], st.qa[kk], b2, b3);
    }
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[nb][e] = valid[nb][e] ? sc[nb][e] : -INFINITY;
    constexpr float kTau = 8.f;
    const float lm0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
    const float lm1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
    const bool need = lm0 * sl2 > st.mr[0] + kTau || lm1 * sl2 > st.mr[1] + kTau;
    if (__any_sync(0xffffffffu, need)) {
        float bm0 = fmaxf(lm0, __shfl_xor_sync(0xffffffffu, lm0, 1));
        bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
        float bm1 = fmaxf(lm1, __shfl_xor_sync(0xffffffffu, lm1, 1));
        bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
        const float mn0 = fmaxf(st.mr[0], bm0 * sl2), mn1 = fmaxf(st.mr[1], bm1 * sl2);
        st.scale_rows(ex2(st.mr[0] - mn0), ex2(st.mr[1] - mn1));
        st.mr[0] = mn0;
        st.mr[1] = mn1;
    }
    uint32_t pa[4];
    st.softmax_pack(sc, sl2, pa); // masked: exp2(-inf) = 0 (the reference max is finite)
#pragma unroll
    for (int jj = 0; jj < G::NB8 / 2; ++jj) {
        uint32_t b0, b1, b2, b3;
        tc::ldsm_x4_t(vaddr[jj] + off, b0, b1, b2, b3);
        tc::mma16816<T>(st.o[2 * jj], pa, b0, b1);
        tc::mma16816<T>(st.o[2 * jj + 1], pa, b2, b3);
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(GT_THREADS) globals_kernel(const __grid_constant__ AttnParams p, const Args a)
{
    using G = tc::Geo<D>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int32_t sG[GT_MAXG];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DevMask &M = p.mask;
    const int ng = (int)M.ng, nb16 = (ng + 15) / 16, h = (int)blockIdx.y;
    const int H = p.H;
    const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sK = sQ + GT_ROWS * G::RB, sV = sK + nb16 * 16 * G::RB;
    const size_t row_bytes = (size_t)H * D * sizeof(T), hoff = (size_t)h * D * sizeof(T);
    for (int k = tid; k < ng; k += GT_THREADS) sG[k] = (int32_t)bb_global_at(M, k);
    // K_G, V_G once per CTA (keys past |G| zero)
    for (int idx = tid; idx < nb16 * 16 * G::NC; idx += GT_THREADS) {
        const int r = idx / G::NC, cc = idx % G::NC;
        if (r < ng) {
            const char *kr, *vr;
            kv_row(p, (int64_t)bb_global_at(M, r), row_bytes, kr, vr);
            tc::cp_async16(sK + tc::swz<D>(r, cc), kr + hoff + cc * 16);
            tc::cp_async16(sV + tc::swz<D>(r, cc), vr + hoff + cc * 16);
        } else {
            tc::sts_zero16(sK + tc::swz<D>(r, cc));
            tc::sts_zero16(sV + tc::swz<D>(r, cc));
        }
    }
    tc::cp_async_commit();
    const int32_t w = (int32_t)imin(M.w, M.L), r = (int32_t)imin(M.r, M.L);
    const float sl2 = p.scale_log2;
    const int g = lane >> 2, t4 = lane & 3;
    uint32_t kaddr[G::KS], vaddr[G::NB8 / 2];
    {
        const int krow = (lane & 7) + (lane >> 4) * 8, vrow = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) kaddr[kk] = sK + tc::swz<D>(krow, 2 * kk + ((lane >> 3) & 1));
#pragma unroll
        for (int jj = 0; jj < G::NB8 / 2; ++jj) vaddr[jj] = sV + tc::swz<D>(vrow, 2 * jj + (lane >> 4));
    }
    const int64_t ntiles = (p.q_rows + GT_ROWS - 1) / GT_ROWS;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t t0 = tile * GT_ROWS;
        const int nrows = (int)imin(GT_ROWS, p.q_rows - t0);
        __syncthreads(); // the previous tile's Q reads are done
        for (int idx = tid; idx < GT_ROWS * G::NC; idx += GT_THREADS) {
            const int rr = idx / G::NC, cc = idx % G::NC;
            if (rr < nrows)
                tc::cp_async16(sQ + tc::swz<D>(rr, cc),
                               reinterpret_cast<const char *>(p.Q) + (size_t)(t0 + rr) * row_bytes + hoff + cc * 16);
            else
                tc::sts_zero16(sQ + tc::swz<D>(rr, cc));
        }
        tc::cp_async_commit();
        tc::cp_async_wait<0>();
        __syncthreads();
        tc::MmaRows<T, D> st;
        st.init_empty();
        st.mr[0] = st.mr[1] = -1e30f; // finite reference: a fully masked block leaves l = 0, no NaN
        st.load_q(sQ, warp * 16, lane);
        // this lane's rows (g, g + 8 of the warp's 16); global rows and pad rows see no key
        int32_t ir[2];
        bool live[2];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            const int rr = warp * 16 + g + 8 * hr;
            ir[hr] = (int32_t)(p.q_begin + t0 + rr);
            bool isg = false;
            for (int k = 0; k < ng && !isg; ++k) isg = sG[k] == ir[hr];
            live[hr] = rr < nrows && !isg;
        }
        for (int b = 0; b < nb16; ++b) {
            bool valid[2][4];
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int k = b * 16 + nb * 8 + 2 * t4 + (e & 1);
                    const int hr = e >> 1;
                    bool ok = live[hr] && k < ng;
                    if (ok) {
                        const int32_t dd = ir[hr] > sG[k] ? ir[hr] - sG[k] : sG[k] - ir[hr];
                        ok = !(dd < w && (r == 1 || dd % r == 0)); // in the window: the window part's edge
                    }
                    valid[nb][e] = ok;
                }
            gblock<T, D>(st, kaddr, vaddr, (uint32_t)(b * 16 * G::RB), sl2, valid);
        }
        st.reduce_l();
        // (+) into the window state of the row, in place
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            if (!live[hr] || !(st.lr[hr] > 0.f)) continue;
            const size_t rh = (size_t)(t0 + warp * 16 + g + 8 * hr) * H + h;
            const float l2 = a.win.l[rh], m2 = a.win.m[rh];
            const float m1 = st.mr[hr], l1 = st.lr[hr];
            const float mn = l2 > 0.f ? fmaxf(m1, m2) : m1;
            const float x = ex2(m1 - mn), y = l2 > 0.f ? ex2(m2 - mn) : 0.f;
            float *so = a.win.o + rh * D;
#pragma unroll
            for (int j = 0; j < G::NB8; ++j) {
                float2 *pp = reinterpret_cast<float2 *>(so + 8 * j + 2 * t4);
                const float2 u = *pp;
                *pp = make_float2(st.o[j][2 * hr] * x + u.x * y, st.o[j][2 * hr + 1] * x + u.y * y);
            }
            if (t4 == 0) {
                a.win.m[rh] = mn;
                a.win.l[rh] = l1 * x + l2 * y;
            }
        }
    }
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

template <typename T, int D> static ga_status launch_globals_t(const AttnParams &p, const Args &a, cudaStream_t s)
{
    using G = tc::Geo<D>;
    const int nb16 = (int)((p.mask.ng + 15) / 16);
    const uint32_t smem = GT_ROWS * G::RB + 2 * nb16 * 16 * G::RB;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(globals_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             GT_ROWS * G::RB + 2 * GT_MAXG * G::RB);
        attr = true;
    }
    const int64_t ntiles = (p.q_rows + GT_ROWS - 1) / GT_ROWS;
    const unsigned gx = (unsigned)imin(ntiles, 148 * 8);
    globals_kernel<T, D><<<dim3(gx, (unsigned)p.H), GT_THREADS, smem, s>>>(p, a);
    GA_CHECK_LAUNCH("bb::globals_kernel");
    return GA_OK;
}

static ga_status launch_globals(const AttnParams &p, const Args &a, ga_dtype dt, cudaStream_t s)
{
    switch (p.d) {
    case 32: return dt == GA_BF16 ? launch_globals_t<__nv_bfloat16, 32>(p, a, s) : launch_globals_t<__half, 32>(p, a, s);
    case 64: return dt == GA_BF16 ? launch_globals_t<__nv_bfloat16, 64>(p, a, s) : launch_globals_t<__half, 64>(p, a, s);
    case 128: return dt == GA_BF16 ? launch_globals_t<__nv_bfloat16, 128>(p, a, s) : launch_globals_t<__half, 128>(p, a, s);
    }
    set_error("d=%d unsupported", p.d);
    return GA_ERR_UNSUPPORTED;
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
    // 2a. global columns on the tensor cores (bf16/fp16, |G| <= GT_MAXG), merged into the state
    const int parts = p.mask.parts ? p.mask.parts : 7;
    if (st == GA_OK && (parts & 2) && p.mask.ng > 0 && p.mask.ng <= bb::GT_MAXG && dt != GA_F32) {
        a.globals_done = 1;
        st = bb::launch_globals(p, a, dt, s);
    }
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

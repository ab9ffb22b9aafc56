// longnet_tc.cu — tensor-core kernel for LongNet masks (bf16 / fp16).
//
// The LongNet mask (reading R11: OR over levels k <= K of BlockDilated(w0 a^k, a^k), PAPER.md
// :138, :181) is a disjoint union of DENSE blocks on strided index sets:
// a row i with s = min(nu_a(i), K) has the neighbour pieces
//     t < s : { j in seg_t(i) : nu(j) == t }        (masks.cuh SKIPMUL piece)
//     t = s : { j in seg_s(i) : a^s | j }           (masks.cuh AFFINE piece)
// and seg_t(i) only depends on the level-0 segment sigma0 containing i.  Hence every row of
// the group G(sigma0, s) = { i in sigma0 : min(nu(i), K) = s } has EXACTLY the same neighbour
// set: (group rows) x (concatenated pieces) is a fully dense block — tensor-core work with no
// masked-out pair and no triangles.
//
// A CTA takes <= 64 rows of one group (4 warps x 16 rows).  Groups with fewer rows (high s:
// few rows, many keys) split the key blocks across warps and merge the partial (m, l, O)
// states at the end.  Keys stream through a double-buffered cp.async ring (64 keys per
// stage); each 16-key block is one mma.sync S = Q K^T + online softmax + O += P V step
// (tc::MmaRows::block16).  A ragged tail of < 16 keys (general w0) runs on CUDA cores.
#include "tc_common.cuh"

namespace ga {
namespace lnet {
using namespace tc;

constexpr int WARPS = 4;
constexpr int ROWS = 16 * WARPS;
constexpr int THREADS = 32 * WARPS;
constexpr int KC = 64;       // keys per stage
constexpr int MAX_ITEMS = 96;
constexpr int MAX_PIECES = 64;

struct LParams {
    AttnParams p;
    int64_t seg0;                 // first level-0 segment overlapping the query range
    int64_t n_seg;                // level-0 segments
    int32_t n_items;              // (s, tile) work items per segment
    int16_t item_s[MAX_ITEMS];
    int16_t item_tile[MAX_ITEMS];
};

template <int D> __host__ __device__ constexpr uint32_t smem_bytes()
{
    static_assert(WARPS * 16 * (D + 2) * 4 <= 4 * KC * Geo<D>::RB, "scratch must fit the stages");
    return (uint32_t)(ROWS * Geo<D>::RB               // Q tile / output staging
                      + 2 * 2 * KC * Geo<D>::RB        // K and V, two stages (then scratch)
                      + ROWS * 8);                     // row list
}

template <typename T, int D>
__global__ void __launch_bounds__(THREADS) longnet_kernel(const LParams lp)
{
    using G = Geo<D>;
    extern __shared__ __align__(128) unsigned char smem[];
    const AttnParams &p = lp.p;
    const DevMask &M = p.mask;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int H = p.H;

    // ---- work item: segment-major (a segment's groups share its level-0 keys, so they run
    // together while those K/V rows are in L2), heaviest group first within a segment
    const int64_t IH = (int64_t)lp.n_items * H;
    const int64_t segl = (int64_t)blockIdx.x / IH;
    const int64_t rem = (int64_t)blockIdx.x - segl * IH;
    const int64_t item = rem / H;
    const int h = (int)(rem - item * H);
    const int64_t seg = lp.seg0 + segl;
    const int s = lp.item_s[item], tile = lp.item_tile[item];
    const int64_t S0 = seg * M.w0, S1 = imin(M.L, S0 + M.w0);
    const int64_t q_end = p.q_begin + p.q_rows;

    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sQ = sbase;
    const uint32_t sK0 = sQ + ROWS * G::RB;                 // stage st: sK0 + st*KC*RB
    const uint32_t sV0 = sK0 + 2 * KC * G::RB;
    // split-merge / ragged-tail scratch aliases the K/V stages (used only after the key loop)
    float *scratch = reinterpret_cast<float *>(smem + ROWS * G::RB);
    int64_t *rows = reinterpret_cast<int64_t *>(smem + ROWS * G::RB + 4 * KC * G::RB);

    // ---- rows of G(seg, s) inside the query range, ranks [64*tile, 64*tile + 64), in closed
    // form: candidates are the multiples i = a^s (f0 + q) in [lo, hi); for s < K the group
    // keeps those with a !| (f0 + q) (one excluded residue of q, as in a SKIPMUL piece) —
    // except i = 0, whose valuation is K by convention; for s = K it keeps every candidate.
    int64_t step = 1;
    for (int t = 0; t < s; ++t) step *= M.alpha;
    const int64_t lo = imax(S0, p.q_begin), hi = imin(S1, q_end);
    const int64_t f0 = (lo + step - 1) / step;
    const int64_t nq = lo < hi && f0 * step < hi ? (hi - 1) / step - f0 + 1 : 0;
    const bool top = s == (int)M.K;
    const int64_t rx = (M.alpha - f0 % M.alpha) % M.alpha; // excluded residue of q (s < K)
    // i = 0 (valuation K) sits at q = 0 when f0 == 0; its residue is the excluded one, so the
    // s < K groups drop it automatically and the s = K group keeps it
    const int64_t count = top ? nq : nq - (nq > rx ? (nq - 1 - rx) / M.alpha + 1 : 0);
    const int nrows = (int)imin(ROWS, count - (int64_t)tile * ROWS);
    if (nrows <= 0) return;
    if (tid < nrows) {
        const int64_t r = (int64_t)tile * ROWS + tid;
        int64_t q = r;
        if (!top) {
            const int64_t a1 = M.alpha - 1, idx = r % a1;
            q = (r / a1) * M.alpha + (idx < rx ? idx : idx + 1);
        }
        rows[tid] = (f0 + q) * step;
    }
    __syncthreads();

    // ---- neighbour pieces shared by the whole group (masks.cuh), from a representative row,
    // cached in shared memory with their prefix offsets
    __shared__ Piece spiece[MAX_PIECES];
    __shared__ int pstart[MAX_PIECES + 1]; // key offsets of the pieces (a group has < 2^31 keys)
    const int64_t irep = rows[0];
    const int np = s + 1;
    if (tid < np) spiece[tid] = get_piece(M, irep, tid);
    __syncthreads();
    if (tid == 0) {
        pstart[0] = 0;
        for (int t = 0; t < np; ++t) pstart[t + 1] = pstart[t] + (int)spiece[t].count;
    }
    __syncthreads();
    const int64_t nkeys = pstart[np];
    const int64_t nblk = nkeys / 16;         // dense 16-key blocks (tensor cores)
    const int ragged = (int)(nkeys - nblk * 16);
    const int64_t nchunks = (nblk * 16 + KC - 1) / KC;

    const size_t row_bytes = (size_t)H * D * sizeof(T);
    const char *Qg = reinterpret_cast<const char *>(p.Q) + (size_t)h * D * sizeof(T);
    const size_t hoff = (size_t)h * D * sizeof(T);

    auto key_token = [&](int k) -> int64_t { // k-th key of the concatenated pieces
        int t = 0;
        while (t + 1 < np && pstart[t + 1] <= k) ++t;
        return piece_at(spiece[t], k - pstart[t]);
    };
    // per-thread piece cursor: a thread's key index only grows (by KC per stage)
    int cur_t = 0;
    auto load_chunk = [&](int64_t c, int st) {
        // 2 threads per key: each moves half of the K row and half of the V row
        const int kl = tid >> 1, hf = tid & 1;
        const int k = (int)(c * KC) + kl;
        if (k < nblk * 16) {
            while (cur_t + 1 < np && pstart[cur_t + 1] <= k) ++cur_t;
            const char *kr, *vr;
            kv_row(p, piece_at(spiece[cur_t], k - pstart[cur_t]), row_bytes, kr, vr);
#pragma unroll
            for (int q = 0; q < G::HC; ++q) {
                const int cc = hf * G::HC + q;
                cp_async16(sK0 + st * KC * G::RB + swz<D>(kl, cc), kr + hoff + cc * 16);
                cp_async16(sV0 + st * KC * G::RB + swz<D>(kl, cc), vr + hoff + cc * 16);
            }
        }
    };

    // Q rows of the tile, then the first two key stages.  Pad rows of the last 16-row slice
    // are zeroed: they take part in the warp's rescale vote, so stale shared memory there
    // would change the rounding of the valid rows from launch to launch.
    for (int idx = tid; idx < ((nrows + 15) & ~15) * G::NC; idx += THREADS) {
        const int r = idx / G::NC, cc = idx % G::NC;
        if (r < nrows)
            cp_async16(sQ + swz<D>(r, cc), Qg + (size_t)(rows[r] - p.q_begin) * row_bytes + cc * 16);
        else
            sts_zero16(sQ + swz<D>(r, cc));
    }
    if (nchunks > 0) load_chunk(0, 0);
    cp_async_commit();
    if (nchunks > 1) load_chunk(1, 1);
    cp_async_commit();

    // ---- warp roles: S row slices of 16, P key splits per slice
    const int S = (nrows + 15) / 16;
    const int P = S == 1 ? 4 : S == 2 ? 2 : 1;
    const int slice = warp / P, split = warp % P;
    const bool active = slice < S;
    const float sl2 = p.scale_log2;

    MmaRows<T, D> st;
    st.init_empty();
    cp_async_wait<1>();
    __syncthreads();
    if (active) st.load_q(sQ, slice * 16, lane);

    // per-lane ldmatrix addresses inside a stage (block b of the stage adds b*16 rows)
    uint32_t kaddr[G::KS], vaddr[G::NB8 / 2];
    {
        const int krow = (lane & 7) + (lane >> 4) * 8, vrow = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) kaddr[kk] = sK0 + swz<D>(krow, 2 * kk + ((lane >> 3) & 1));
#pragma unroll
        for (int jj = 0; jj < G::NB8 / 2; ++jj) vaddr[jj] = sV0 + swz<D>(vrow, 2 * jj + (lane >> 4));
    }

    for (int64_t c = 0; c < nchunks; ++c) {
        const int stg = (int)(c & 1);
        if (c > 0) { // chunk c landed (one younger group may still be in flight)
            cp_async_wait<1>();
            __syncthreads();
        }
        if (active) {
            const int blocks_here = (int)imin(KC / 16, nblk - c * (KC / 16));
            const uint32_t soff = (uint32_t)(stg * KC * G::RB);
            int b = split;
            for (; b + P < blocks_here; b += 2 * P) // pairs: one vote and one rescale check
                st.block16x2(kaddr, vaddr, soff + b * 16 * G::RB, soff + (b + P) * 16 * G::RB, sl2);
            if (b < blocks_here) st.block16(kaddr, vaddr, soff + b * 16 * G::RB, sl2);
        }
        __syncthreads(); // stage stg free
        if (c + 2 < nchunks) load_chunk(c + 2, stg);
        cp_async_commit();
    }
    cp_async_wait<0>();
    // ragged tail (< 16 keys, every one valid for every row): CUDA cores, two lanes per row,
    // merged into the MMA state through this warp's scratch (split 0 only; the scratch
    // aliases the now idle K/V stages)
    if (ragged > 0 && active && split == 0) {
        const int x = lane >> 1, hf = lane & 1;
        const bool row_ok = slice * 16 + x < nrows;
        const char *qrow = Qg + (size_t)((row_ok ? rows[slice * 16 + x] : rows[0]) - p.q_begin) * row_bytes;
        float sc[16], mc = -INFINITY, lc = 0.f, oc[D / 2];
#pragma unroll
        for (int e = 0; e < D / 2; ++e) oc[e] = 0.f;
        uint32_t qv[G::HC * 4];
#pragma unroll
        for (int q = 0; q < G::HC; ++q) {
            const uint4 u = ldg16(qrow + (hf * G::HC + q) * 16);
            qv[4 * q] = u.x; qv[4 * q + 1] = u.y; qv[4 * q + 2] = u.z; qv[4 * q + 3] = u.w;
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t >= ragged) break;
            const char *kr, *vr_unused;
            kv_row(p, key_token(nblk * 16 + t), row_bytes, kr, vr_unused);
            kr += hoff;
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int q = 0; q < G::HC; ++q) {
                const uint4 u = ldg16(kr + (hf * G::HC + q) * 16);
                s0 = fma2h<T>(qv[4 * q], u.x, s0);
                s1 = fma2h<T>(qv[4 * q + 1], u.y, s1);
                s0 = fma2h<T>(qv[4 * q + 2], u.z, s0);
                s1 = fma2h<T>(qv[4 * q + 3], u.w, s1);
            }
            float sv = s0 + s1;
            sv += __shfl_xor_sync(0xffffffffu, sv, 1);
            sc[t] = sv * sl2;
            mc = fmaxf(mc, sc[t]);
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t >= ragged) break;
            const float pr = ex2(sc[t] - mc);
            lc += pr;
            const char *kr_unused, *vr;
            kv_row(p, key_token(nblk * 16 + t), row_bytes, kr_unused, vr);
            vr += hoff;
            const uint32_t p2 = pack2<T>(pr, pr);
#pragma unroll
            for (int q = 0; q < G::HC; ++q) {
                const uint4 u = ldg16(vr + (hf * G::HC + q) * 16);
                axpy2h<T>(p2, u.x, oc[8 * q + 0], oc[8 * q + 1]);
                axpy2h<T>(p2, u.y, oc[8 * q + 2], oc[8 * q + 3]);
                axpy2h<T>(p2, u.z, oc[8 * q + 4], oc[8 * q + 5]);
                axpy2h<T>(p2, u.w, oc[8 * q + 6], oc[8 * q + 7]);
            }
        }
        float *srow = scratch + warp * 16 * (D + 2) + x * (D + 2);
#pragma unroll
        for (int e = 0; e < D / 2; ++e) srow[2 + hf * (D / 2) + e] = oc[e];
        if (hf == 0) { srow[0] = mc; srow[1] = lc; }
        __syncwarp();
        const int g = lane >> 2, t4 = lane & 3;
        const float *r0 = scratch + warp * 16 * (D + 2) + g * (D + 2), *r1 = r0 + 8 * (D + 2);
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) { // (m,l,o) (+) (m2,l2,o2)
            const float *rw = hr == 0 ? r0 : r1;
            const float m2 = rw[0], l2 = t4 == 0 ? rw[1] : 0.f;
            const float mn = fmaxf(st.mr[hr], m2);
            const float a = st.mr[hr] == -INFINITY ? 0.f : ex2(st.mr[hr] - mn);
            const float b = m2 == -INFINITY ? 0.f : ex2(m2 - mn);
            st.lr[hr] = st.lr[hr] * a + l2 * b;
#pragma unroll
            for (int j = 0; j < G::NB8; ++j) {
                st.o[j][2 * hr] = st.o[j][2 * hr] * a + rw[2 + 8 * j + 2 * t4] * b;
                st.o[j][2 * hr + 1] = st.o[j][2 * hr + 1] * a + rw[2 + 8 * j + 2 * t4 + 1] * b;
            }
            st.mr[hr] = mn;
        }
        __syncwarp();
    }


    // ---- merge key splits, normalise, stage through the Q rows, store
    const int g = lane >> 2, t4 = lane & 3;
    if (active) st.reduce_l();
    if (P > 1) {
        if (active && split > 0) {
            float *sw = scratch + warp * 16 * (D + 2);
            if (t4 == 0) { sw[g * (D + 2)] = st.mr[0]; sw[(g + 8) * (D + 2)] = st.mr[1];
                           sw[g * (D + 2) + 1] = st.lr[0]; sw[(g + 8) * (D + 2) + 1] = st.lr[1]; }
#pragma unroll
            for (int j = 0; j < G::NB8; ++j) {
                sw[g * (D + 2) + 2 + 8 * j + 2 * t4] = st.o[j][0];
                sw[g * (D + 2) + 2 + 8 * j + 2 * t4 + 1] = st.o[j][1];
                sw[(g + 8) * (D + 2) + 2 + 8 * j + 2 * t4] = st.o[j][2];
                sw[(g + 8) * (D + 2) + 2 + 8 * j + 2 * t4 + 1] = st.o[j][3];
            }
        }
        __syncthreads();
        if (active && split == 0) {
            for (int q = 1; q < P; ++q) {
                const float *sw = scratch + (warp + q) * 16 * (D + 2);
#pragma unroll
                for (int hr = 0; hr < 2; ++hr) {
                    const float *rw = sw + (g + 8 * hr) * (D + 2);
                    const float m2 = rw[0], l2 = rw[1];
                    const float mn = fmaxf(st.mr[hr], m2);
                    const float a = st.mr[hr] == -INFINITY ? 0.f : ex2(st.mr[hr] - mn);
                    const float b = m2 == -INFINITY ? 0.f : ex2(m2 - mn);
                    st.lr[hr] = st.lr[hr] * a + l2 * b;
#pragma unroll
                    for (int j = 0; j < G::NB8; ++j) {
                        st.o[j][2 * hr] = st.o[j][2 * hr] * a + rw[2 + 8 * j + 2 * t4] * b;
                        st.o[j][2 * hr + 1] = st.o[j][2 * hr + 1] * a + rw[2 + 8 * j + 2 * t4 + 1] * b;
                    }
                    st.mr[hr] = mn;
                }
            }
        }
    }
    if (!active || split != 0) return;
    const float inv0 = st.lr[0] > 0.f ? 1.f / st.lr[0] : 0.f, inv1 = st.lr[1] > 0.f ? 1.f / st.lr[1] : 0.f;
    const int r0 = slice * 16;
#pragma unroll
    for (int j = 0; j < G::NB8; ++j) {
        const uint32_t w0 = pack2<T>(st.o[j][0] * inv0, st.o[j][1] * inv0);
        const uint32_t w1 = pack2<T>(st.o[j][2] * inv1, st.o[j][3] * inv1);
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sQ + swz<D>(r0 + g, j) + 4 * t4), "r"(w0));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sQ + swz<D>(r0 + g + 8, j) + 4 * t4), "r"(w1));
    }
    __syncwarp();
    char *Og = reinterpret_cast<char *>(p.out) + (size_t)h * D * sizeof(T);
    for (int idx = lane; idx < 16 * G::NC; idx += 32) {
        const int r = idx / G::NC, cc = idx % G::NC;
        if (r0 + r >= nrows) continue;
        stg16(Og + (size_t)(rows[r0 + r] - p.q_begin) * row_bytes + cc * 16, lds16(sQ + swz<D>(r0 + r, cc)));
    }
}

template <typename T, int D> static ga_status launch_t(const LParams &lp, cudaStream_t s)
{
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(longnet_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem_bytes<D>());
        if (e != cudaSuccess) return cuda_fail(e, "longnet_kernel: set smem");
        configured = true;
    }
    const int64_t blocks = (int64_t)lp.n_items * lp.n_seg * lp.p.H;
    if (blocks == 0) return GA_OK;
    longnet_kernel<T, D><<<(unsigned)blocks, THREADS, smem_bytes<D>(), s>>>(lp);
    GA_CHECK_LAUNCH("longnet_kernel");
    return GA_OK;
}

} // namespace lnet

bool longnet_tc_supported(const AttnParams &p, ga_dtype dt)
{
    if (p.mask.kind != K_LONGNET || (dt != GA_BF16 && dt != GA_F16)) return false;
    if (p.mask.parts != 0) return false; // multiset (overlapping pieces) / per-head offsets: edge kernel
    return p.mask.K + 1 <= lnet::MAX_PIECES && p.mask.w0 >= 16;
}

ga_status launch_longnet_umma(const AttnParams &p, ga_dtype dt, int64_t seg0, int64_t n_seg, int s_max,
                              float *partials, cudaStream_t s);
size_t longnet_umma_workspace(const AttnParams &p, int h0);

// groups s = 0..s_umma fill 128-row tiles (about w0/a^t - w0/a^(t+1) rows): tcgen05 group
// mode; -1 when none does (then the mma.sync kernel takes every group)
int longnet_umma_levels(const AttnParams &p, ga_dtype dt)
{
    const DevMask &M = p.mask;
    int s_umma = -1;
    if (p.d == 64 && (dt == GA_BF16 || dt == GA_F16)) {
        int64_t st2 = 1;
        for (int t = 0; t <= M.K; ++t) {
            const int64_t rows_t = t < M.K ? M.w0 / st2 - M.w0 / (st2 * M.alpha) : M.w0 / st2;
            if (rows_t < 128) break;
            s_umma = t;
            st2 *= M.alpha;
        }
    }
    return s_umma;
}

ga_status launch_longnet_tc(const AttnParams &p, ga_dtype dt, cudaStream_t s, bool use_umma)
{
    lnet::LParams lp;
    lp.p = p;
    const DevMask &M = p.mask;
    // segments overlapping the query range
    const int64_t seg_lo = p.q_begin / M.w0, seg_hi = (p.q_begin + p.q_rows + M.w0 - 1) / M.w0;
    lp.seg0 = seg_lo;
    lp.n_seg = seg_hi - seg_lo;
    // work items (s, tile), heaviest first: group sizes are bounded by the count of
    // multiples of a^s in a segment
    int n = 0;
    int64_t stp = 1;
    int64_t cnt[lnet::MAX_PIECES];
    for (int t = 0; t <= M.K; ++t) {
        cnt[t] = M.w0 / stp + 1;
        stp *= M.alpha;
    }
    // tcgen05: groups s <= s_umma in group mode, the rows with s > s_umma block-wise with
    // partial states (workspace: the caller's, else stream-ordered) and a merge
    const int s_umma = use_umma ? longnet_umma_levels(p, dt) : -1;
    int s_done = s_umma; // groups s > s_done still need the mma.sync kernel
    if (s_umma >= 0) {
        float *partials = nullptr;
        bool owned = false;
        if (s_umma < (int)M.K) {
            const size_t need = longnet_umma_workspace(p, s_umma + 1);
            if (p.workspace && p.workspace_bytes >= need) {
                partials = reinterpret_cast<float *>(p.workspace);
            } else {
                void *w = nullptr;
                cudaError_t e = scratch_alloc((void **)&w, need, s);
                if (e != cudaSuccess) return cuda_fail(e, "LongNet partials: scratch allocation");
                partials = reinterpret_cast<float *>(w);
                owned = true;
            }
        }
        ga_status st = launch_longnet_umma(p, dt, lp.seg0, lp.n_seg, s_umma, partials, s);
        if (owned) scratch_free(partials, s);
        if (st != GA_OK) return st;
        s_done = (int)M.K;
    }
    for (int t = (int)M.K; t > s_done; --t) {
        const int64_t tiles = (cnt[t] + lnet::ROWS - 1) / lnet::ROWS;
        for (int64_t k = 0; k < tiles; ++k) {
            if (n >= lnet::MAX_ITEMS) { set_error("LongNet: too many work items"); return GA_ERR_UNSUPPORTED; }
            lp.item_s[n] = (int16_t)t;
            lp.item_tile[n] = (int16_t)k;
            ++n;
        }
    }
    lp.n_items = n;
    if (n == 0) return GA_OK;
    if ((int64_t)n * lp.n_seg * p.H > (int64_t)INT32_MAX) { set_error("LongNet grid too large"); return GA_ERR_UNSUPPORTED; }
    if (dt == GA_BF16) {
        switch (p.d) {
        case 32: return lnet::launch_t<__nv_bfloat16, 32>(lp, s);
        case 64: return lnet::launch_t<__nv_bfloat16, 64>(lp, s);
        case 128: return lnet::launch_t<__nv_bfloat16, 128>(lp, s);
        }
    } else {
        switch (p.d) {
        case 32: return lnet::launch_t<__half, 32>(lp, s);
        case 64: return lnet::launch_t<__half, 64>(lp, s);
        case 128: return lnet::launch_t<__half, 128>(lp, s);
        }
    }
    set_error("LongNet kernel: unsupported d");
    return GA_ERR_UNSUPPORTED;
}

} // namespace ga

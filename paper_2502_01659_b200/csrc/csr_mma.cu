// csr_mma.cu — explicit-CSR graph attention for bf16/fp16 with the per-edge dot products
// and the aggregation on mma.sync (K2).
//
// Algorithm 1 for one (query row i, head h) per warp, the neighbours
// j in col_idx[row_ptr[i] .. row_ptr[i+1]) taken 16 at a time:
//
//   W = Q_i . K_j  as S^T = K_blk q^T, an m16n8k16 MMA per 16 dims with the
//                  16 edges on M and q replicated in all 8 columns of B, so every lane's C
//                  fragment holds the scores of its two edges (g, g+8) without a shuffle;
//   m, l           online softmax in the exp2 domain (score * log2(e)/sqrt(d), Eq. 1 /
//                  reading R4), lazy rescale when the block max exceeds m by > 2^8;
//   O += p V_j as O^T = V_blk^T P^T with the 16 edges on K: lane
//                  (g, t) puts p of its edge g (or g+8) into column g of P^T only where that
//                  column meets row 2t / 2t+1 (resp. +8), zeros elsewhere, so the 8 columns
//                  of O^T are partial sums of disjoint edge sets — summed once per row at
//                  the end.  No shuffle on the per-block path.
//
// Operands come straight from global memory into MMA fragments (no shared memory): the
// d dimension is permuted consistently in K and q (lane t's 16-byte-aligned slice of a K row
// feeds k-step s through words 2s, 2s+1), and O's dims are permuted so that lane g's V slice
// (8 consecutive dims for d = 64) forms its A fragments by byte permutes of two edges' words.
// Per 16 edges a lane issues 2 x (d/64 ... ) 16-byte K loads and 4 x (d/64) V loads; with
// one block prefetched every warp keeps 16 edges (4 KB at d = 64 bf16) in flight.
//
// Replaces the edge kernel's 8-lane FHFMA groups (~23 warp-instructions per edge, issue
// bound at cfg3, profiles/r01_cfg3_edge_ncu.txt) with ~5.
#include <cstdlib>

#include "csr_mma.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace ga {
namespace csrmma {

static bool getenv_flag(const char *name)
{
    const char *v = getenv(name);
    return v != nullptr && v[0] != 0 && v[0] != '0';
}

constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;

// Carried state (ga_opts.state) for one (row, head) at the end of a CSR row:
// (m, l) of this call's edges (warp-uniform, log2 domain) and NV of this lane's unnormalised
// o~ values at dims dim[k] (lanes may share dims: they hold equal values).  WRITE overwrites,
// ACCUMULATE (+)-combines with the buffers; with p.out also the normalised row (bf16/fp16).
// Returns the 1/l the caller's output uses.
template <typename T, int NV>
__device__ __forceinline__ float state_merge(const AttnParams &p, int64_t tq, int h, float m, float l, const int *dim,
                                             float *val, bool writer)
{
    const size_t rh = (size_t)tq * p.H + h;
    float *so = p.state.o + rh * p.d;
    if (p.state_mode == GA_STATE_ACCUMULATE) {
        const float l2 = p.state.l[rh];
        if (l2 > 0.f) { // l == 0 marks an empty state (its m is ignored)
            const float m2 = p.state.m[rh];
            const float mn = l > 0.f ? fmaxf(m, m2) : m2;
            const float a = l > 0.f ? ex2(m - mn) : 0.f, b = ex2(m2 - mn);
#pragma unroll
            for (int k = 0; k < NV; ++k) val[k] = val[k] * a + so[dim[k]] * b;
            l = l * a + l2 * b;
            m = mn;
        }
    }
    __syncwarp(); // every lane has read the old state before any lane overwrites it
    if (writer) {
#pragma unroll
        for (int k = 0; k < NV; ++k) so[dim[k]] = val[k];
    }
    if ((threadIdx.x & 31) == 0) {
        p.state.m[rh] = m;
        p.state.l[rh] = l;
    }
    return l > 0.f ? 1.f / l : 0.f;
}

template <typename T, int D>
__global__ void __launch_bounds__(THREADS, (D <= 64 ? 2 : 1)) csr_mma_kernel(const __grid_constant__ AttnParams p)
{
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int64_t gw = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
    const int H = p.H;
    if (gw >= p.q_rows * H) return;
    const int64_t tq = div_heads(gw, H);
    const int h = (int)(gw - tq * H);
    const int64_t i = p.q_begin + tq;
    const int64_t rb = p.mask.row_ptr[i], cnt = p.mask.row_ptr[i + 1] - rb;
    if (p.heavy_threshold > 0 && cnt > p.heavy_threshold) return; // split path (csr_heavy.cu)
    const size_t row_bytes = (size_t)H * D * sizeof(T);
    const size_t hoff = (size_t)h * D * sizeof(T);

    RowAcc<T, D> acc;
    acc.init(p, tq, h, lane);
    acc.run(p, p.mask.col_idx + rb, cnt, h, lane);
    float r[2 * RowAcc<T, D>::KS];
    const float l = acc.finish(r);
    float inv = l > 0.f ? 1.f / l : 0.f; // empty row -> 0 (reading R6)
    if (p.state.m) { // lane (g, t = 0) holds dims g D/8 .. + D/8
        int dims[2 * RowAcc<T, D>::KS];
#pragma unroll
        for (int k = 0; k < 2 * RowAcc<T, D>::KS; ++k) dims[k] = g * (D / 8) + k;
        inv = state_merge<T, 2 * RowAcc<T, D>::KS>(p, tq, h, cnt > 0 ? acc.m : -INFINITY, l, dims, r, t == 0);
        if (!p.out) return;
    }
    if (t != 0) return;
    uint32_t out[RowAcc<T, D>::KS];
#pragma unroll
    for (int x = 0; x < RowAcc<T, D>::KS; ++x) out[x] = pack2<T>(r[2 * x] * inv, r[2 * x + 1] * inv);
    char *op = reinterpret_cast<char *>(p.out) + (size_t)tq * row_bytes + hoff + g * (D / 8 * sizeof(T));
    if constexpr (RowAcc<T, D>::KS == 2) {
        asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(op), "r"(out[0]), "r"(out[1]) : "memory");
    } else {
#pragma unroll
        for (int c = 0; c < RowAcc<T, D>::KS / 4; ++c)
            stg16(op + 16 * c, make_uint4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]));
    }
}

// ---------------------------------------------------------------- TMA gather4 variant (d = 64)
// Same per-block math; the K/V rows of each 16-edge block arrive by 8 tile::gather4 loads (4
// rows each, issued by lanes 0-7 of the warp) into a per-warp ring of TS stages
// (16 K + 16 V rows x 128 B, 128B-swizzled), completing on the stage's mbarrier.  In-flight
// data costs no registers, so each warp keeps TS blocks (12 KB) in flight — what the random
// columns of a CSR need to cover DRAM latency — and the per-edge address arithmetic of the
// LDG variant disappears (TMA takes token coordinates).
#ifndef GA_CSR_TW
#define GA_CSR_TW 8
#endif
#ifndef GA_CSR_TS
#define GA_CSR_TS 3 // measured cfg3: TS 2 -> 8.77, 3 -> 8.79 ms; TS 4 with 6 warps -> 10.5 ms
#endif
constexpr int TW = GA_CSR_TW; // warps per CTA
constexpr int TS = GA_CSR_TS; // stages per warp
constexpr int STAGE = 4096; // bytes per stage
constexpr int IR = 8;       // column-index ring slots per warp (32 edges each)
#ifndef GA_CSR_PD
#define GA_CSR_PD 7 // cfg3, same box: 3 -> 8.777, 5 -> 8.708, 7 -> 8.686 ms (7 = IR - 1, the most the ring allows)
#endif
constexpr int PD = GA_CSR_PD; // index pairs staged ahead
static_assert(PD < IR, "a slot is refilled only after its pair was issued");

struct TmaParams {
    AttnParams p;
    CUtensorMap tmK, tmV;   // gather4: one-row boxes
    CUtensorMap tbK, tbV;   // 16 consecutive rows (a contiguous block of columns)
};

__device__ __forceinline__ uint4 lds128(uint32_t a)
{
    uint4 u;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(a));
    return u;
}

// 16-byte chunk c of stage row r (128B swizzle: chunk ^ row within each 1024-byte atom)
__device__ __forceinline__ uint32_t srow(uint32_t st, int r, int c) { return st + r * 128 + ((c ^ (r & 7)) << 4); }

// Per-(row, head) state of the staged variants (d = 64).  Operands come from the stage by
// ldmatrix in the natural dim order: K rows as the A operand of S^T = K q^T (x4), V rows
// transposed as the A operand of O^T = V^T P^T (x4.trans) — no register permutes.
template <typename T> struct SAcc {
    uint32_t q[8];   // B of k-step s: q[2s] = dims 16s + 2t, +1; q[2s+1] = dims 16s + 8 + 2t, +1
    float o[4][4];   // O^T m-tile x: rows dims 16x + g (c0, c1) and 16x + g + 8 (c2, c3)
    float m, l;
    uint32_t sel;
    float sl2;
    uint32_t kofs[4], vofs[4]; // this lane's ldmatrix row addresses inside a stage

    __device__ __forceinline__ void init(const AttnParams &p, int64_t tq, int h, int lane)
    {
        const int g = lane >> 2, t = lane & 3, mi = lane >> 3, r = lane & 7;
        const uint32_t *qw = reinterpret_cast<const uint32_t *>(
            reinterpret_cast<const char *>(p.Q) + ((size_t)tq * p.H + h) * 64 * sizeof(T));
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            q[2 * s] = __ldg(qw + 8 * s + t);
            q[2 * s + 1] = __ldg(qw + 8 * s + 4 + t);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x) o[x][0] = o[x][1] = o[x][2] = o[x][3] = 0.f;
        m = -INFINITY;
        l = 0.f;
        sl2 = p.scale_log2;
        sel = g == 2 * t ? 0x0000ffffu : (g == 2 * t + 1 ? 0xffff0000u : 0u);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            // K (A of S^T): matrix mi = rows (edges) 8 (mi & 1) + r, 8 dims 16 s + 8 (mi >> 1)
            const int krow = r + 8 * (mi & 1), kch = 2 * s + (mi >> 1);
            kofs[s] = krow * 128 + ((kch ^ r) << 4);
            // V^T (A of O^T, transposed load): matrix mi = V rows (edges) 8 (mi >> 1) + r,
            // 8 dims 16 x + 8 (mi & 1)
            const int vrow = 16 + r + 8 * (mi >> 1), vch = 2 * s + (mi & 1);
            vofs[s] = vrow * 128 + ((vch ^ r) << 4);
        }
    }

    // one 16-edge block from stage fragments ka (K) and va (V^T)
    __device__ __forceinline__ void compute(const uint32_t (*ka)[4], const uint32_t (*va)[4], bool ok0, bool ok8)
    {
        float c[4] = {0.f, 0.f, 0.f, 0.f}, e[4] = {0.f, 0.f, 0.f, 0.f}; // two MMA chains
        tc::mma16816<T>(c, ka[0], q[0], q[1]);
        tc::mma16816<T>(e, ka[1], q[2], q[3]);
        tc::mma16816<T>(c, ka[2], q[4], q[5]);
        tc::mma16816<T>(e, ka[3], q[6], q[7]);
        const float s0 = ok0 ? (c[0] + e[0]) * sl2 : -INFINITY;
        const float s8 = ok8 ? (c[2] + e[2]) * sl2 : -INFINITY;
        // lazy rescale: only when some score exceeds the reference max by > 2^8 (one vote in
        // the common case; the block max by shuffles only then)
        if (__any_sync(0xffffffffu, fmaxf(s0, s8) > m + 8.f)) {
            float bm = fmaxf(s0, s8);
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 4));
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
            const float a = ex2(m - bm);
            l *= a;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                o[x][0] *= a;
                o[x][1] *= a;
                o[x][2] *= a;
                o[x][3] *= a;
            }
            m = bm;
        }
        const float p0 = ex2(s0 - m), p8 = ex2(s8 - m);
        l += p0 + p8;
        const uint32_t b0 = pack2<T>(p0, p0) & sel, b1 = pack2<T>(p8, p8) & sel;
#pragma unroll
        for (int x = 0; x < 4; ++x) tc::mma16816<T>(o[x], va[x], b0, b1);
    }

    // l total and the column sums: every lane ends with u[x] = o~ of dim 16x + g, w[x] of 16x + g + 8
    __device__ __forceinline__ float finish(float *u, float *w) const
    {
        float lt = l;
        lt += __shfl_xor_sync(0xffffffffu, lt, 4);
        lt += __shfl_xor_sync(0xffffffffu, lt, 8);
        lt += __shfl_xor_sync(0xffffffffu, lt, 16);
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            float a = o[x][0] + o[x][1], b = o[x][2] + o[x][3];
            a += __shfl_xor_sync(0xffffffffu, a, 1);
            b += __shfl_xor_sync(0xffffffffu, b, 1);
            a += __shfl_xor_sync(0xffffffffu, a, 2);
            b += __shfl_xor_sync(0xffffffffu, b, 2);
            u[x] = a;
            w[x] = b;
        }
        return lt;
    }
};

template <typename T, bool CPA>
__global__ void __launch_bounds__(TW * 32, 2) csr_tma_kernel(const __grid_constant__ TmaParams tp)
{
    constexpr int D = 64;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const AttnParams &p = tp.p;
    const uint32_t sw = sbase + warp * TS * STAGE;
    const uint32_t mb = sbase + TW * TS * STAGE + warp * TS * 8;

    const int H = p.H;
    const int64_t ntask = p.q_rows * H, nwarps = (int64_t)gridDim.x * TW;
    if (lane < TS) umma::mbar_init(mb + 8 * lane, CPA ? 32 : 1);
    umma::fence_proxy_async(); // barrier init visible to the async proxy
    __syncwarp();
    uint32_t doff[4]; // shared offsets of this lane's copy chunks (128B-swizzled rows 4 (lane>>3) + q)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int e = 4 * (lane >> 3) + q, c = lane & 7;
        doff[q] = e * 128 + ((c ^ (e & 7)) << 4);
    }
    uint32_t ph = 0; // completed uses per stage, carried across rows (bit s of the parity word)
    // persistent warps: (row, head) tasks gw, gw + nwarps, ...; the next task's column
    // indices are prefetched into L2 while this one runs (its first index loads would
    // otherwise wait on DRAM once per row)
    for (int64_t gw = (int64_t)blockIdx.x * TW + warp; gw < ntask; gw += nwarps) {
    const int64_t tq = div_heads(gw, H);
    const int h = (int)(gw - tq * H);
    const int64_t i = p.q_begin + tq;
    const int64_t rb = p.mask.row_ptr[i], cnt = p.mask.row_ptr[i + 1] - rb;
    if (gw + nwarps < ntask) {
        const int64_t i2 = p.q_begin + div_heads(gw + nwarps, H);
        const int64_t r2 = p.mask.row_ptr[i2], n2 = p.mask.row_ptr[i2 + 1] - r2;
        const char *c2 = reinterpret_cast<const char *>(p.mask.col_idx + r2);
        if (n2 <= p.heavy_threshold || p.heavy_threshold <= 0)
            for (int64_t off = (int64_t)lane * 128; off < n2 * 4 && off < 8192; off += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(c2 + off));
    }
    if (p.heavy_threshold > 0 && cnt > p.heavy_threshold) continue; // split path (csr_heavy.cu)
    const int32_t *cols = p.mask.col_idx + rb;

    SAcc<T> acc;
    acc.init(p, tq, h, lane);
    const int ncnt = (int)cnt; // a light row has < 2^31 edges (int32 columns)
    const int nblk = (ncnt + 15) / 16, npair = (ncnt + 31) / 32;
    const int kv0 = (int)p.kv_begin;
    // column indices: pair P (32 edges, lane l holds edge 32P + l) is loaded into registers
    // PD + 2 pairs ahead, stored to the per-warp ring slot P % IR when pair P - PD retires,
    // and read from there by the issue of P's blocks (past the row's end: kv_begin -> row 0)
    const uint32_t sidx = sbase + TW * TS * STAGE + TW * TS * 8 + warp * IR * 128;
    // Indices are stored relative to kv_begin, with one flag word per pair: bit k set iff block k
    // of the pair is 16 consecutive columns (a window run: one 16-row TMA box) — every column
    // checked, computed by the whole warp once per pair (a shuffle and a ballot) instead of by
    // the issuing lane once per block.
    const uint32_t sflag = sbase + TW * TS * STAGE + TW * TS * 8 + TW * IR * 128 + warp * IR * 4;
    auto ld_pair = [&](int P) -> int {
        const int e = P * 32 + lane;
        return (P < npair && e < ncnt) ? cols[e] - kv0 : 0;
    };
    auto st_pair = [&](int P, int v) {
        const int nx = __shfl_down_sync(0xffffffffu, v, 1);
        const unsigned bal = __ballot_sync(0xffffffffu, (lane & 15) == 15 || nx == v + 1);
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sidx + (P % IR) * 128 + lane * 4), "r"(v) : "memory");
        if (lane == 0) {
            const uint32_t f = ((bal & 0xffffu) == 0xffffu ? 1u : 0u) | ((bal >> 16) == 0xffffu ? 2u : 0u);
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(sflag + (P % IR) * 4), "r"(f) : "memory");
        }
    };
    // pairs PD .. PD + RQ - 1 in flight in registers (global loads of the column indices)
#ifndef GA_CSR_RQ
#define GA_CSR_RQ 6 // measured cfg3: 2 -> 8.86, 3 -> 8.83, 4 -> 8.78 ms; later, same box: 4 -> 8.727, 6 -> 8.709, 8 -> 8.832
#endif
    constexpr int RQ = GA_CSR_RQ;
    static_assert(RQ >= 2 && RQ <= 8, "index register queue");
    int rq[RQ];
    for (int P = 0; P < PD; ++P) st_pair(P, ld_pair(P));
#pragma unroll
    for (int u = 0; u < RQ; ++u) rq[u] = ld_pair(PD + u);
    __syncwarp();
    const uint32_t row_bytes = (uint32_t)(H * D * sizeof(T));
    // lane (r8, c) copies 16-byte chunk c of the K and V rows of edges 4 r8 + q: its global
    // base folds in the head, the chunk and -kv_begin rows; its shared offsets are fixed
    const char *kbase = reinterpret_cast<const char *>(p.K) + (size_t)h * D * sizeof(T) + (lane & 7) * 16;
    const ptrdiff_t vdelta = reinterpret_cast<const char *>(p.V) - reinterpret_cast<const char *>(p.K);
    // block n -> stage s = n % TS (passed in by the caller's stage counter)
    auto issue = [&](int n, int s) {
        const uint32_t bar = mb + 8 * s, dst = sw + s * STAGE;
        const uint32_t src = sidx + ((n >> 1) % IR) * 128 + (n & 1) * 64;
        if constexpr (CPA) { // 16-byte cp.async, 8 lanes per 128-byte row, 4 rows per instruction
            const int r8 = lane >> 3;
            const uint4 jv = lds128(src + 16 * r8); // edges 4 r8 .. 4 r8 + 3
            const uint32_t js[4] = {jv.x, jv.y, jv.z, jv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) { // instruction q: rows (edges) q, 4 + q, 8 + q, 12 + q
                const char *ka = kbase + (uint64_t)js[q] * row_bytes;
                const uint32_t d = dst + doff[q];
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(ka) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d + 2048), "l"(ka + vdelta) : "memory");
            }
            umma::cp_async_mbar_arrive(bar);
        } else if (lane == 0) {
            tma::expect_tx(bar, STAGE);
            // a block of 16 consecutive columns (e.g. the window run of a BigBird row) is one
            // 16-row box for K and one for V; otherwise 4 + 4 tile::gather4 loads.  Every
            // column is checked (duplicate columns of a multiset CSR can span 15 too).
            uint32_t f;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(f) : "r"(sflag + ((n >> 1) % IR) * 4));
            if ((f >> (n & 1)) & 1u) {
                int jb;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(jb) : "r"(src));
                tma::load_3d(dst, &tp.tbK, 0, h, jb, bar);
                tma::load_3d(dst + 2048, &tp.tbV, 0, h, jb, bar);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 j = lds128(src + 16 * q);
                    tma::gather4(dst + q * 512, &tp.tmK, h * D, (int)j.x, (int)j.y, (int)j.z, (int)j.w, bar);
                    tma::gather4(dst + 2048 + q * 512, &tp.tmV, h * D, (int)j.x, (int)j.y, (int)j.z, (int)j.w, bar);
                }
            }
        }
        if (n & 1) { // pair n/2 retires: every lane's reads of its slot are done before the refill
            __syncwarp();
            st_pair((n >> 1) + PD, rq[0]);
#pragma unroll
            for (int u = 0; u + 1 < RQ; ++u) rq[u] = rq[u + 1];
            rq[RQ - 1] = ld_pair((n >> 1) + PD + RQ);
            __syncwarp();
        }
    };
    for (int n = 0; n < nblk && n < TS; ++n) issue(n, n);
    int s = 0;
    for (int b = 0; b < nblk; ++b, s = s + 1 == TS ? 0 : s + 1) {
        umma::mbar_wait(mb + 8 * s, (ph >> s) & 1u);
        ph ^= 1u << s;
        const uint32_t st = sw + s * STAGE;
        uint32_t ka[4][4], va[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            tc::ldsm_x4(st + acc.kofs[x], ka[x][0], ka[x][1], ka[x][2], ka[x][3]);
            tc::ldsm_x4_t(st + acc.vofs[x], va[x][0], va[x][1], va[x][2], va[x][3]);
        }
        if (b + TS < nblk) { // stage s is read: refill it with block b + TS
            __syncwarp();
            if (!CPA) umma::fence_proxy_async();
            issue(b + TS, s);
        }
        acc.compute(ka, va, b * 16 + g < ncnt, b * 16 + g + 8 < ncnt);
    }

    float u[4], w[4];
    const float l = acc.finish(u, w);
    float inv = l > 0.f ? 1.f / l : 0.f; // empty row -> 0 (reading R6)
    // lane (g, t) stores dims 16t + g and 16t + g + 8 (all four t-lanes hold every column sum)
    float uo = u[0], wo = w[0];
#pragma unroll
    for (int x = 1; x < 4; ++x)
        if (t == x) { uo = u[x]; wo = w[x]; }
    bool store = true;
    if (p.state.m) {
        const int dims[2] = {16 * t + g, 16 * t + g + 8};
        float vals[2] = {uo, wo};
        inv = state_merge<T, 2>(p, tq, h, ncnt > 0 ? acc.m : -INFINITY, l, dims, vals, true);
        uo = vals[0];
        wo = vals[1];
        store = p.out != nullptr;
    }
    if (store) {
        T *op = reinterpret_cast<T *>(p.out) + ((size_t)tq * H + h) * D;
        op[16 * t + g] = (T)(uo * inv);
        op[16 * t + g + 8] = (T)(wo * inv);
    }
    __syncwarp(); // the index ring and stages are reused by the next task
    }
}

template <typename T, bool CPA> static ga_status launch_tma_m(const TmaParams &tp, int64_t warps, cudaStream_t s)
{
    const int smem = TW * TS * STAGE + TW * TS * 8 + TW * IR * 128 + TW * IR * 4 + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(csr_tma_kernel<T, CPA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t blocks = (warps + TW - 1) / TW, resident = (int64_t)nsm * 2; // 2 CTAs per SM
    csr_tma_kernel<T, CPA><<<(unsigned)(blocks < resident ? blocks : resident), TW * 32, smem, s>>>(tp);
    GA_CHECK_LAUNCH("csr_tma_kernel");
    return GA_OK;
}

// staged variants (d = 64, local K/V): TMA gather4 (default; cfg3 10.7 ms) or the 16-byte
// cp.async ring (GA_CSR_CPASYNC=1; 11.1 ms)
template <typename T> static ga_status launch_tma(const AttnParams &p, cudaStream_t s, bool &done)
{
    done = false;
    if (p.k_peer != nullptr || p.kv_rows >= INT32_MAX) return GA_OK; // LDG variant
    TmaParams tp;
    tp.p = p;
    const bool g4 = !getenv_flag("GA_CSR_CPASYNC");
    if (g4 && (!tma::encode_gather(&tp.tmK, p.K, p.kv_rows, p.H, 64) ||
               !tma::encode_gather(&tp.tmV, p.V, p.kv_rows, p.H, 64) ||
               !tma::encode_block(&tp.tbK, p.K, p.kv_rows, p.H, 64, 16) ||
               !tma::encode_block(&tp.tbV, p.V, p.kv_rows, p.H, 64, 16)))
        return GA_OK;
    const int64_t warps = p.q_rows * p.H;
    done = true;
    if (warps == 0) return GA_OK;
    return g4 ? launch_tma_m<T, false>(tp, warps, s) : launch_tma_m<T, true>(tp, warps, s);
}

template <typename T, int D> static ga_status launch_t(const AttnParams &p, cudaStream_t s)
{
    const int64_t warps = p.q_rows * p.H;
    if (warps == 0) return GA_OK;
    const int64_t blocks = (warps + WARPS - 1) / WARPS;
    csr_mma_kernel<T, D><<<(unsigned)blocks, THREADS, 0, s>>>(p);
    GA_CHECK_LAUNCH("csr_mma_kernel");
    return GA_OK;
}

template <typename T> static ga_status launch_d(const AttnParams &p, cudaStream_t s)
{
    if (p.d == 64 && !getenv_flag("GA_CSR_LDG")) {
        bool done;
        const ga_status st = launch_tma<T>(p, s, done);
        if (st != GA_OK || done) return st;
    }
    switch (p.d) {
    case 32: return launch_t<T, 32>(p, s);
    case 64: return launch_t<T, 64>(p, s);
    case 128: return launch_t<T, 128>(p, s);
    }
    set_error("csr_mma: d=%d unsupported", p.d);
    return GA_ERR_UNSUPPORTED;
}

} // namespace csrmma

bool csr_mma_supported(const AttnParams &p, ga_dtype dt)
{
    return p.mask.kind == K_CSR && (dt == GA_BF16 || dt == GA_F16) && (p.d == 32 || p.d == 64 || p.d == 128) &&
           p.kv_begin + p.kv_rows <= INT32_MAX;
}

ga_status launch_csr_mma(const AttnParams &p, ga_dtype dt, cudaStream_t s)
{
    if (dt == GA_BF16) return csrmma::launch_d<__nv_bfloat16>(p, s);
    if (dt == GA_F16) return csrmma::launch_d<__half>(p, s);
    set_error("csr_mma: bf16/fp16 only");
    return GA_ERR_UNSUPPORTED;
}

} // namespace ga

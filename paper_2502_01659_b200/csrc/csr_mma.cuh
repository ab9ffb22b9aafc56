// csr_mma.cuh — explicit-CSR edge blocks on mma.sync (see csr_mma.cu for the mapping):
// one warp runs one (row, head) or one chunk of a heavy row (csr_heavy.cu).
#pragma once
#include "common.cuh"
#include "tc_common.cuh"

namespace ga {
namespace csrmma {

template <int NW> __device__ __forceinline__ void ldg_words(const char *p, uint32_t *w)
{
    static_assert(NW % 4 == 0 || NW == 2, "16- or 8-byte slices");
    if constexpr (NW == 2) {
        uint2 r;
        asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
        w[0] = r.x;
        w[1] = r.y;
    } else {
#pragma unroll
        for (int c = 0; c < NW / 4; ++c) {
            const uint4 r = ldg16(p + 16 * c);
            w[4 * c + 0] = r.x;
            w[4 * c + 1] = r.y;
            w[4 * c + 2] = r.z;
            w[4 * c + 3] = r.w;
        }
    }
}

// One 16-edge block's operands for one lane.
template <int D> struct Blk {
    static constexpr int KW = D / 8;  // words of a K row slice (lane t: elements [t D/4, (t+1) D/4))
    static constexpr int VW = D / 16; // words of a V row slice (lane g: dims [g D/8, (g+1) D/8))
    uint32_t k0[KW], k8[KW];          // K rows of edges g and g+8
    uint32_t v[4][VW];                // V rows of edges 2t, 2t+1, 2t+8, 2t+9
    bool ok0, ok8;                    // edges g, g+8 exist
};

template <typename T, int D>
__device__ __forceinline__ void load_blk(const AttnParams &p, Blk<D> &b, int idx_lane_val, int half, int64_t e0,
                                         int64_t cnt, int g, int t, size_t row_bytes, size_t hoff)
{
    // idx_lane_val: lane l holds the column of edge (block pair base + l); this block is
    // edges [16 half, 16 half + 16) of the pair
    const int base = 16 * half;
    const int j0 = __shfl_sync(0xffffffffu, idx_lane_val, base + g);
    const int j8 = __shfl_sync(0xffffffffu, idx_lane_val, base + g + 8);
    const int ja = __shfl_sync(0xffffffffu, idx_lane_val, base + 2 * t);
    const int jb = __shfl_sync(0xffffffffu, idx_lane_val, base + 2 * t + 1);
    const int jc = __shfl_sync(0xffffffffu, idx_lane_val, base + 2 * t + 8);
    const int jd = __shfl_sync(0xffffffffu, idx_lane_val, base + 2 * t + 9);
    b.ok0 = e0 + g < cnt;
    b.ok8 = e0 + g + 8 < cnt;
    constexpr int KB = D / 4 * (int)sizeof(T); // bytes of a lane's K slice
    constexpr int VB = D / 8 * (int)sizeof(T); // bytes of a lane's V slice
    const char *kr, *vr;
    kv_row(p, j0, row_bytes, kr, vr);
    ldg_words<Blk<D>::KW>(kr + hoff + t * KB, b.k0);
    kv_row(p, j8, row_bytes, kr, vr);
    ldg_words<Blk<D>::KW>(kr + hoff + t * KB, b.k8);
    kv_row(p, ja, row_bytes, kr, vr);
    ldg_words<Blk<D>::VW>(vr + hoff + g * VB, b.v[0]);
    kv_row(p, jb, row_bytes, kr, vr);
    ldg_words<Blk<D>::VW>(vr + hoff + g * VB, b.v[1]);
    kv_row(p, jc, row_bytes, kr, vr);
    ldg_words<Blk<D>::VW>(vr + hoff + g * VB, b.v[2]);
    kv_row(p, jd, row_bytes, kr, vr);
    ldg_words<Blk<D>::VW>(vr + hoff + g * VB, b.v[3]);
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

template <typename T, int D> struct RowAcc {
    static constexpr int KS = D / 16; // k-steps of q.k and m-tiles of O^T
    uint32_t q[D / 8];                // q slice (lane t), replicated over g
    float o[KS][4];                   // O^T accumulator fragments
    float m, l;                       // running max (exp2 domain), partial sum of this lane's edges
    uint32_t sel;                     // which half of P^T's packed pair this lane owns (or 0)
    float sl2;

    __device__ __forceinline__ void compute(const Blk<D> &b)
    {
        // S^T = K_blk q^T: c[0] = score of edge g, c[2] = score of edge g+8 (all columns equal)
        float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const uint32_t a[4] = {b.k0[2 * s], b.k8[2 * s], b.k0[2 * s + 1], b.k8[2 * s + 1]};
            tc::mma16816<T>(c, a, q[2 * s], q[2 * s + 1]);
        }
        const float s0 = b.ok0 ? c[0] * sl2 : -INFINITY;
        const float s8 = b.ok8 ? c[2] * sl2 : -INFINITY;
        float bm = fmaxf(s0, s8);
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 4));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
        if (bm > m + 8.f) { // warp-uniform lazy rescale (weights stay <= 2^8 otherwise)
            const float a = ex2(m - bm);
            l *= a;
#pragma unroll
            for (int x = 0; x < KS; ++x) {
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
        // O^T += V_blk^T P^T; A of m-tile x: rows (dim g D/8 + 2x, +1), columns (edges 2t, 2t+1 | 2t+8, 2t+9)
#pragma unroll
        for (int x = 0; x < KS; ++x) {
            const uint32_t a[4] = {prmt(b.v[0][x], b.v[1][x], 0x5410), prmt(b.v[0][x], b.v[1][x], 0x7632),
                                   prmt(b.v[2][x], b.v[3][x], 0x5410), prmt(b.v[2][x], b.v[3][x], 0x7632)};
            tc::mma16816<T>(o[x], a, b0, b1);
        }
    }
    // this lane's q slice and an empty state
    __device__ __forceinline__ void init(const AttnParams &p, int64_t tq, int h, int lane)
    {
        const int g = lane >> 2, t = lane & 3;
        const size_t row_bytes = (size_t)p.H * D * sizeof(T);
        ldg_words<D / 8>(reinterpret_cast<const char *>(p.Q) + (size_t)tq * row_bytes + (size_t)h * D * sizeof(T) +
                             t * (D / 4 * sizeof(T)),
                         q);
#pragma unroll
        for (int x = 0; x < KS; ++x) o[x][0] = o[x][1] = o[x][2] = o[x][3] = 0.f;
        m = -INFINITY;
        l = 0.f;
        sl2 = p.scale_log2;
        sel = g == 2 * t ? 0x0000ffffu : (g == 2 * t + 1 ? 0xffff0000u : 0u);
    }

    // edges cols[0 .. cnt): 16 per block, the next block's K/V (and the next 32 column
    // indices) loaded before the current block is consumed
    __device__ __forceinline__ void run(const AttnParams &p, const int32_t *cols, int64_t cnt, int h, int lane)
    {
        if (cnt <= 0) return;
        const int g = lane >> 2, t = lane & 3;
        const size_t row_bytes = (size_t)p.H * D * sizeof(T);
        const size_t hoff = (size_t)h * D * sizeof(T);
        const int jpad = (int)p.kv_begin; // any readable row for the lanes past the row's end
        Blk<D> A, B;
        int idx = lane < cnt ? cols[lane] : jpad;
        load_blk<T, D>(p, A, idx, 0, 0, cnt, g, t, row_bytes, hoff);
        for (int64_t e = 0;; e += 32) { // A holds edges [e, e+16)
            const bool hasB = e + 16 < cnt, hasN = e + 32 < cnt;
            if (hasB) load_blk<T, D>(p, B, idx, 1, e + 16, cnt, g, t, row_bytes, hoff);
            int nidx = jpad;
            if (hasN && e + 32 + lane < cnt) nidx = cols[e + 32 + lane];
            compute(A);
            if (!hasB) break;
            if (hasN) load_blk<T, D>(p, A, nidx, 0, e + 32, cnt, g, t, row_bytes, hoff);
            compute(B);
            if (!hasN) break;
            idx = nidx;
        }
    }

    // column sums of O^T (lanes t of one g) and the row sum l (lanes g of one t): every
    // lane ends with l_tot and r[2x], r[2x+1] = unnormalised o of dims g D/8 + 2x, +1
    __device__ __forceinline__ float finish(float *r) const
    {
        float lt = l;
        lt += __shfl_xor_sync(0xffffffffu, lt, 4);
        lt += __shfl_xor_sync(0xffffffffu, lt, 8);
        lt += __shfl_xor_sync(0xffffffffu, lt, 16);
#pragma unroll
        for (int x = 0; x < KS; ++x) {
            float u = o[x][0] + o[x][1], w = o[x][2] + o[x][3];
            u += __shfl_xor_sync(0xffffffffu, u, 1);
            w += __shfl_xor_sync(0xffffffffu, w, 1);
            u += __shfl_xor_sync(0xffffffffu, u, 2);
            w += __shfl_xor_sync(0xffffffffu, w, 2);
            r[2 * x] = u;
            r[2 * x + 1] = w;
        }
        return lt;
    }
};


} // namespace csrmma
} // namespace ga

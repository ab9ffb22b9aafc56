// tc_common.cuh — shared-memory staging and mma.sync helpers for the tensor-core kernels
// (band kernel for windows, dense-group kernel for LongNet).
#pragma once
#include "edge_core.cuh"

namespace ga {
namespace tc {

template <int D> struct Geo {
    static constexpr int RB = 2 * D;    // bytes per (token, head) row (bf16/fp16)
    static constexpr int NC = RB / 16;  // 16-byte chunks per row
    static constexpr int HC = NC / 2;   // chunks per half row (CUDA-core lanes)
    static constexpr int KS = D / 16;   // k16 steps over d for Q K^T
    static constexpr int NB8 = D / 8;   // n8 blocks over d for P V
};

// byte offset of chunk `ch` of row `row` in a swizzled [rows][RB] tile: the 16-byte chunk
// index is XORed with the row's low bits so 8 consecutive rows hit 8 different bank groups
template <int D> __device__ __forceinline__ uint32_t swz(int row, int ch)
{
    constexpr int NC = Geo<D>::NC;
    const int f = NC >= 8 ? (row & 7) : ((row >> 1) & 3);
    return (uint32_t)(row * Geo<D>::RB + ((ch ^ f) * 16));
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *g)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N> __device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void sts_zero16(uint32_t a)
{
    asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(0u));
}

__device__ __forceinline__ uint4 lds16(uint32_t a)
{
    uint4 u;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(a));
    return u;
}

__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3)
{
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3)
{
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(a));
}

template <typename T>
__device__ __forceinline__ void mma16816(float *c, const uint32_t *a, uint32_t b0, uint32_t b1);

template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float *c, const uint32_t *a, uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <>
__device__ __forceinline__ void mma16816<__half>(float *c, const uint32_t *a, uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// (x0, x1) * s - m for a pair of fp32 values in one FFMA2 (sm_100 packed fp32 FMA)
__device__ __forceinline__ void ffma2_sm(float &x0, float &x1, float s, float negm)
{
    unsigned long long a, b, c, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(x0), "f"(x1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(s));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(negm));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(d));
}

// (2^x0, 2^x1) on the FMA pipe instead of MUFU (offloads the exp unit, as FA4 does):
// n = round(x) via the 1.5 * 2^23 magic add, f = x - n in [-0.5, 0.5], 2^f by a degree-3
// minimax polynomial (max relative error 7.6e-5: below the bf16/fp16 rounding of P), then
// n added to the exponent field with one IMAD.  x is clamped to >= -126 (2^-126 ~ 1e-38
// stands in for 0, e.g. for a masked -inf score).
__device__ __forceinline__ void ex2_poly2(float &x0, float &x1)
{
    x0 = fmaxf(x0, -126.f);
    x1 = fmaxf(x1, -126.f);
    unsigned long long x, t, r, f, pp, c;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(12582912.f));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(x), "l"(c));  // t = x + 1.5*2^23 (round)
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(t), "l"(c));  // r = round(x)
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(x), "l"(r));  // f in [-0.5, 0.5]
    unsigned long long c3, c2, c1, c0;
    asm("mov.b64 %0, {%1, %1};" : "=l"(c3) : "f"(0.055194102227687836f));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c2) : "f"(0.24260859191417694f));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c1) : "f"(0.6932564377784729f));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c0) : "f"(0.9999281167984009f));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(c3), "l"(f), "l"(c2));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(f), "l"(c1));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(f), "l"(c0));
    uint32_t p0, p1, t0, t1;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(p0), "=r"(p1) : "l"(pp));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(t0), "=r"(t1) : "l"(t));
    // the low bits of t hold n (two's complement); t << 23 keeps exactly n << 23
    x0 = __uint_as_float(p0 + (t0 << 23));
    x1 = __uint_as_float(p1 + (t1 << 23));
}

// acc += (x0, x1) in one packed fp32 add (sm_100 add.f32x2)
__device__ __forceinline__ void fadd2_acc(float2 &acc, float x0, float x1)
{
    unsigned long long a, b, d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(acc.x), "f"(acc.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(x0), "f"(x1));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(d));
}

// Running flash-attention state of one warp's 16 rows in the m16n8 accumulator layout:
// lane (g = lane/4, t4 = lane%4) owns rows g and g+8 and dims 8j + 2*t4 + {0,1}.
template <typename T, int D> struct MmaRows {
    using G = Geo<D>;
    uint32_t qa[G::KS][4]; // A fragments of the 16 query rows
    float o[G::NB8][4];
    float mr[2], lr[2];     // reference max (exp2 domain) and per-lane partial sums

    __device__ __forceinline__ void load_q(uint32_t sQ, int row0, int lane)
    {
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) {
            const int row = row0 + (lane & 7) + ((lane >> 3) & 1) * 8;
            const int chk = 2 * kk + (lane >> 4);
            ldsm_x4(sQ + swz<D>(row, chk), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
        }
    }

    __device__ __forceinline__ void init_empty()
    {
        mr[0] = mr[1] = -INFINITY;
        lr[0] = lr[1] = 0.f;
#pragma unroll
        for (int j = 0; j < G::NB8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    }

    // multiply the state of rows g / g+8 by a0 / a1 (online-softmax rescale)
    __device__ __forceinline__ void scale_rows(float a0, float a1)
    {
        lr[0] *= a0;
        lr[1] *= a1;
#pragma unroll
        for (int j = 0; j < G::NB8; ++j) {
            o[j][0] *= a0;
            o[j][1] *= a0;
            o[j][2] *= a1;
            o[j][3] *= a1;
        }
    }

    // P (fp32 scores in the accumulator layout, 2 n8 blocks) -> exp2(s * sl2 - m) (one
    // FFMA2 per pair), row partial sums, packed to the input type as the A fragment of P V
    __device__ __forceinline__ void softmax_pack(float (*sv)[4], float sl2, uint32_t *pa)
    {
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
            float x0 = sv[nb][0], x1 = sv[nb][1], x2 = sv[nb][2], x3 = sv[nb][3];
            ffma2_sm(x0, x1, sl2, -mr[0]);
            ffma2_sm(x2, x3, sl2, -mr[1]);
            x0 = ex2(x0);
            x1 = ex2(x1);
            x2 = ex2(x2);
            x3 = ex2(x3);
            lr[0] += x0 + x1;
            lr[1] += x2 + x3;
            pa[2 * nb] = pack2<T>(x0, x1);
            pa[2 * nb + 1] = pack2<T>(x2, x3);
        }
    }

    // One fully dense block of 16 keys whose rows start at kaddr/vaddr (per-lane ldmatrix
    // addresses prepared by the caller: kaddr[kk] for chunk 2kk + ((lane>>3)&1) of key row
    // (lane&7) + (lane>>4)*8, vaddr[jj] for chunk 2jj + (lane>>4) of key row
    // (lane&7) + ((lane>>3)&1)*8).
    __device__ __forceinline__ void block16(const uint32_t *kaddr, const uint32_t *vaddr, uint32_t off, float sl2)
    {
        float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kaddr[kk] + off, b0, b1, b2, b3);
            mma16816<T>(s[0], qa[kk], b0, b1);
            mma16816<T>(s[1], qa[kk], b2, b3);
        }
        // lazy rescale: keep the reference max unless a score exceeds it by more than 2^kTau
        // (exact: l and O share the reference; weights stay <= 2^kTau); the common case
        // needs only per-lane maxima and one warp vote.
        constexpr float kTau = 8.f;
        const float lm0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
        const float lm1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
        const bool need = lm0 * sl2 > mr[0] + kTau || lm1 * sl2 > mr[1] + kTau;
        if (__any_sync(0xffffffffu, need)) {
            float bm0 = fmaxf(lm0, __shfl_xor_sync(0xffffffffu, lm0, 1));
            bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
            float bm1 = fmaxf(lm1, __shfl_xor_sync(0xffffffffu, lm1, 1));
            bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
            const float mn0 = fmaxf(mr[0], bm0 * sl2), mn1 = fmaxf(mr[1], bm1 * sl2);
            scale_rows(ex2(mr[0] - mn0), ex2(mr[1] - mn1));
            mr[0] = mn0;
            mr[1] = mn1;
        }
        uint32_t pa[4];
        softmax_pack(s, sl2, pa);
#pragma unroll
        for (int jj = 0; jj < G::NB8 / 2; ++jj) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vaddr[jj] + off, b0, b1, b2, b3);
            mma16816<T>(o[2 * jj], pa, b0, b1);
            mma16816<T>(o[2 * jj + 1], pa, b2, b3);
        }
    }

    // Two dense 16-key blocks at offsets off0 and off1: both S tiles first (16 independent
    // MMAs), one max/vote for the pair, then both P V updates — half the serialisation
    // points of two block16 calls.
    __device__ __forceinline__ void block16x2(const uint32_t *kaddr, const uint32_t *vaddr, uint32_t off0,
                                              uint32_t off1, float sl2)
    {
        float s[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q][0] = s[q][1] = s[q][2] = s[q][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) {
            uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
            ldsm_x4(kaddr[kk] + off0, b0, b1, b2, b3);
            ldsm_x4(kaddr[kk] + off1, c0, c1, c2, c3);
            mma16816<T>(s[0], qa[kk], b0, b1);
            mma16816<T>(s[1], qa[kk], b2, b3);
            mma16816<T>(s[2], qa[kk], c0, c1);
            mma16816<T>(s[3], qa[kk], c2, c3);
        }
        constexpr float kTau = 8.f;
        float lm0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
        float lm1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
        lm0 = fmaxf(lm0, fmaxf(fmaxf(s[2][0], s[2][1]), fmaxf(s[3][0], s[3][1])));
        lm1 = fmaxf(lm1, fmaxf(fmaxf(s[2][2], s[2][3]), fmaxf(s[3][2], s[3][3])));
        const bool need = lm0 * sl2 > mr[0] + kTau || lm1 * sl2 > mr[1] + kTau;
        if (__any_sync(0xffffffffu, need)) {
            float bm0 = fmaxf(lm0, __shfl_xor_sync(0xffffffffu, lm0, 1));
            bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
            float bm1 = fmaxf(lm1, __shfl_xor_sync(0xffffffffu, lm1, 1));
            bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
            const float mn0 = fmaxf(mr[0], bm0 * sl2), mn1 = fmaxf(mr[1], bm1 * sl2);
            scale_rows(ex2(mr[0] - mn0), ex2(mr[1] - mn1));
            mr[0] = mn0;
            mr[1] = mn1;
        }
        uint32_t pa[2][4];
        softmax_pack(s, sl2, pa[0]);
        softmax_pack(s + 2, sl2, pa[1]);
#pragma unroll
        for (int jj = 0; jj < G::NB8 / 2; ++jj) {
            uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
            ldsm_x4_t(vaddr[jj] + off0, b0, b1, b2, b3);
            ldsm_x4_t(vaddr[jj] + off1, c0, c1, c2, c3);
            mma16816<T>(o[2 * jj], pa[0], b0, b1);
            mma16816<T>(o[2 * jj + 1], pa[0], b2, b3);
            mma16816<T>(o[2 * jj], pa[1], c0, c1);
            mma16816<T>(o[2 * jj + 1], pa[1], c2, c3);
        }
    }

    // sum the per-lane partial l over the quad
    // sum the per-lane partial l over the quad
    __device__ __forceinline__ void reduce_l()
    {
        lr[0] += __shfl_xor_sync(0xffffffffu, lr[0], 1);
        lr[0] += __shfl_xor_sync(0xffffffffu, lr[0], 2);
        lr[1] += __shfl_xor_sync(0xffffffffu, lr[1], 1);
        lr[1] += __shfl_xor_sync(0xffffffffu, lr[1], 2);
    }
};

} // namespace tc
} // namespace ga

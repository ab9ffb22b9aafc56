// backward_tc.cu — backward pass of Window(w, r) masks on the tensor cores (bf16 / fp16,
// d = 64, the training use case of PAPER.md:555).
//
// Same chain rule as backward.cu (reading R25): P = 2^(S log2(e) - lse), dP = dO V^T,
// D = rowsum(dO o O), dS = P o (dP - D), dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d),
// dV = P^T dO — but the residue class of a dilated window is a band (class rows x, y with
// |x - y| <= m, m = floor((w-1)/r); readings R1/R2), so 16 x 16 blocks of the band are dense
// contractions for mma.sync m16n8k16 (the forward band kernel's fragment layouts, tc_common):
//
//   row pass     CTA = 64 class rows of one (class, head), 4 warps x 16 rows; the Q / dO tile
//                and the K / V band they reach ([x0 - m, x0 + 63 + m]) staged in shared
//                memory by cp.async; per warp and 16-key block: S = Q K^T, dP = dO V^T
//                (8 + 8 MMAs), P and dS in registers (masked pairs -> 0), dQ += dS K (8 MMAs).
//                lse (unless given) comes from a first sweep of S blocks; D from dO and O.
//                Writes dQ and the rows' lse, D for the column pass.
//   column pass  CTA = 64 key class rows; the Q / dO band, its lse and D staged; per warp and
//                16-query block: S^T = K Q^T, dP^T = V dO^T, dV += P^T dO, dK += dS^T Q.
//
// Blocks straddling the band's edge are computed whole with per-element masks (pairs outside
// the band get P = dS = 0): at m = 127 a warp's 17 key blocks hold 4,352 products for 4,080
// band edges (+7%; the tensor-core granularity of reading R23).  P and dS are rounded to the
// input type before their MMAs (as the forward rounds P).  Deterministic, no atomics.
#include "tc_common.cuh"

namespace ga {
namespace bwdtc {

using tc::Geo;
using tc::ldsm_x4;
using tc::ldsm_x4_t;
using tc::swz;
constexpr int D = 64, RB = 2 * D, ROWS = 64, WARPS = 4, THREADS = 32 * WARPS, KS = D / 16, NB8 = D / 8;
constexpr int64_t MAX_M = 255;
#ifndef GA_BWD_UNROLL
#define GA_BWD_UNROLL 2 // key / query blocks in flight per warp (1: 1.34 ms, 2: 1.16 ms at cfg2)
#endif
constexpr int UNROLL = GA_BWD_UNROLL;

// the two 16-bit elements of a 32-bit word as floats
template <typename T> __device__ __forceinline__ void unpack2(uint32_t w, float &lo, float &hi);
template <> __device__ __forceinline__ void unpack2<__nv_bfloat16>(uint32_t w, float &lo, float &hi) { bf2_to_f(w, lo, hi); }
template <> __device__ __forceinline__ void unpack2<__half>(uint32_t w, float &lo, float &hi)
{
    const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w));
    lo = f.x;
    hi = f.y;
}

struct Params {
    AttnParams p;
    const void *O, *dO;
    const float *lse_in; // forward lse (log2 domain) or nullptr
    float *lse, *Dv;     // [L, H]: written by the row pass, read by the column pass
    float *dQ, *dK, *dV; // fp32 [L, H, d]
    int64_t m, r, tiles;
};

__host__ __device__ constexpr int64_t band_rows(int64_t m) { return ROWS + (2 * m + 15) / 16 * 16 + 16; }
__host__ __device__ inline uint32_t smem_bytes(int64_t m) { return (uint32_t)(2 * ROWS * RB + 2 * band_rows(m) * RB + 2 * band_rows(m) * 4); }

// A fragments (16 rows x 64) of a swizzled [rows][RB] tile, rows row0..row0+15
__device__ __forceinline__ void load_a(uint32_t base, int row0, int lane, uint32_t (*a)[4])
{
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int row = row0 + (lane & 7) + ((lane >> 3) & 1) * 8;
        ldsm_x4(base + swz<D>(row, 2 * kk + (lane >> 4)), a[kk][0], a[kk][1], a[kk][2], a[kk][3]);
    }
}

// C (16 x 16, 2 n8 blocks) += A (16 x 64) B^T with B = 16 rows x 64 of a swizzled tile at row
// offset `off` bytes (the rows form the N dimension: "B = rows^T")
template <typename T>
__device__ __forceinline__ void mma_abt(float (*c)[4], const uint32_t (*a)[4], uint32_t base, uint32_t off, int lane)
{
    const int krow = (lane & 7) + (lane >> 4) * 8;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(base + swz<D>(krow, 2 * kk + ((lane >> 3) & 1)) + off, b0, b1, b2, b3);
        tc::mma16816<T>(c[0], a[kk], b0, b1);
        tc::mma16816<T>(c[1], a[kk], b2, b3);
    }
}

// acc (16 x 64, NB8 n8 blocks) += P (16 x 16 keys, packed A fragment) B with B = 16 rows x 64
// of a swizzled tile at row offset `off` (the rows form the K dimension)
template <typename T>
__device__ __forceinline__ void mma_pb(float (*acc)[4], const uint32_t *pa, uint32_t base, uint32_t off, int lane)
{
    const int vrow = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
    for (int jj = 0; jj < NB8 / 2; ++jj) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(base + swz<D>(vrow, 2 * jj + (lane >> 4)) + off, b0, b1, b2, b3);
        tc::mma16816<T>(acc[2 * jj], pa, b0, b1);
        tc::mma16816<T>(acc[2 * jj + 1], pa, b2, b3);
    }
}

// stage class rows y0 .. y0 + n - 1 of one (class, head) of a [L, H, D] tensor (zero outside
// [0, Nc)) into a swizzled tile
template <typename T>
__device__ __forceinline__ void stage(uint32_t dst, const void *src, int64_t y0, int n, int64_t Nc, int64_t c,
                                      int64_t r, int H, int h)
{
    // thread t copies chunk t & 7 of rows t / 8 + 16 k: the row's swizzle (row & 7) is the same
    // for every k, so the shared and global addresses advance by constants (no per-copy 64-bit
    // index arithmetic; the staging loops held ~30% of the stall samples)
    static_assert(THREADS % 8 == 0 && (THREADS / 8) % 8 == 0, "16-row steps keep the swizzle phase");
    constexpr int RSTEP = THREADS / 8;
    const int cc = threadIdx.x & 7, b0 = threadIdx.x >> 3;
    const int64_t row_bytes = (int64_t)H * D * sizeof(T), gstep = RSTEP * r * row_bytes;
    uint32_t d = dst + swz<D>(b0, cc);
    int64_t y = y0 + b0, goff = (c + y * r) * row_bytes + (int64_t)h * D * sizeof(T) + cc * 16;
    for (int b = b0; b < n; b += RSTEP, y += RSTEP, d += RSTEP * RB, goff += gstep) {
        if (y >= 0 && y < Nc) tc::cp_async16(d, reinterpret_cast<const char *>(src) + goff);
        else tc::sts_zero16(d);
    }
}

template <typename T>
__device__ __forceinline__ void store_rows(float *dst, const float (*acc)[4], int64_t row_g, int64_t row_g8, bool ok_g,
                                           bool ok_g8, int H, int h, float scale, int lane)
{
    const int t4 = lane & 3;
#pragma unroll
    for (int j = 0; j < NB8; ++j) {
        if (ok_g)
            *reinterpret_cast<float2 *>(dst + ((size_t)row_g * H + h) * D + 8 * j + 2 * t4) =
                make_float2(acc[j][0] * scale, acc[j][1] * scale);
        if (ok_g8)
            *reinterpret_cast<float2 *>(dst + ((size_t)row_g8 * H + h) * D + 8 * j + 2 * t4) =
                make_float2(acc[j][2] * scale, acc[j][3] * scale);
    }
}

template <typename T> __global__ void __launch_bounds__(THREADS) row_kernel(const __grid_constant__ Params bp)
{
    extern __shared__ __align__(1024) unsigned char smem[];
    const AttnParams &p = bp.p;
    const int H = p.H, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
    const int64_t r = bp.r, m = bp.m, L = p.mask.L;
    const int64_t st = blockIdx.y, c = st / H;
    const int h = (int)(st - c * H);
    const int64_t Nc = c < L ? (L - c + r - 1) / r : 0;
    const int64_t x0 = (int64_t)blockIdx.x * ROWS;
    if (x0 >= Nc) return;
    const int nb = (int)band_rows(m);
    const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(smem), sdO = sQ + ROWS * RB, sK = sdO + ROWS * RB,
                   sV = sK + nb * RB;
    float *sD = reinterpret_cast<float *>(smem + 2 * ROWS * RB + 2 * nb * RB);
    const int64_t y0 = x0 - m; // band row 0
    // D = rowsum(dO o O) of the tile's rows (warp w: rows 16w..16w+15): the warp's 32 loads are
    // issued first and used after the staging copies are issued (one memory round trip under
    // the staging; a load-reduce loop per row waited ~16 of them, ~30% of the stall samples)
    const size_t row_bytes = (size_t)H * D * sizeof(T);
    uint32_t wdo[16], wo[16];
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
        const int64_t x = x0 + 16 * warp + rr;
        wdo[rr] = wo[rr] = 0u; // (0 unpacks to +0 in bf16 and fp16)
        if (x < Nc) {
            const size_t off = (size_t)(c + x * r) * row_bytes + (size_t)h * D * sizeof(T) + lane * 4;
            wdo[rr] = __ldg(reinterpret_cast<const unsigned int *>(reinterpret_cast<const char *>(bp.dO) + off));
            wo[rr] = __ldg(reinterpret_cast<const unsigned int *>(reinterpret_cast<const char *>(bp.O) + off));
        }
    }
    stage<T>(sQ, p.Q, x0, ROWS, Nc, c, r, H, h);
    stage<T>(sdO, bp.dO, x0, ROWS, Nc, c, r, H, h);
    stage<T>(sK, p.K, y0, nb, Nc, c, r, H, h);
    stage<T>(sV, p.V, y0, nb, Nc, c, r, H, h);
    tc::cp_async_commit();
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
        float a0, a1, b0, b1;
        unpack2<T>(wdo[rr], a0, a1);
        unpack2<T>(wo[rr], b0, b1);
        float v = a0 * b0 + a1 * b1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sD[16 * warp + rr] = v;
    }
    tc::cp_async_wait<0>();
    __syncthreads();
    const float sl2 = p.scale_log2;
    uint32_t qa[KS][4], da[KS][4];
    load_a(sQ, 16 * warp, lane, qa);
    load_a(sdO, 16 * warp, lane, da);
    const int64_t xg = x0 + 16 * warp + g, xg8 = xg + 8;
    const float Dg = sD[16 * warp + g], Dg8 = sD[16 * warp + g + 8];
    const int nblk = (16 + 2 * (int)m + 15) / 16; // key blocks of the warp: band rows 16w + 16b ..
    // keys of row x in band-row coordinates (y - y0, y0 = x0 - m): [max(0, x - m), min(Nc - 1,
    // x + m)] - y0 = [max(m - x0, x - x0), min(Nc - 1 - y0, x - x0 + 2m)], empty for x >= Nc;
    // 32-bit per-lane bounds instead of 64-bit tests per element
    const int mi = (int)m, xl = 16 * warp + g;
    const int blo = (int)imax(m - x0, 0);
    const int bhi = (int)imin(Nc - 1 - y0, (int64_t)(16 * warp + 16 + 2 * mi + 16));
    const int lo_g = max(blo, xl), hi_g = xg < Nc ? min(bhi, xl + 2 * mi) : -1;
    const int lo_g8 = max(blo, xl + 8), hi_g8 = xg8 < Nc ? min(bhi, xl + 8 + 2 * mi) : -1;
    auto valid = [&](int hr, int yb) { return hr ? (yb >= lo_g8 && yb <= hi_g8) : (yb >= lo_g && yb <= hi_g); };
    // lse of rows g, g + 8 (log2 domain): given (the forward's), or accumulated online in one
    // sweep — dQ is then summed against the running reference max m (P' = 2^(s - m), lazy
    // rescale with a 2^8 threshold like the forward) and divided by l at the end, so S is
    // computed once instead of in a separate lse sweep
    float lse_g = 0.f, lse_g8 = 0.f;
    float dq[NB8][4];
#pragma unroll
    for (int j = 0; j < NB8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
    if (bp.lse_in) {
        lse_g = xg < Nc ? bp.lse_in[(size_t)(c + xg * r) * H + h] : 0.f;
        lse_g8 = xg8 < Nc ? bp.lse_in[(size_t)(c + xg8 * r) * H + h] : 0.f;
#pragma unroll UNROLL
        for (int b = 0; b < nblk; ++b) {
            const int kb = 16 * warp + 16 * b;
            float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}}, dp[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
            mma_abt<T>(s, qa, sK, (uint32_t)kb * RB, lane);
            mma_abt<T>(dp, da, sV, (uint32_t)kb * RB, lane);
            uint32_t pa[4];
#pragma unroll
            for (int n = 0; n < 2; ++n) {
                float ds[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int hr = e >> 1;
                    const float pw = valid(hr, kb + n * 8 + 2 * t4 + (e & 1)) ? ex2(s[n][e] * sl2 - (hr ? lse_g8 : lse_g)) : 0.f;
                    ds[e] = pw * (dp[n][e] - (hr ? Dg8 : Dg));
                }
                pa[2 * n] = pack2<T>(ds[0], ds[1]);
                pa[2 * n + 1] = pack2<T>(ds[2], ds[3]);
            }
            mma_pb<T>(dq, pa, sK, (uint32_t)kb * RB, lane);
        }
    } else {
        float mr[2] = {-INFINITY, -INFINITY}, lr[2] = {0.f, 0.f};
#pragma unroll UNROLL
        for (int b = 0; b < nblk; ++b) {
            const int kb = 16 * warp + 16 * b;
            float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}}, dp[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
            mma_abt<T>(s, qa, sK, (uint32_t)kb * RB, lane);
            mma_abt<T>(dp, da, sV, (uint32_t)kb * RB, lane);
            float v[2][4], bm[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int hr = e >> 1;
                    v[n][e] = valid(hr, kb + n * 8 + 2 * t4 + (e & 1)) ? s[n][e] * sl2 : -INFINITY;
                    bm[hr] = fmaxf(bm[hr], v[n][e]);
                }
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) { // the row's block max over its quad of lanes
                bm[hr] = fmaxf(bm[hr], __shfl_xor_sync(0xffffffffu, bm[hr], 1));
                bm[hr] = fmaxf(bm[hr], __shfl_xor_sync(0xffffffffu, bm[hr], 2));
            }
            const bool n0 = bm[0] > mr[0] + 8.f, n1 = bm[1] > mr[1] + 8.f;
            if (__any_sync(0xffffffffu, n0 || n1)) {
                const float a0 = n0 ? (mr[0] == -INFINITY ? 0.f : ex2(mr[0] - bm[0])) : 1.f;
                const float a1 = n1 ? (mr[1] == -INFINITY ? 0.f : ex2(mr[1] - bm[1])) : 1.f;
                if (n0) mr[0] = bm[0];
                if (n1) mr[1] = bm[1];
                lr[0] *= a0;
                lr[1] *= a1;
#pragma unroll
                for (int j = 0; j < NB8; ++j) {
                    dq[j][0] *= a0;
                    dq[j][1] *= a0;
                    dq[j][2] *= a1;
                    dq[j][3] *= a1;
                }
            }
            const float mu0 = mr[0] == -INFINITY ? 0.f : mr[0], mu1 = mr[1] == -INFINITY ? 0.f : mr[1];
            uint32_t pa[4];
#pragma unroll
            for (int n = 0; n < 2; ++n) {
                float ds[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int hr = e >> 1;
                    const float pw = ex2(v[n][e] - (hr ? mu1 : mu0)); // invalid: 2^-inf = 0
                    lr[hr] += pw;
                    ds[e] = pw * (dp[n][e] - (hr ? Dg8 : Dg));
                }
                pa[2 * n] = pack2<T>(ds[0], ds[1]);
                pa[2 * n + 1] = pack2<T>(ds[2], ds[3]);
            }
            mma_pb<T>(dq, pa, sK, (uint32_t)kb * RB, lane);
        }
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            lr[hr] += __shfl_xor_sync(0xffffffffu, lr[hr], 1);
            lr[hr] += __shfl_xor_sync(0xffffffffu, lr[hr], 2);
        }
        lse_g = lr[0] > 0.f ? mr[0] + __log2f(lr[0]) : 0.f;
        lse_g8 = lr[1] > 0.f ? mr[1] + __log2f(lr[1]) : 0.f;
        const float i0 = lr[0] > 0.f ? 1.f / lr[0] : 0.f, i1 = lr[1] > 0.f ? 1.f / lr[1] : 0.f;
#pragma unroll
        for (int j = 0; j < NB8; ++j) {
            dq[j][0] *= i0;
            dq[j][1] *= i0;
            dq[j][2] *= i1;
            dq[j][3] *= i1;
        }
    }
    const float isd = sl2 * 0.69314718055994531f; // 1 / sqrt(d)
    const int64_t tg = c + xg * r, tg8 = c + xg8 * r;
    store_rows<T>(bp.dQ, dq, tg, tg8, xg < Nc, xg8 < Nc, H, h, isd, lane);
    if (t4 == 0) {
        if (xg < Nc) { bp.lse[(size_t)tg * H + h] = lse_g; bp.Dv[(size_t)tg * H + h] = Dg; }
        if (xg8 < Nc) { bp.lse[(size_t)tg8 * H + h] = lse_g8; bp.Dv[(size_t)tg8 * H + h] = Dg8; }
    }
}

template <typename T> __global__ void __launch_bounds__(THREADS) col_kernel(const __grid_constant__ Params bp)
{
    extern __shared__ __align__(1024) unsigned char smem[];
    const AttnParams &p = bp.p;
    const int H = p.H, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
    const int64_t r = bp.r, m = bp.m, L = p.mask.L;
    const int64_t st = blockIdx.y, c = st / H;
    const int h = (int)(st - c * H);
    const int64_t Nc = c < L ? (L - c + r - 1) / r : 0;
    const int64_t y0 = (int64_t)blockIdx.x * ROWS; // this CTA's key class rows
    if (y0 >= Nc) return;
    const int nb = (int)band_rows(m);
    const uint32_t sK = (uint32_t)__cvta_generic_to_shared(smem), sV = sK + ROWS * RB, sQ = sV + ROWS * RB,
                   sdO = sQ + nb * RB;
    float *sL = reinterpret_cast<float *>(smem + 2 * ROWS * RB + 2 * nb * RB), *sD = sL + nb;
    const int64_t x0 = y0 - m; // query band row 0
    // lse and D of the query band: loads issued before the staging copies, stored after them
    constexpr int NL = (int)((band_rows(MAX_M) + THREADS - 1) / THREADS);
    float lsev[NL], dval[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        const int b = threadIdx.x + k * THREADS;
        const int64_t x = x0 + b;
        const bool in = b < nb && x >= 0 && x < Nc;
        lsev[k] = in ? __ldg(bp.lse + (size_t)(c + x * r) * H + h) : 0.f;
        dval[k] = in ? __ldg(bp.Dv + (size_t)(c + x * r) * H + h) : 0.f;
    }
    stage<T>(sK, p.K, y0, ROWS, Nc, c, r, H, h);
    stage<T>(sV, p.V, y0, ROWS, Nc, c, r, H, h);
    stage<T>(sQ, p.Q, x0, nb, Nc, c, r, H, h);
    stage<T>(sdO, bp.dO, x0, nb, Nc, c, r, H, h);
    tc::cp_async_commit();
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        const int b = threadIdx.x + k * THREADS;
        if (b < nb) {
            sL[b] = lsev[k];
            sD[b] = dval[k];
        }
    }
    tc::cp_async_wait<0>();
    __syncthreads();
    const float sl2 = p.scale_log2;
    uint32_t ka[KS][4], va[KS][4];
    load_a(sK, 16 * warp, lane, ka);
    load_a(sV, 16 * warp, lane, va);
    const int64_t yg = y0 + 16 * warp + g, yg8 = yg + 8;
    const int nblk = (16 + 2 * (int)m + 15) / 16;
    // queries of key y in query-band coordinates (x - x0, x0 = y0 - m): [max(0, y - m), min(Nc - 1,
    // y + m)] - x0 (32-bit per-lane bounds, empty for y >= Nc)
    const int mi = (int)m, yl = 16 * warp + g;
    const int blo = (int)imax(m - y0, 0);
    const int bhi = (int)imin(Nc - 1 - x0, (int64_t)(16 * warp + 16 + 2 * mi + 16));
    const int lo_g = max(blo, yl), hi_g = yg < Nc ? min(bhi, yl + 2 * mi) : -1;
    const int lo_g8 = max(blo, yl + 8), hi_g8 = yg8 < Nc ? min(bhi, yl + 8 + 2 * mi) : -1;
    auto valid = [&](int hr, int xb) { return hr ? (xb >= lo_g8 && xb <= hi_g8) : (xb >= lo_g && xb <= hi_g); };
    float dk[NB8][4], dv[NB8][4];
#pragma unroll
    for (int j = 0; j < NB8; ++j) dk[j][0] = dk[j][1] = dk[j][2] = dk[j][3] = dv[j][0] = dv[j][1] = dv[j][2] = dv[j][3] = 0.f;
#pragma unroll UNROLL
    for (int b = 0; b < nblk; ++b) {
        const int qb = 16 * warp + 16 * b; // query band rows
        float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}}, dp[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        mma_abt<T>(s, ka, sQ, (uint32_t)qb * RB, lane);   // S^T: rows = keys, columns = queries
        mma_abt<T>(dp, va, sdO, (uint32_t)qb * RB, lane); // dP^T
        uint32_t pp[4], pd[4];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
            float pw[4], ds[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int hr = e >> 1, col = qb + n * 8 + 2 * t4 + (e & 1);
                pw[e] = valid(hr, col) ? ex2(s[n][e] * sl2 - sL[col]) : 0.f;
                ds[e] = pw[e] * (dp[n][e] - sD[col]);
            }
            pp[2 * n] = pack2<T>(pw[0], pw[1]);
            pp[2 * n + 1] = pack2<T>(pw[2], pw[3]);
            pd[2 * n] = pack2<T>(ds[0], ds[1]);
            pd[2 * n + 1] = pack2<T>(ds[2], ds[3]);
        }
        mma_pb<T>(dv, pp, sdO, (uint32_t)qb * RB, lane); // dV += P^T dO
        mma_pb<T>(dk, pd, sQ, (uint32_t)qb * RB, lane);  // dK += dS^T Q
    }
    const float isd = sl2 * 0.69314718055994531f;
    const int64_t tg = c + yg * r, tg8 = c + yg8 * r;
    store_rows<T>(bp.dK, dk, tg, tg8, yg < Nc, yg8 < Nc, H, h, isd, lane);
    store_rows<T>(bp.dV, dv, tg, tg8, yg < Nc, yg8 < Nc, H, h, 1.f, lane);
}

template <typename T> static ga_status launch_t(const Params &bp, cudaStream_t s)
{
    const uint32_t smem = smem_bytes(bp.m);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(row_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes(MAX_M));
        cudaFuncSetAttribute(col_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes(MAX_M));
        attr = true;
    }
    const dim3 grid((unsigned)bp.tiles, (unsigned)(bp.r * bp.p.H));
    row_kernel<T><<<grid, THREADS, smem, s>>>(bp);
    GA_CHECK_LAUNCH("bwdtc::row_kernel");
    col_kernel<T><<<grid, THREADS, smem, s>>>(bp);
    GA_CHECK_LAUNCH("bwdtc::col_kernel");
    return GA_OK;
}

} // namespace bwdtc

bool backward_tc_supported(const AttnParams &p, ga_dtype dt)
{
    if (p.mask.kind != K_WINDOW || (dt != GA_BF16 && dt != GA_F16) || p.d != 64) return false;
    const int64_t m = p.mask.m, r = p.mask.r;
    return m >= 1 && m <= bwdtc::MAX_M && r * p.H <= 65535 && (p.mask.L + r - 1) / r / bwdtc::ROWS + 1 < 2147483647;
}

ga_status launch_backward_tc(const AttnParams &p, ga_dtype dt, const void *O, const void *dO, const float *lse_in,
                             float *lse, float *Dv, float *dQ, float *dK, float *dV, cudaStream_t s)
{
    bwdtc::Params bp;
    bp.p = p;
    bp.O = O;
    bp.dO = dO;
    bp.lse_in = lse_in;
    bp.lse = lse;
    bp.Dv = Dv;
    bp.dQ = dQ;
    bp.dK = dK;
    bp.dV = dV;
    bp.m = p.mask.m;
    bp.r = p.mask.r;
    const int64_t Nc0 = (p.mask.L + bp.r - 1) / bp.r; // longest class
    bp.tiles = (Nc0 + bwdtc::ROWS - 1) / bwdtc::ROWS;
    if (bp.tiles == 0) return GA_OK;
    return dt == GA_BF16 ? bwdtc::launch_t<__nv_bfloat16>(bp, s) : bwdtc::launch_t<__half>(bp, s);
}

} // namespace ga

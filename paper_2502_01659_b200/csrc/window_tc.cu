// window_tc.cu — tcgen05 (5th-gen tensor core, TMEM accumulators) kernel for Window(w, r)
// masks, bf16/fp16, d = 64, band half-width 64 <= m <= 128 (cfg2: Window(256, 2), cfg5:
// Window(128, 1); both m = 127).
//
// Residue class c of a dilated window is a band (readings R1/R2): class
// row x sees class rows [x - m, x + m] ∩ [0, Nc).  A 128-row query tile (thread = row = TMEM
// lane) meets the keys of 64-key chunks g (class rows [64g, 64g + 64)) with
// g in [floor((a0 - m)/64), floor((a0 + 127 + m)/64)] — 6 chunks at m = 127, of which the
// middle two are dense for every row and the outer ones hold the band's two triangles.  Per
// chunk:
//
//   S  = Q K_g^T      tcgen05.mma.cta_group::1.kind::f16 M=128 N=64 (K=16 x 4), A (Q tile) and
//                     B (K chunk) from 128B-swizzled shared memory, fp32 accumulator in TMEM
//   softmax           each thread tcgen05.ld's its row of S, 32 columns at a time; a 32-column
//                     half no row of the warp reaches is neither loaded nor exponentiated
//                     (P = 0), a half every row reaches fully is used as is, and only the
//                     halves the band's edges cross are masked per element (keys outside the
//                     row's band get weight exactly 0); chunk max first, online softmax in the
//                     exp2 domain with lazy rescale (2^8); P (bf16/fp16 pairs) to TMEM
//   O += P V_g        tcgen05.mma with A = P from TMEM, B = V_g (MN-major) from shared memory
//
// The tensor cores see whole 128 x 64 chunks (66% of the products valid at m = 127: 32,640
// band edges of 49,152 per tile; reading R23); exponentials, sums and weights are computed
// only for the 32-column halves a warp's rows reach, and a masked pair contributes exactly 0
// — the result is the Algorithm 1 result over the band's edges.
//
// CTA organisation (persistent, one CTA per SM, 512 TMEM columns, 16 warps = 4 warpgroups):
//   warps 0-3   softmax warpgroup A: even tiles of a tile pair   (TMEM cols   0..255)
//   warps 4-7   softmax warpgroup B: odd tiles                    (TMEM cols 256..511)
//   warps 8-11  epilogue warpgroup: O of a finished tile from TMEM, normalised by the row sum
//               the softmax left in shared memory, staged in the tile's Q buffer and stored by
//               TMA (or the carried (m, l, o~) state) — off the softmax warps' critical path
//   warp 12     loader: TMA boxes of the Q tiles (2 x 64 class rows, element stride r) and the
//               K/V chunks into a 9-slot ring (slot = g mod 9); peer rows (sharded runs) by
//               cp.async from the owner's memory
//   warps 13-14 MMA issuers, one per softmax warpgroup (one elected lane issues); warp 15 idle
//               (it completes warpgroup 3 for setmaxnreg: softmax 160 registers, epilogue 104,
//               loader / issuers 88)
// TMEM of a warpgroup: S[2] (64 columns each) | P[2] (32 each: 16-bit pairs) | O (64).  S(c + 2)
// is issued into S(c)'s buffer as soon as P(c) arrived (the softmax has read S(c)), so S is
// computed two chunks ahead of the softmax; the epilogue reads a finished tile's O while the
// softmax works on the next tile's first chunk, before that chunk's P V may overwrite it
// (GA_WTC_PSEP=0: P over S, S(c + 2) after P V(c) completed, O[k & 1]).  A CTA walks a contiguous run of
// tile pairs of one (class, head) stream (an item cursor, no per-tile divisions): consecutive
// pairs share 4 of their 8 chunks, which stay resident (each K/V row is read from L2/HBM about
// once per run).
#include <cstdlib>

#include "tc_common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace ga {
namespace wtc {
using namespace tc;
using namespace umma;

constexpr int ROWS = 128, KC = 64, NSLOT = 9, D = 64, RB = 2 * D;
#ifndef GA_WTC_PRELOAD
#define GA_WTC_PRELOAD 0 // 1: load S(c + 1) right after issuing the P(c) stores (measured slower: 25.5 vs 24.4 ms at cfg5)
#endif
constexpr int W_EPI = 8, W_LOAD = 12, W_MMA = 13; // warp 15 only completes warpgroup 3
constexpr int THREADS = 32 * 16;
// registers per thread after setmaxnreg (per SM sub-partition: one warp of each warpgroup,
// 2 x 160 + 104 + 88 = 512 = the 16K registers of the sub-partition / 32 lanes).  168 for the
// softmax left the loader / issuers 72 and they spilled (20 B); 160 / 88 is spill-free and
// measured 0.4-1.1% faster at cfg5 (same box); 176 spills 144 B, and the epilogue spills below
// 104 (96: 24 B, 88 with the softmax at 168: 32 B).
#ifndef GA_WTC_REG_SMX
#define GA_WTC_REG_SMX 160
#endif
#ifndef GA_WTC_REG_EPI
#define GA_WTC_REG_EPI 104
#endif
constexpr int REG_SMX = GA_WTC_REG_SMX, REG_EPI = GA_WTC_REG_EPI, REG_PROD = 512 - 2 * REG_SMX - REG_EPI;
static_assert(REG_SMX % 8 == 0 && REG_EPI % 8 == 0 && REG_PROD % 8 == 0 && REG_PROD >= 24 && REG_SMX <= 256,
              "setmaxnreg takes multiples of 8 in [24, 256]");
constexpr uint32_t QBYTES = ROWS * RB;   // 16 KB
constexpr uint32_t CBYTES = KC * RB;     // 8 KB: one K or V chunk
constexpr uint32_t OFF_Q = 0;            // Q[wg][buf]: 4 x 16 KB (a finished tile's O is staged in its Q buffer)
constexpr uint32_t OFF_KV = 4 * QBYTES;  // slot s: K at OFF_KV + 2 s CBYTES, V right after
constexpr uint32_t OFF_LM = OFF_KV + NSLOT * 2 * CBYTES; // float [wg][buf][l | m][128]
constexpr uint32_t OFF_BAR = OFF_LM + 2 * 2 * 2 * ROWS * 4;
constexpr uint32_t SMEM_BYTES = 1024 + OFF_BAR + 64 * 8;
static_assert(SMEM_BYTES <= 232448, "shared memory");

// TMEM columns within a warpgroup's 256: S[2] | P[2] | O — P in columns of its own, so S(c + 2)
// is issued as soon as P(c) arrived (no wait for P V(c)); one O accumulator: a tile's first
// P V waits for the epilogue to have read the previous tile's O, which it does while the
// softmax works on the tile's first chunk (cfg5 25.03 -> 24.81 ms, cfg2 109 -> 108 us, same
// box).  GA_WTC_PSEP=0: P over the first 32 columns of S[c & 1], O[2].
#ifndef GA_WTC_PSEP
#define GA_WTC_PSEP 1
#endif
#if GA_WTC_PSEP
constexpr uint32_t COL_S = 0, COL_P = 128, COL_O = 192;
#else
constexpr uint32_t COL_S = 0, COL_O = 128;
#endif

// mbarrier indices (8 bytes each from OFF_BAR); [w] = softmax warpgroup, [b] = buffer parity
constexpr int B_QFULL = 0,             // [w][b] (loader TMA)
    B_QEMPTY = 4,                      // [w][b] 4 epilogue warps: O store read the staging buffer
    B_KVFULL = 8,                      // [slot]
    B_KVEMPTY = B_KVFULL + NSLOT,      // [slot] 2 issuers
    B_SFULL = B_KVEMPTY + NSLOT,       // [w][c & 1] S MMA committed
    B_PFULL = B_SFULL + 4,             // [w][c & 1] 128 softmax threads read S and wrote P
    B_OFULL = B_PFULL + 4,             // [w][c & 1] P V MMA committed
    B_OTILE = B_OFULL + 4,             // [w][k & 1] last P V of tile k committed
    B_EPI = B_OTILE + 4,               // [w][k & 1] 128 softmax threads wrote (l, m) of tile k
    B_OFREE = B_EPI + 4,               // [w][k & 1] 128 epilogue threads read O of tile k
    B_TMEM = B_OFREE + 4;              // tcgen05.alloc writes the TMEM base here
static_assert(B_TMEM < 64, "barrier area");

struct TcParams {
    CUtensorMap tmQ, tmK, tmV, tmO; // one head, element stride r, 64-row boxes
    AttnParams p;
    int64_t m, r;
    int64_t pps;   // tile pairs per (class, head) stream
    int64_t items; // streams x pps
};

__host__ __device__ inline int64_t floordiv(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Position of a work item (a pair of consecutive 128-row tiles of one (class, head) stream).
// A CTA walks a contiguous run of items, so every role keeps a cursor and advances it: the
// divisions by runtime values (items per stream, heads, dilation) run once per stream, not per
// tile — on sm_100 they use MUFU.RCP, which the softmax warps' exponentials keep busy.
struct Cur {
    int32_t st, u, c, h;    // stream = class * H + head, pair index in the stream
    int32_t Nc, a_lo, a_hi; // class rows, query class rows [a_lo, a_hi)
};

__device__ __forceinline__ void cur_stream(const TcParams &tp, Cur &C)
{
    const AttnParams &p = tp.p;
    const uint32_t r = (uint32_t)tp.r, L = (uint32_t)p.mask.L, c = (uint32_t)C.c;
    const uint32_t Nc = c < L ? (L - c + r - 1) / r : 0;
    const uint32_t qb = (uint32_t)p.q_begin, qe = (uint32_t)(p.q_begin + p.q_rows);
    C.Nc = (int32_t)Nc;
    C.a_lo = (int32_t)(qb > c ? (qb - c + r - 1) / r : 0);
    C.a_hi = (int32_t)(qe > c ? min((qe - c + r - 1) / r, Nc) : 0);
}

__device__ __forceinline__ Cur cur_init(const TcParams &tp, int32_t it)
{
    // 32-bit arithmetic throughout: L < 2^31 (window_tc_supported)
    const uint32_t H = (uint32_t)tp.p.H, pps = (uint32_t)tp.pps, iu = (uint32_t)it, st = iu / pps;
    Cur C;
    C.st = (int32_t)st;
    C.u = (int32_t)(iu - st * pps);
    C.c = (int32_t)(st / H);
    C.h = (int32_t)(st - (uint32_t)C.c * H);
    cur_stream(tp, C);
    return C;
}

__device__ __forceinline__ void cur_next(const TcParams &tp, Cur &C)
{
    if (++C.u == (int32_t)tp.pps) {
        C.u = 0;
        ++C.st;
        if (++C.h == tp.p.H) {
            C.h = 0;
            ++C.c;
            cur_stream(tp, C);
        }
    }
}

struct Pair {
    int32_t stream, u, c, Nc, a_lo, a_hi;
    int h;
    int32_t a0[2];  // first class row of tile A / B
    bool valid[2];
    int32_t F[2], n[2]; // chunks [F, F + n) per tile
    int32_t lo, hi;     // union of the chunk ranges
    bool any;
};

__device__ __forceinline__ Pair pair_at(const TcParams &tp, const Cur &C)
{
    const int32_t m = (int32_t)tp.m;
    Pair P;
    P.stream = C.st;
    P.u = C.u;
    P.c = C.c;
    P.h = C.h;
    P.Nc = C.Nc;
    P.a_lo = C.a_lo;
    P.a_hi = C.a_hi;
    const int32_t t0 = (C.a_lo >> 7) + 2 * C.u; // ROWS = 128
    const int32_t lastc = (C.Nc - 1) >> 6;       // KC = 64
    P.lo = INT32_MAX;
    P.hi = -1;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
        const int32_t a0 = (t0 + w) * ROWS;
        P.a0[w] = a0;
        P.valid[w] = C.a_lo < C.a_hi && a0 < C.a_hi;
        // floor((a0 - m) / 64) by arithmetic shift (exact for negative values too)
        const int32_t f = max((a0 - m) >> 6, 0), e = min((a0 + ROWS - 1 + m) >> 6, lastc);
        P.F[w] = f;
        P.n[w] = P.valid[w] ? e - f + 1 : 0;
        if (P.valid[w]) {
            P.lo = min(P.lo, f);
            P.hi = max(P.hi, e);
        }
    }
    P.any = P.valid[0];
    return P;
}

// One warpgroup's tile of a work item (scalar fields: no dynamically indexed arrays, which
// would live in local memory)
struct Tile {
    int32_t c, h, Nc, a_lo, a_hi, a0, F, n;
    bool valid;
};

__device__ __forceinline__ Tile tile_at(const TcParams &tp, const Cur &C, int w)
{
    const int32_t m = (int32_t)tp.m;
    Tile T;
    T.c = C.c;
    T.h = C.h;
    T.Nc = C.Nc;
    T.a_lo = C.a_lo;
    T.a_hi = C.a_hi;
    T.a0 = ((C.a_lo >> 7) + 2 * C.u + w) * ROWS;
    T.valid = C.a_lo < C.a_hi && T.a0 < C.a_hi;
    T.F = max((T.a0 - m) >> 6, 0);
    T.n = T.valid ? min((T.a0 + ROWS - 1 + m) >> 6, (C.Nc - 1) >> 6) - T.F + 1 : 0;
    return T;
}

__device__ __forceinline__ uint32_t bar(uint32_t base, int i) { return base + 8u * (uint32_t)i; }

#ifdef GA_WTC_TRACE
// debug timeline of CTA 0: (value << 56 | event << 48 | warp << 40 | (clock - t0)) per event
constexpr int TRACE_N = 16384;
__device__ unsigned long long g_trace[TRACE_N];
// per-warp private slots (no atomics: a trace point costs one store)
#define TRACE2(ev, val) do { if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && t_cnt < TRACE_N / 16) { \
    g_trace[(threadIdx.x >> 5) * (TRACE_N / 16) + t_cnt++] = ((unsigned long long)((val) & 0xff) << 56) | \
        ((unsigned long long)(ev) << 48) | ((unsigned long long)(threadIdx.x >> 5) << 40) | \
        (unsigned long long)((clock64() - t_origin) & 0xffffffffffull); } } while (0)
#define TRACE(ev) TRACE2(ev, 0)
#else
#define TRACE(ev)
#define TRACE2(ev, val)
#endif

// keys outside [il, ih] (row-relative column bounds within a 32-column half) -> -inf
__device__ __forceinline__ void mask_half(float *s, int il, int ih, bool left, bool right)
{
    if (left) {
#pragma unroll
        for (int i = 0; i < 32; ++i) s[i] = i >= il ? s[i] : -INFINITY;
    }
    if (right) {
#pragma unroll
        for (int i = 0; i < 32; ++i) s[i] = i <= ih ? s[i] : -INFINITY;
    }
}

__device__ __forceinline__ float max32(const float *s)
{
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaxf(s[i], fmaxf(s[i + 8], s[i + 16]));
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaxf(a[i], s[i + 24]);
    return fmaxf(fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3])), fmaxf(fmaxf(a[4], a[5]), fmaxf(a[6], a[7])));
}

// P of one 32-column half: pk = pack(2^(s * sl2 - m)) (16 words), row-sum partials in acc.
// With POLY > 0 the first POLY pairs take 2^x from a degree-3 polynomial on the FMA pipe
// (ex2_poly2, relative error 7.6e-5, below the bf16/fp16 rounding of P) instead of MUFU, which
// the two softmax warps of a sub-partition share; only for halves without masked keys
// (ex2_poly2 maps -inf to 2^-126, not 0).
#ifndef GA_WTC_POLY
#define GA_WTC_POLY 0
#endif
template <typename T, int POLY>
__device__ __forceinline__ void exps_half(float *s, float sl2, float negm, uint32_t *pk, float2 *acc)
{
#pragma unroll
    for (int i = 0; i < 16; ++i) ffma2_sm(s[2 * i], s[2 * i + 1], sl2, negm);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (i < POLY) {
            ex2_poly2(s[2 * i], s[2 * i + 1]);
        } else {
            s[2 * i] = ex2(s[2 * i]);
            s[2 * i + 1] = ex2(s[2 * i + 1]);
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        fadd2_acc(acc[i & 3], s[2 * i], s[2 * i + 1]);
        pk[i] = pack2<T>(s[2 * i], s[2 * i + 1]);
    }
}

template <typename T, bool PROBE> // PROBE: count (edge_counter / tensor_counter), a separate instantiation
__global__ void __launch_bounds__(THREADS, 1) window_tc_kernel(const __grid_constant__ TcParams tp)
{
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    unsigned char *const sgen = smem_raw + (sbase - raw); // generic pointer to sbase
    const uint32_t bars = sbase + OFF_BAR;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sgen + OFF_BAR + 8 * B_TMEM);
    float *const lmbuf = reinterpret_cast<float *>(sgen + OFF_LM); // [w][b][l | m][128]
    const AttnParams &p = tp.p;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m = tp.m, r = tp.r;
    const int H = p.H;
    const size_t row_bytes = (size_t)H * D * sizeof(T);

    // contiguous run of work items
    const int32_t it_begin = (int32_t)(tp.items * blockIdx.x / gridDim.x),
                  it_end = (int32_t)(tp.items * (blockIdx.x + 1) / gridDim.x);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(bar(bars, B_QFULL + i), 1);
            mbar_init(bar(bars, B_QEMPTY + i), 4);
            mbar_init(bar(bars, B_PFULL + i), 128);
            mbar_init(bar(bars, B_OFULL + i), 1);
            mbar_init(bar(bars, B_OTILE + i), 1);
            mbar_init(bar(bars, B_EPI + i), 128);
            mbar_init(bar(bars, B_OFREE + i), 128);
        }
        for (int i = 0; i < 4; ++i) mbar_init(bar(bars, B_SFULL + i), 1);
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(bar(bars, B_KVFULL + s), 1);
            mbar_init(bar(bars, B_KVEMPTY + s), 2); // both issuers release every fill
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
#ifdef GA_WTC_TRACE
    const long long t_origin = clock64();
    int t_cnt = 0;
#endif

    if (warp >= 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REG_PROD));
    if (warp == W_LOAD) {
        // ============================ loader ============================
        // per slot: filled before (bit s of `used`), parity of the fill count (bit s of `par`);
        // bitmasks, not arrays (a dynamically indexed array would live in local memory)
        uint32_t used = 0, par = 0;
        int nq[2] = {0, 0};
        int32_t prev_stream = -1, prev_u = -1, prev_hi = -1;
        Cur C = cur_init(tp, it_begin);
        for (int32_t it = it_begin; it < it_end; ++it, cur_next(tp, C)) {
            const Pair P = pair_at(tp, C);
            if (!P.any) continue;
            // Q tiles
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                if (!P.valid[w]) continue;
                const int b = nq[w] & 1;
                if (nq[w] >= 2) mbar_wait(bar(bars, B_QEMPTY + 2 * w + b), ((nq[w] >> 1) - 1) & 1);
                ++nq[w];
                if (elect_one()) {
                    const uint32_t fb = bar(bars, B_QFULL + 2 * w + b);
                    tma::expect_tx(fb, QBYTES);
                    const uint32_t dst = sbase + OFF_Q + (uint32_t)(2 * w + b) * QBYTES;
                    const int tok = (int)(P.c + P.a0[w] * r - p.q_begin);
                    tma::load_3d(dst, &tp.tmQ, 0, P.h, tok, fb);
                    tma::load_3d(dst + QBYTES / 2, &tp.tmQ, 0, P.h, tok + 64 * (int)r, fb);
                }
                __syncwarp();
            }
            // K/V chunks not resident from the previous pair
            const bool cont = P.stream == prev_stream && P.u == prev_u + 1;
            for (int32_t g = P.lo; g <= P.hi; ++g) {
                if (cont && g <= prev_hi) continue;
                const int s = (int)((uint32_t)g % NSLOT);
                // fill n of slot s waits for release n - 1 (parity of n - 1 = complement of n's)
                if ((used >> s) & 1u) mbar_wait(bar(bars, B_KVEMPTY + s), ((par >> s) & 1u) ^ 1u);
                TRACE2(20, g);
                used |= 1u << s;
                par ^= 1u << s;
                const uint32_t fb = bar(bars, B_KVFULL + s);
                const uint32_t dK = sbase + OFF_KV + (uint32_t)s * 2 * CBYTES, dV = dK + CBYTES;
                const int64_t tok0 = P.c + (int64_t)g * KC * r;                     // first row's token
                const int64_t tokL = P.c + (int64_t)min(g * KC + KC - 1, P.Nc - 1) * r; // last in-range row
                const bool local = p.k_peer == nullptr || (tok0 >= p.kv_begin && tokL < p.kv_begin + p.kv_rows);
                if (local) {
                    if (elect_one()) {
                        tma::expect_tx(fb, 2 * CBYTES);
                        tma::load_3d(dK, &tp.tmK, 0, P.h, (int)(tok0 - p.kv_begin), fb);
                        tma::load_3d(dV, &tp.tmV, 0, P.h, (int)(tok0 - p.kv_begin), fb);
                    }
                } else {
                    // rows owned by other ranks: 16-byte cp.async from the owner's buffer
                    const size_t hoff = (size_t)P.h * D * sizeof(T);
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const int row = lane + 32 * half;
                        const int32_t kr = g * KC + row;
                        if (kr < P.Nc) {
                            const char *kp, *vp;
                            kv_row(p, P.c + (int64_t)kr * r, row_bytes, kp, vp);
#pragma unroll
                            for (int cc = 0; cc < RB / 16; ++cc) {
                                cp_async16(dK + swz<D>(row, cc), kp + hoff + cc * 16);
                                cp_async16(dV + swz<D>(row, cc), vp + hoff + cc * 16);
                            }
                        } else {
#pragma unroll
                            for (int cc = 0; cc < RB / 16; ++cc) {
                                sts_zero16(dK + swz<D>(row, cc));
                                sts_zero16(dV + swz<D>(row, cc));
                            }
                        }
                    }
                    cp_async_commit(); // wait_group only covers committed groups
                    cp_async_wait<0>();
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(fb);
                }
                __syncwarp();
            }
            prev_stream = P.stream;
            prev_u = P.u;
            prev_hi = P.hi;
        }
    } else if (warp == W_MMA || warp == W_MMA + 1) {
        // ============================ MMA issuers ============================
        // Issuer w serves softmax warpgroup w (its tile of every item).  Warp-uniform control
        // flow (the whole warp runs the schedule and the blocking waits; one elected lane
        // issues).  Per chunk j of a tile (c: running counter over the warpgroup's tiles):
        //     S(c + 1) into S buffer (c + 1) & 1, whose S(c - 1) the softmax has read (P(c - 1)
        //     arrived; with GA_WTC_PSEP=0, P(c - 1) lives there and P V(c - 1) must complete
        //     first); then P V(c) once P(c) arrived — so S runs two chunks ahead of the softmax.
        // The first two S of the next tile are issued around this tile's last P V (when the next
        // Q tile has landed).  Both issuers arrive once on a slot's empty barrier per fill: after
        // their last P V reading the chunk, or — for a chunk their tile does not read — after
        // observing the fill, so an arrival never lands in the previous fill's phase.
        const int w = warp - W_MMA;
        const uint32_t idS = idesc<T>(ROWS, KC, false), idO = idesc<T>(ROWS, D, true);
        // smem descriptors: constant high part | (address >> 4); the operand tiles stay below
        // 256 KB so the 14-bit start field never carries
        const uint64_t dbase = sdesc_sw128(0);
        const uint32_t tw = tmem + 256u * (uint32_t)w;
        uint32_t seen = 0;      // parity of the fills waited for, bit per slot
        int nq = 0;             // Q tiles waited
        uint32_t cs = 0;        // S MMAs issued (chunk counter of the warpgroup)
        uint32_t k = 0;         // tiles of the warpgroup (O buffer parity)
        int pre = 0;            // S MMAs of this item's tile already issued (end of the previous item)
        bool preq = false;      // ... and its Q tile waited for
        int32_t prev_stream = -1, prev_u = -1, prev_lo = 0;
        uint32_t waited = 0; // fills this issuer observed, bit g - lo of the previous item
        Cur C = cur_init(tp, it_begin);
        Pair N = pair_at(tp, C);
        for (int32_t it = it_begin; it < it_end; ++it) {
            const Pair P = N;
            const bool has_next = it + 1 < it_end;
            cur_next(tp, C);
            if (has_next) N = pair_at(tp, C);
            if (!P.any) continue;
            const bool cont = P.stream == prev_stream && P.u == prev_u + 1;
            const bool next_cont = has_next && N.any && N.stream == P.stream && N.u == P.u + 1;
            const int32_t keep_from = next_cont ? N.lo : INT32_MAX;
            // chunks resident from the previous item whose fill this issuer already observed
            uint32_t ready = cont ? waited >> (P.lo - prev_lo) : 0u;
            const bool valid = w == 0 ? P.valid[0] : P.valid[1];
            const int32_t f = w == 0 ? P.F[0] : P.F[1], n = valid ? (w == 0 ? P.n[0] : P.n[1]) : 0;
            auto chunk_ready = [&](int32_t g) {
                const int gi = (int)(g - P.lo);
                if ((ready >> gi) & 1u) return;
                const int sl = (int)((uint32_t)g % NSLOT);
                mbar_wait(bar(bars, B_KVFULL + sl), (seen >> sl) & 1u);
                seen ^= 1u << sl;
                ready |= 1u << gi;
                fence_after();
            };
            auto release_unread = [&](int32_t g) {
                chunk_ready(g);
                if (elect_one()) mma_commit(bar(bars, B_KVEMPTY + (int)((uint32_t)g % NSLOT)));
                __syncwarp();
            };
            int qb = 0;
            if (valid) {
                if (preq) {
                    qb = (nq - 1) & 1;
                } else {
                    qb = nq & 1;
                    mbar_wait(bar(bars, B_QFULL + 2 * w + qb), (nq >> 1) & 1);
                    ++nq;
                    fence_after();
                }
            }
            // chunks of the item below this tile's range that the next item does not keep
            for (int32_t g = P.lo; g < (n ? f : P.hi + 1) && g < keep_from; ++g) release_unread(g);
            auto issue_S = [&](uint32_t c, int32_t g, int qbuf) {
                // S buffer c & 1 held S / P of chunk c - 2: free once P V(c - 2) completed
                // (P in its own columns: once the softmax read S(c - 2), i.e. P(c - 2) arrived)
                if (!GA_WTC_PSEP && c >= 2) mbar_wait(bar(bars, B_OFULL + 2 * w + (int)(c & 1)), ((c - 2) >> 1) & 1);
                fence_after();
                const uint32_t aq = sbase + OFF_Q + (uint32_t)(2 * w + qbuf) * QBYTES;
                const uint32_t ak = sbase + OFF_KV + ((uint32_t)g % NSLOT) * 2 * CBYTES;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        mma_ss(tw + COL_S + (c & 1u) * KC, dbase | ((aq + kk * 32) >> 4), dbase | ((ak + kk * 32) >> 4),
                               idS, kk > 0);
                    mma_commit(bar(bars, B_SFULL + 2 * w + (int)(c & 1)));
                    if (PROBE && p.tensor_counter) atomicAdd(p.tensor_counter, (unsigned long long)(ROWS * KC)); // probe
                }
                __syncwarp();
                TRACE2(6, g);
            };
            const uint32_t c0 = cs - (uint32_t)pre; // chunk counter of this tile's chunk 0
            int32_t si = pre;                       // S MMAs of this tile issued
            auto issue_PV = [&](int32_t j) {
                const uint32_t c = c0 + (uint32_t)j;
                const int32_t g = f + j;
                mbar_wait(bar(bars, B_PFULL + 2 * w + (int)(c & 1)), (c >> 1) & 1);
                TRACE2(3, g);
#if GA_WTC_PSEP
                if (j == 0 && k >= 1) mbar_wait(bar(bars, B_OFREE + 2 * w + (int)((k - 1) & 1)), ((k - 1) >> 1) & 1);
#else
                if (j == 0 && k >= 2) mbar_wait(bar(bars, B_OFREE + 2 * w + (int)(k & 1)), ((k - 2) >> 1) & 1);
#endif
                fence_after();
                const int sl = (int)((uint32_t)g % NSLOT);
                const uint32_t av = sbase + OFF_KV + (uint32_t)sl * 2 * CBYTES + CBYTES;
#if GA_WTC_PSEP
                const uint32_t tP = tw + COL_P + (c & 1u) * (KC / 2);
                const uint32_t tO = tw + COL_O;
#else
                const uint32_t tP = tw + COL_S + (c & 1u) * KC;
                const uint32_t tO = tw + COL_O + (k & 1u) * D;
#endif
                const bool release = g < keep_from; // each chunk is read once per tile
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < KC / 16; ++kk) // 16 keys per MMA: 8 P columns, 16 V rows
                        mma_ts(tO, tP + kk * 8, dbase | ((av + kk * 16 * RB) >> 4), idO, (j > 0 || kk > 0));
                    mma_commit(bar(bars, B_OFULL + 2 * w + (int)(c & 1)));
                    if (j == n - 1) mma_commit(bar(bars, B_OTILE + 2 * w + (int)(k & 1)));
                    if (release) mma_commit(bar(bars, B_KVEMPTY + sl));
                }
                __syncwarp();
            };
            // next tile's first S MMAs (chunks resident, Q landed): issued at the end of this tile
            int npre = 0;
            bool nqw = false;
            const bool nvalid = n > 0 && next_cont && (w == 0 ? N.valid[0] : N.valid[1]);
            const int32_t nf = w == 0 ? N.F[0] : N.F[1], nn = w == 0 ? N.n[0] : N.n[1];
            auto prefetch = [&](int jn) {
                if (!nvalid || jn >= nn || npre != jn) return;
                const int32_t g = nf + jn;
                if (g > P.hi || !((ready >> (int)(g - P.lo)) & 1u)) return;
                if (!nqw) {
                    const uint32_t qf = bar(bars, B_QFULL + 2 * w + (nq & 1));
                    if (!mbar_test(qf, (nq >> 1) & 1)) return;
                    ++nq;
                    nqw = true;
                }
                issue_S(cs, g, (nq - 1) & 1);
                ++cs;
                ++npre;
            };
            for (int32_t j = 0; j < n; ++j) {
                // S two chunks ahead of the softmax (S[2] in TMEM)
                for (; si <= min(j + 1, n - 1); ++si) {
                    chunk_ready(f + si);
                    issue_S(cs, f + si, qb);
                    ++cs;
                }
                if (j == n - 1) prefetch(0);
                issue_PV(j);
            }
            if (n > 0) ++k;
            prefetch(1);
            // chunks above this tile's range that the next item does not keep
            for (int32_t g = (n ? f + n : P.hi + 1); g <= P.hi && g < keep_from; ++g) release_unread(g);
            pre = npre;
            preq = nqw;
            prev_stream = P.stream;
            prev_u = P.u;
            prev_lo = P.lo;
            waited = ready;
        }
    }
    } else if (warp >= W_EPI) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REG_EPI));
        // ============================ epilogue warpgroup ============================
        // Tiles in item order (A then B): wait for the tile's last P V and its row sums, read O
        // (then hand the O buffer back to the issuer), normalise, store.  Warp q owns TMEM lanes
        // 32q..32q+31 (rows 32q.. of both warpgroups' tiles).
        const int q = warp - W_EPI;
        uint32_t ke0 = 0, ke1 = 0; // tiles per warpgroup (scalars: no local memory)
        bool pend_rel = false;
        int pend_w = 0;
        uint32_t pend_b = 0;
        auto release = [&]() { // the previous O store has read its staging buffer
            if (lane == 0) {
                tma::store_wait_read();
                mbar_arrive(bar(bars, B_QEMPTY + 2 * pend_w + (int)pend_b));
            }
            __syncwarp();
            pend_rel = false;
        };
        Cur C = cur_init(tp, it_begin);
        for (int32_t it = it_begin; it < it_end; ++it, cur_next(tp, C)) {
#pragma unroll 1
            for (int w = 0; w < 2; ++w) {
                const Tile Tq = tile_at(tp, C, w);
                if (!Tq.valid) continue;
                const uint32_t k = w == 0 ? ke0++ : ke1++, b = k & 1u;
                mbar_wait(bar(bars, B_EPI + 2 * w + (int)b), (k >> 1) & 1);
                mbar_wait(bar(bars, B_OTILE + 2 * w + (int)b), (k >> 1) & 1);
                fence_after();
                TRACE2(18 + w, 0);
                const int row = 32 * q + lane;
                const float l = lmbuf[((w * 2 + (int)b) * 2 + 0) * ROWS + row];
                const float mrow = lmbuf[((w * 2 + (int)b) * 2 + 1) * ROWS + row];
                const uint32_t tO = tmem + 256u * (uint32_t)w + ((uint32_t)(q * 32) << 16) + COL_O + (GA_WTC_PSEP ? 0u : b * D);
                float o[64];
                tmem_ld32(tO, o);
                tmem_ld32(tO + 32, o + 32);
                tmem_wait_ld();
                fence_before();
                mbar_arrive(bar(bars, B_OFREE + 2 * w + (int)b)); // O buffer and (l, m) read
                if (pend_rel) release();
                const int32_t x = Tq.a0 + row;
                const bool cut = !(Tq.a0 >= Tq.a_lo && Tq.a0 + ROWS <= Tq.a_hi);
                const bool xv = x >= Tq.a_lo && x < Tq.a_hi;
                const int64_t t = (int64_t)Tq.c + (int64_t)x * r - p.q_begin; // local query row
                if (p.state.m) {
                    // carried state (ga_state): this row's (m, l, o~) in the log2
                    // domain, written or (+)-combined into the caller's fp32 buffers (m is the
                    // row's softmax reference: its running max, or within 2^8 of it after a lazy
                    // rescale — any reference combines exactly); with p.out also the normalised row
                    if (xv) {
                        const size_t rh = (size_t)t * H + Tq.h;
                        float mm = mrow, ll = l, a = 1.f, bb = 0.f;
                        bool mix = false;
                        if (p.state_mode == GA_STATE_ACCUMULATE) {
                            const float l2 = p.state.l[rh];
                            if (l2 > 0.f) { // l == 0 marks an empty state (its m is ignored)
                                const float m2 = p.state.m[rh];
                                const float mn = ll > 0.f ? fmaxf(mm, m2) : m2;
                                a = ll > 0.f ? ex2(mm - mn) : 0.f;
                                bb = ex2(m2 - mn);
                                ll = ll * a + l2 * bb;
                                mm = mn;
                                mix = true;
                            }
                        }
                        const float inv = ll > 0.f ? 1.f / ll : 0.f;
                        float4 *so = reinterpret_cast<float4 *>(p.state.o + rh * D);
#pragma unroll
                        for (int qq = 0; qq < 16; ++qq) {
                            float4 v = make_float4(o[4 * qq], o[4 * qq + 1], o[4 * qq + 2], o[4 * qq + 3]);
                            if (mix) {
                                const float4 uu = so[qq];
                                v.x = v.x * a + uu.x * bb;
                                v.y = v.y * a + uu.y * bb;
                                v.z = v.z * a + uu.z * bb;
                                v.w = v.w * a + uu.w * bb;
                            }
                            so[qq] = v;
                            o[4 * qq] = v.x * inv;
                            o[4 * qq + 1] = v.y * inv;
                            o[4 * qq + 2] = v.z * inv;
                            o[4 * qq + 3] = v.w * inv;
                        }
                        if (p.out) {
                            char *orow = reinterpret_cast<char *>(p.out) + (size_t)t * row_bytes + (size_t)Tq.h * D * sizeof(T);
#pragma unroll
                            for (int qq = 0; qq < 8; ++qq) stg16(orow + qq * 16, pack<T>(o + 8 * qq));
                        }
                        p.state.m[rh] = mm;
                        p.state.l[rh] = ll;
                    }
                    if (lane == 0) mbar_arrive(bar(bars, B_QEMPTY + 2 * w + (int)b));
                    __syncwarp();
                    continue;
                }
                const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
                for (int i = 0; i < 64; ++i) o[i] *= inv;
                if (cut) {
                    // tile cut by the query range / sequence end: plain stores of valid rows
                    if (xv) {
                        char *orow = reinterpret_cast<char *>(p.out) + (size_t)t * row_bytes + (size_t)Tq.h * D * sizeof(T);
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq) stg16(orow + qq * 16, pack<T>(o + 8 * qq));
                    }
                    if (lane == 0) mbar_arrive(bar(bars, B_QEMPTY + 2 * w + (int)b));
                    __syncwarp();
                    continue;
                }
                // full tile: stage this warp's 32 rows in the tile's Q buffer (all the tile's S
                // MMAs completed before the softmax finished) in the TMA layout and store them
                // with one 32-row box; the buffer goes back to the loader after the store read it
                const uint32_t sO = sbase + OFF_Q + (uint32_t)(2 * w + (int)b) * QBYTES;
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) {
                    const uint4 v = pack<T>(o + 8 * qq);
                    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sO + swz<D>(row, qq)), "r"(v.x),
                                 "r"(v.y), "r"(v.z), "r"(v.w)
                                 : "memory");
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    const int tok = (int)((int64_t)Tq.c + (int64_t)(Tq.a0 + 32 * q) * r - p.q_begin);
                    tma::store_3d(&tp.tmO, 0, Tq.h, tok, sO + (uint32_t)q * (32 * RB));
                    tma::store_commit();
                }
                __syncwarp();
                pend_rel = true;
                pend_w = w;
                pend_b = b;
            }
        }
        if (pend_rel) release();
        if (lane == 0) tma::store_wait_all(); // bulk stores complete before the CTA exits
        __syncwarp();
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REG_SMX));
        // ============================ softmax warpgroups ============================
        const int w = warp >> 2, q = warp & 3;
        const uint32_t tl = tmem + 256u * w + ((uint32_t)(q * 32) << 16); // this warp's TMEM lanes
        const float sl2 = p.scale_log2;
        constexpr float kTau = 8.f;
        const int32_t mi = (int32_t)m;
        uint32_t c = 0; // running chunk counter (matches the issuer's)
        uint32_t k = 0; // tiles of this warpgroup
        Cur C = cur_init(tp, it_begin);
        for (int32_t it = it_begin; it < it_end; ++it, cur_next(tp, C)) {
            const Tile Tt = tile_at(tp, C, w);
            if (!Tt.valid) continue;
            const int32_t xr0 = Tt.a0 + 32 * q, x = xr0 + lane;
            const uint32_t tO = tl + COL_O + (GA_WTC_PSEP ? 0u : (k & 1u) * D); // this tile's O accumulator
            // keys of this warp's rows: union [ulo, uhi], every row: [ilo, ihi]; this row: [klo, khi]
            const int32_t ulo = max(xr0 - mi, 0), uhi = min(xr0 + 31 + mi, Tt.Nc - 1);
            const int32_t ilo = max(xr0 + 31 - mi, 0), ihi = min(xr0 + mi, Tt.Nc - 1);
            const int32_t klo = max(x - mi, 0), khi = min(x + mi, Tt.Nc - 1);
            float m_run = -INFINITY, l_run = 0.f;
            const int32_t n = Tt.n;
            uint32_t ecnt = 0; // probe (edge_counter): this row's weighted pairs
            // the 32-column halves of chunk j this warp loads (no row of the warp reaches a
            // skipped one) and those every row reaches fully (warp-uniform)
            auto ldh = [&](int32_t j, int hh) { const int32_t b = (Tt.F + j) * KC + 32 * hh; return !(b > uhi || b + 31 < ulo); };
            // S(c) is loaded at the end of the previous chunk of the tile (its TMEM load overlaps
            // that chunk's P store, fence and arrival); the first chunk of a tile loads here
            float s[64];
#if GA_WTC_PRELOAD
            auto load_S = [&](uint32_t cc, int32_t jj) {
                mbar_wait(bar(bars, B_SFULL + 2 * w + (int)(cc & 1)), (cc >> 1) & 1);
                fence_after();
                const uint32_t tS = tl + COL_S + (cc & 1u) * KC;
                if (ldh(jj, 0)) tmem_ld32(tS, s);
                if (ldh(jj, 1)) tmem_ld32(tS + 32, s + 32);
            };
            load_S(c, 0);
#endif
            for (int32_t j = 0; j < n; ++j, ++c) {
                const int32_t kmin = (Tt.F + j) * KC;
                const int32_t h0 = kmin, h1 = kmin + 32;
                const bool ld0 = ldh(j, 0), ld1 = ldh(j, 1);
                const bool full0 = h0 >= ilo && h0 + 31 <= ihi, full1 = h1 >= ilo && h1 + 31 <= ihi;
                TRACE(10 + w);
                const uint32_t tS = tl + COL_S + (c & 1u) * KC; // S(c); P(c) is written over it
#if !GA_WTC_PRELOAD
                mbar_wait(bar(bars, B_SFULL + 2 * w + (int)(c & 1)), (c >> 1) & 1);
                fence_after();
                TRACE(12 + w);
                if (ld0) tmem_ld32(tS, s);
                if (ld1) tmem_ld32(tS + 32, s + 32);
#endif
                tmem_wait_ld();
                TRACE(24 + w);
                // masks: left edge inside the half iff the last lane's klo is past its start
                if (ld0 && !full0)
                    mask_half(s, klo - h0, khi - h0, max(xr0 + 31 - mi, 0) > h0, min(xr0 + mi, Tt.Nc - 1) < h0 + 31);
                if (ld1 && !full1)
                    mask_half(s + 32, klo - h1, khi - h1, max(xr0 + 31 - mi, 0) > h1, min(xr0 + mi, Tt.Nc - 1) < h1 + 31);
                if (PROBE && p.edge_counter) { // probe: pairs left unmasked (they get a weight) of a query row
#pragma unroll
                    for (int i = 0; i < 32; ++i) ecnt += (ld0 && s[i] != -INFINITY) + (ld1 && s[32 + i] != -INFINITY);
                }
                // chunk max (log2 domain) and lazy rescale: a row moves its reference max only
                // when the chunk's max exceeds it by more than kTau (weights stay <= 2^kTau); O
                // needs rescaling only for rows that already hold weight
                float lm = -INFINITY;
                if (ld0) lm = max32(s);
                if (ld1) lm = fmaxf(lm, max32(s + 32));
                const float lm2 = lm * sl2;
                const bool need = lm2 > m_run + kTau;
                // rows whose O and l must be scaled by a = 2^(m_run - lm2) < 2^-kTau (never 1);
                // the vote does not wait for an exponential (a MUFU op queued behind the other
                // warpgroup's would delay it by up to one chunk of exponentials)
                const bool resc = need && m_run != -INFINITY;
                float a = 1.f;
                if (__any_sync(0xffffffffu, resc)) { // (resc implies j > 0: m_run is -inf at a tile's start)
                    a = resc ? ex2(m_run - lm2) : 1.f;
                    // O stable: P V of the previous chunk completed
                    mbar_wait(bar(bars, B_OFULL + 2 * w + (int)((c - 1) & 1)), ((c - 1) >> 1) & 1);
                    fence_after();
#pragma unroll
                    for (int qq = 0; qq < D / 16; ++qq) { // 16 columns at a time (registers)
                        uint32_t ov[16];
                        tmem_ld16(tO + 16 * qq, ov);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * a);
                        tmem_st16(tO + 16 * qq, ov);
                    }
                    tmem_wait_st();
                }
                if (need) {
                    l_run *= a;
                    m_run = lm2;
                }
                const float negm = m_run == -INFINITY ? 0.f : -m_run;
                TRACE(26 + w);
#if GA_WTC_PSEP
                // P(c) into P buffer c & 1: P V(c - 2) read it and completed, since the commit of
                // S(c) (waited above) follows P V(c - 2) in the issuer's order
                const uint32_t tP = tl + COL_P + (c & 1u) * (KC / 2);
#else
                const uint32_t tP = tS;
#endif
                float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                 make_float2(0.f, 0.f)};
                uint32_t pk[16];
                if (ld0) {
                    if (full0) exps_half<T, GA_WTC_POLY>(s, sl2, negm, pk, acc);
                    else exps_half<T, 0>(s, sl2, negm, pk, acc);
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk[i] = 0u;
                }
                tmem_st16(tP, pk);
                if (ld1) {
                    if (full1) exps_half<T, GA_WTC_POLY>(s + 32, sl2, negm, pk, acc);
                    else exps_half<T, 0>(s + 32, sl2, negm, pk, acc);
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk[i] = 0u;
                }
                tmem_st16(tP + 16, pk);
                l_run += (acc[0].x + acc[1].x) + (acc[2].x + acc[3].x) + ((acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
                TRACE(28 + w);
#if GA_WTC_PRELOAD
                if (j + 1 < n) load_S(c + 1, j + 1); // (S(c + 1) never waits for P(c))
#endif
                tmem_wait_st();
                TRACE(30 + w);
                fence_before();
                mbar_arrive(bar(bars, B_PFULL + 2 * w + (int)(c & 1)));
                TRACE(14 + w);
            }
            if (PROBE && p.edge_counter) { // probe: query rows of the range only (others are not stored)
                const uint32_t wc = __reduce_add_sync(0xffffffffu, x >= Tt.a_lo && x < Tt.a_hi ? ecnt : 0u);
                if (lane == 0 && wc) atomicAdd(p.edge_counter, (unsigned long long)wc);
            }
            // row sum and reference max for the epilogue (its read of the previous use of
            // this buffer, tile k - 2, completed before it released that tile's O)
            TRACE(16 + w);
            if (k >= 2) mbar_wait(bar(bars, B_OFREE + 2 * w + (int)(k & 1)), ((k - 2) >> 1) & 1);
            TRACE(22 + w);
            const int row = 32 * q + lane;
            lmbuf[((w * 2 + (int)(k & 1)) * 2 + 0) * ROWS + row] = l_run;
            lmbuf[((w * 2 + (int)(k & 1)) * 2 + 1) * ROWS + row] = m_run;
            mbar_arrive(bar(bars, B_EPI + 2 * w + (int)(k & 1)));
            ++k;
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

static int sm_count()
{
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

// chunks spanned by a pair of tiles (the ring holds NSLOT)
static int64_t pair_span(int64_t m) { return floordiv(2 * ROWS - 1 + m, KC) - floordiv(-m, KC) + 1; }

template <typename T, bool PROBE> static ga_status launch_t(const TcParams &tp, int64_t grid, cudaStream_t s)
{
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(window_tc_kernel<T, PROBE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        if (e != cudaSuccess) return cuda_fail(e, "window_tc_kernel: set smem");
        configured = true;
    }
    window_tc_kernel<T, PROBE><<<(unsigned)grid, THREADS, SMEM_BYTES, s>>>(tp);
    GA_CHECK_LAUNCH("window_tc_kernel");
    return GA_OK;
}

} // namespace wtc

int64_t window_tc_tile_rows() { return wtc::ROWS; }

#ifdef GA_WTC_TRACE
extern "C" int ga_wtc_trace_read(unsigned long long *out, int n)
{
    if (n < wtc::TRACE_N) return -1;
    cudaMemcpyFromSymbol(out, wtc::g_trace, sizeof(unsigned long long) * wtc::TRACE_N);
    static unsigned long long z[wtc::TRACE_N];
    cudaMemcpyToSymbol(wtc::g_trace, z, sizeof(z));
    return wtc::TRACE_N;
}
#endif

bool window_tc_supported(const AttnParams &p, ga_dtype dt)
{
    if (p.mask.kind != K_WINDOW || (dt != GA_BF16 && dt != GA_F16) || p.d != 64) return false;
    const int64_t m = p.mask.m, r = p.mask.r;
    if (m < 64 || m > 128 || r > 4 || wtc::pair_span(m) > 8) return false; // 8 chunks per item (bitmasks)
    if (p.mask.L >= ((int64_t)1 << 31) || p.q_rows <= 0) return false; // TMA coordinates are int32
    // without peer memory the local K/V must hold every key the query range reaches
    if (p.k_peer == nullptr && !(p.kv_begin == 0 && p.kv_rows == p.mask.L)) {
        const int64_t reach = m * r; // farthest key token a query row reaches
        if (p.kv_begin > imax(0, p.q_begin - reach) || p.kv_begin + p.kv_rows < imin(p.mask.L, p.q_begin + p.q_rows + reach))
            return false;
    }
    return true;
}

ga_status launch_window_tc(const AttnParams &p, ga_dtype dt, cudaStream_t s)
{
    wtc::TcParams tp;
    tp.p = p;
    tp.m = p.mask.m;
    tp.r = p.mask.r;
    const int64_t L = p.mask.L, r = tp.r, q_end = p.q_begin + p.q_rows;
    int64_t pps = 0;
    for (int64_t c = 0; c < r && c < L; ++c) {
        const int64_t Nc = (L - c + r - 1) / r;
        const int64_t a_lo = p.q_begin > c ? (p.q_begin - c + r - 1) / r : 0;
        const int64_t a_hi = q_end > c ? imin((q_end - c + r - 1) / r, Nc) : 0;
        if (a_hi <= a_lo) continue;
        const int64_t tiles = (a_hi + wtc::ROWS - 1) / wtc::ROWS - a_lo / wtc::ROWS;
        pps = imax(pps, (tiles + 1) / 2);
    }
    tp.pps = pps;
    tp.items = pps * r * p.H;
    if (tp.items == 0) return GA_OK;
    if (!tma::encode_rows(&tp.tmQ, p.Q, p.q_rows, p.H, p.d, (int)r, 64) ||
        !tma::encode_rows(&tp.tmO, p.out, p.q_rows, p.H, p.d, (int)r, 32) ||
        !tma::encode_rows(&tp.tmK, p.K, p.kv_rows, p.H, p.d, (int)r, 64) ||
        !tma::encode_rows(&tp.tmV, p.V, p.kv_rows, p.H, p.d, (int)r, 64)) {
        set_error("tcgen05 window kernel: tensor-map encoding failed");
        return GA_ERR_UNSUPPORTED;
    }
    int64_t grid = imin(wtc::sm_count(), tp.items);
    // debug: fewer CTAs, so each walks a long run of items (sanitizer coverage of the cursor,
    // the ring reuse and the cross-item S prefetch at small shapes)
    if (const char *e = getenv("GA_WTC_GRID")) grid = imax(1, imin(grid, (int64_t)atoi(e)));
    if (p.edge_counter || p.tensor_counter)
        return dt == GA_BF16 ? wtc::launch_t<__nv_bfloat16, true>(tp, grid, s) : wtc::launch_t<__half, true>(tp, grid, s);
    return dt == GA_BF16 ? wtc::launch_t<__nv_bfloat16, false>(tp, grid, s) : wtc::launch_t<__half, false>(tp, grid, s);
}

} // namespace ga

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
//   softmax           each thread tcgen05.ld's its row of S; keys outside the row's band get
//                     weight exactly 0; online softmax in the exp2 domain (lazy rescale, 2^8);
//                     P (bf16/fp16 pairs) written back to TMEM with tcgen05.st.  A warp skips
//                     chunks its 32 rows do not reach (P = 0 without reading S) and masks only
//                     chunks its rows reach partially
//   O += P V_g        tcgen05.mma with A = P from TMEM, B = V_g (MN-major) from shared memory
//
// The tensor cores see whole 128 x 64 chunks (66% of the products valid at m = 127: 32,640
// band edges of 49,152 per tile); exponentials, sums and weights are computed only for the
// chunks a warp's rows reach, and a masked pair contributes exactly 0 — the result is the
// Algorithm 1 result over the band's edges, computed in O(nnz d) work.
//
// CTA organisation (persistent, one CTA per SM, 512 TMEM columns):
//   warps 0-3  softmax warpgroup A: even tiles of a tile pair   (TMEM cols   0..255)
//   warps 4-7  softmax warpgroup B: odd tiles                    (TMEM cols 256..511)
//   warp 8     loader: TMA boxes of the Q tiles (2 x 64 class rows, element stride r) and the
//              K/V chunks into an 8-slot ring (slot = g mod 8); peer rows (sharded runs) by
//              cp.async from the owner's memory
//   warp 9     MMA issuer (one elected lane)
// A CTA walks a contiguous run of tile pairs of one (class, head) stream: consecutive pairs
// share 4 of their 8 chunks, which stay resident (each K/V row is read from L2/HBM about once
// per run), and the two warpgroups alternate on the tensor and MUFU pipes.
#include "tc_common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace ga {
namespace wtc {
using namespace tc;
using namespace umma;

constexpr int ROWS = 128, KC = 64, NSLOT = 10, D = 64, RB = 2 * D;
#ifndef GA_WTC_DUAL
#define GA_WTC_DUAL 0
#endif
// MMA issuer warps: one per softmax warpgroup (GA_WTC_DUAL = 1), or one for both.  Measured
// (tools/r2_dual.sh, ms): cfg2 0.1256 / 0.1270 dual vs 0.1228 / 0.1219 single, cfg5 30.41 /
// 30.44 vs 30.56 / 30.84 — within noise of each other: the cross-warpgroup head-of-line
// blocking of one issuer is not what bounds the kernel.  Parity, synccheck and racecheck
// pass for both.
constexpr int NISSUE = GA_WTC_DUAL ? 2 : 1;
constexpr int THREADS = 32 * (9 + NISSUE); // 8 softmax warps + loader + MMA issuer(s)
constexpr uint32_t QBYTES = ROWS * RB;   // 16 KB
constexpr uint32_t CBYTES = KC * RB;     // 8 KB: one K or V chunk
constexpr uint32_t OFF_Q = 0;            // Q[wg][buf]: 4 x 16 KB
constexpr uint32_t OFF_KV = 4 * QBYTES;  // slot s: K at OFF_KV + 2 s CBYTES, V right after
constexpr uint32_t OFF_BAR = OFF_KV + NSLOT * 2 * CBYTES;
constexpr uint32_t SMEM_BYTES = 1024 + OFF_BAR + 64 * 8;

// mbarrier indices (8 bytes each from OFF_BAR)
#ifndef GA_WTC_NSB
#define GA_WTC_NSB 2
#endif
constexpr int NSB = GA_WTC_NSB; // S buffers per warpgroup (P is written over its S buffer)
constexpr int B_QFULL = 0, B_QEMPTY = 4, B_KVFULL = 8, B_KVEMPTY = 8 + NSLOT, B_SFULL = 8 + 2 * NSLOT,
              B_PFULL = B_SFULL + 2 * NSB, B_OFULL = B_PFULL + 2 * NSB;
constexpr int B_TMEM = B_OFULL + 4; // tcgen05.alloc writes the TMEM base here

#ifndef GA_WTC_SEPP
#define GA_WTC_SEPP 1
#endif
#if GA_WTC_SEPP
// TMEM columns of warpgroup w: S[NSB] at 256w + 64 b, P[2] (chunk c's 16-bit pairs in P[c & 1],
// 32 columns each), one O accumulator.  S_{c+NSB} reuses S_c's buffer as soon as the softmax
// has read it (P_c arrived), with no wait for any MMA to complete; the softmax writes P_c only
// after P V_{c-2} has read that P buffer.  One O suffices: a tile's epilogue reads O before the
// same threads release P of the next tile's first chunk, so the next tile's first P V (which
// overwrites O, accumulate = 0) is issued after those reads.
constexpr uint32_t COL_S = 0, COL_P = NSB * KC, COL_O = COL_P + 2 * (KC / 2);
static_assert(COL_O + D <= 256, "TMEM: 256 columns per warpgroup");
#else
// TMEM columns of warpgroup w: S[NSB] at 256w + 64 b (P of chunk c, 16-bit pairs, is written over
// the first 32 columns of its S buffer), O[2] (tile k accumulates in O[k & 1]) after them
constexpr uint32_t COL_S = 0, COL_O = NSB * KC;
static_assert(NSB * KC + 2 * D <= 256, "TMEM: 256 columns per warpgroup");
#endif

struct TcParams {
    CUtensorMap tmQ, tmK, tmV, tmO; // one head, element stride r, 64-row boxes
    AttnParams p;
    int64_t m, r;
    int64_t pps;   // tile pairs per (class, head) stream
    int64_t items; // streams x pps
};

__host__ __device__ inline int64_t floordiv(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Geometry of one work item (a pair of consecutive 128-row tiles of one stream); every role
// derives it independently from the item index, so all agree without communication.
struct Pair {
    int32_t stream, u, c, Nc, a_lo, a_hi;
    int h;
    int32_t a0[2];  // first class row of tile A / B
    bool valid[2];
    int32_t F[2], n[2]; // chunks [F, F + n) per tile
    int32_t lo, hi;     // union of the chunk ranges
    bool any;
};

__device__ __forceinline__ Pair pair_geo(const TcParams &tp, int32_t it)
{
    // 32-bit arithmetic throughout: L < 2^31 (window_tc_supported), so class rows, tiles and
    // item indices fit; 64-bit division would cost hundreds of instructions per item
    const AttnParams &p = tp.p;
    const uint32_t r = (uint32_t)tp.r, L = (uint32_t)p.mask.L, H = (uint32_t)p.H, pps = (uint32_t)tp.pps;
    const int32_t m = (int32_t)tp.m;
    Pair P;
    const uint32_t iu = (uint32_t)it, st = iu / pps;
    P.stream = st;
    P.u = iu - st * pps;
    const uint32_t c = st / H;
    P.c = c;
    P.h = (int)(st - c * H);
    const uint32_t Nc = c < L ? (L - c + r - 1) / r : 0;
    P.Nc = Nc;
    const uint32_t qb = (uint32_t)p.q_begin, qe = (uint32_t)(p.q_begin + p.q_rows);
    const uint32_t a_lo = qb > c ? (qb - c + r - 1) / r : 0;
    const uint32_t a_hi = qe > c ? min((qe - c + r - 1) / r, Nc) : 0;
    P.a_lo = a_lo;
    P.a_hi = a_hi;
    const int32_t t0 = (int32_t)(a_lo / ROWS + 2 * (uint32_t)P.u);
    const int32_t lastc = ((int32_t)Nc - 1) >> 6; // KC = 64
    P.lo = INT32_MAX;
    P.hi = -1;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
        const int32_t a0 = (t0 + w) * ROWS;
        P.a0[w] = a0;
        P.valid[w] = a_lo < a_hi && (uint32_t)a0 < a_hi;
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

__device__ __forceinline__ Tile tile_geo(const TcParams &tp, int32_t it, int w)
{
    const AttnParams &p = tp.p;
    const uint32_t r = (uint32_t)tp.r, L = (uint32_t)p.mask.L, H = (uint32_t)p.H, pps = (uint32_t)tp.pps;
    const int32_t m = (int32_t)tp.m;
    Tile T;
    const uint32_t iu = (uint32_t)it, st = iu / pps, u = iu - st * pps;
    const uint32_t c = st / H;
    T.c = (int32_t)c;
    T.h = (int32_t)(st - c * H);
    const uint32_t Nc = c < L ? (L - c + r - 1) / r : 0;
    const uint32_t qb = (uint32_t)p.q_begin, qe = (uint32_t)(p.q_begin + p.q_rows);
    const uint32_t a_lo = qb > c ? (qb - c + r - 1) / r : 0;
    const uint32_t a_hi = qe > c ? min((qe - c + r - 1) / r, Nc) : 0;
    T.Nc = (int32_t)Nc;
    T.a_lo = (int32_t)a_lo;
    T.a_hi = (int32_t)a_hi;
    T.a0 = (int32_t)((a_lo / ROWS + 2 * u + (uint32_t)w) * ROWS);
    T.valid = a_lo < a_hi && (uint32_t)T.a0 < a_hi;
    T.F = max((T.a0 - m) >> 6, 0);
    T.n = T.valid ? min((T.a0 + ROWS - 1 + m) >> 6, ((int32_t)Nc - 1) >> 6) - T.F + 1 : 0;
    return T;
}

__device__ __forceinline__ uint32_t bar(uint32_t base, int i) { return base + 8u * (uint32_t)i; }

#ifdef GA_WTC_TRACE
// debug timeline of CTA 0: (event << 48 | warp << 40 | (clock - t0)) per event
constexpr int TRACE_N = 16384;
__device__ unsigned long long g_trace[TRACE_N];
__device__ unsigned int g_trace_n;
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

template <typename T>
__global__ void __launch_bounds__(THREADS, 1) window_tc_kernel(const __grid_constant__ TcParams tp)
{
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    const uint32_t bars = sbase + OFF_BAR;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem_raw + (sbase - raw) + OFF_BAR + 8 * B_TMEM);
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
            mbar_init(bar(bars, B_QEMPTY + i), 4); // each warp's O store has read its rows
            mbar_init(bar(bars, B_OFULL + i), 1);
        }
        for (int i = 0; i < 2 * NSB; ++i) {
            mbar_init(bar(bars, B_SFULL + i), 1);
            mbar_init(bar(bars, B_PFULL + i), 128);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(bar(bars, B_KVFULL + s), 1);
            mbar_init(bar(bars, B_KVEMPTY + s), NISSUE); // every issuer releases every fill
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

    if (warp == 8) {
        // ============================ loader ============================
        // per slot: filled before (bit s of `used`), parity of the fill count (bit s of `par`);
        // bitmasks, not arrays (a dynamically indexed array would live in local memory)
        uint32_t used = 0, par = 0;
        int nq[2] = {0, 0};
        int32_t prev_stream = -1, prev_u = -1, prev_hi = -1;
        for (int32_t it = it_begin; it < it_end; ++it) {
            const Pair P = pair_geo(tp, it);
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
            }
            // K/V chunks not resident from the previous pair
            const bool cont = P.stream == prev_stream && P.u == prev_u + 1;
            for (int32_t g = P.lo; g <= P.hi; ++g) {
                if (cont && g <= prev_hi) continue;
                const int s = (int)((uint32_t)g % NSLOT);
                TRACE2(21, g);
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
    } else if (warp >= 9) {
        // ============================ MMA issuer(s) ============================
        // Warp-uniform control flow (the whole warp runs the schedule and the blocking waits;
        // one elected lane issues), so descriptors and counters live in uniform registers.
        // Per warpgroup w the schedule keeps S one chunk ahead of the softmax:
        //     S_w(0), S_w(1); for j: [P_w(j)] P V_w(j), S_w(j+2)
        // S_w(j+2) reuses S buffer j&1, which the softmax finished reading before P_w(j).  When
        // a warpgroup finishes its tile it starts the S MMAs of its next tile (chunks resident)
        // while it runs its epilogue.  With GA_WTC_DUAL each warpgroup has its own issuer warp
        // (warp 9 + w), so a warpgroup waiting for its softmax never holds up the other's MMAs
        // (one issuer serving both interleaves them chunk by chunk and waits in order).  Both
        // issuers walk the same items; every issuer arrives once on a slot's empty barrier per
        // fill (count NISSUE): after its last P V reading the chunk, or — for a chunk its tile
        // does not read — after it has observed the fill, so an arrival never lands in the
        // previous fill's phase.
        const bool mine0 = NISSUE == 1 || warp == 9, mine1 = NISSUE == 1 || warp == 10;
        auto mine = [&](int w) { return w == 0 ? mine0 : mine1; };
        const uint32_t idS = idesc<T>(ROWS, KC, false), idO = idesc<T>(ROWS, D, true);
        // smem descriptors: constant high part | (address >> 4); the operand tiles stay below
        // 256 KB so the 14-bit start field never carries
        const uint64_t dbase = sdesc_sw128(0);
        uint32_t seen = 0;      // parity of the fills waited for, bit per slot
        int nq[2] = {0, 0};     // Q tiles waited per warpgroup
        uint32_t cw[2] = {0, 0}; // running chunk counters per warpgroup (S/P/O buffer parity)
        int pre[2] = {0, 0};    // S MMAs of this item's tile already issued (end of the previous item)
        bool preq[2] = {false, false};
        int32_t prev_stream = -1, prev_u = -1, prev_lo = 0;
        uint32_t waited = 0; // fills this issuer observed, bit g - lo of the previous item
        Pair N = pair_geo(tp, it_begin);
        for (int32_t it = it_begin; it < it_end; ++it) {
            const Pair P = N;
            const bool has_next = it + 1 < it_end;
            if (has_next) N = pair_geo(tp, it + 1);
            if (!P.any) continue;
            const bool cont = P.stream == prev_stream && P.u == prev_u + 1;
            const bool next_cont = has_next && N.any && N.stream == P.stream && N.u == P.u + 1;
            const int32_t keep_from = next_cont ? N.lo : INT32_MAX;
            uint32_t readers = 0; // 4 bits per chunk g - lo: this issuer's P V MMAs still to come
            // chunks resident from the previous item whose fill this issuer already observed
            uint32_t ready = cont ? waited >> (P.lo - prev_lo) : 0u;
#pragma unroll
            for (int w = 0; w < 2; ++w)
                if (mine(w))
                    for (int32_t j = 0; j < P.n[w]; ++j) readers += 1u << (4 * (P.F[w] + j - P.lo));
            int qb[2] = {0, 0};
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                if (!mine(w) || !P.valid[w]) continue;
                if (preq[w]) {
                    qb[w] = (nq[w] - 1) & 1;
                } else {
                    qb[w] = nq[w] & 1;
                    mbar_wait(bar(bars, B_QFULL + 2 * w + qb[w]), (nq[w] >> 1) & 1);
                    ++nq[w];
                }
            }
            fence_after();
            auto chunk_ready = [&](int32_t g) {
                const int gi = (int)(g - P.lo);
                if ((ready >> gi) & 1u) return;
                const int sl = (int)((uint32_t)g % NSLOT);
                mbar_wait(bar(bars, B_KVFULL + sl), (seen >> sl) & 1u);
                seen ^= 1u << sl;
                ready |= 1u << gi;
                TRACE2(1, g);
                fence_after();
            };
            // release of a chunk released by this item that this issuer's tile does not read
            auto release_unread = [&](int32_t g) {
                chunk_ready(g);
                if (elect_one()) mma_commit(bar(bars, B_KVEMPTY + (int)((uint32_t)g % NSLOT)));
                __syncwarp();
            };
            // this issuer's chunk range [rf, re) (dual: its own tile's; single: the union)
            int32_t rf = P.lo, re = P.hi + 1;
            if (NISSUE == 2) {
                const int32_t f = mine0 ? P.F[0] : P.F[1], n = mine0 ? P.n[0] : P.n[1]; // (static indices)
                rf = n == 0 ? P.hi + 1 : f;
                re = n == 0 ? P.hi + 1 : f + n;
                for (int32_t g = P.lo; g < rf && g < keep_from; ++g) release_unread(g);
            }
            auto issue_S = [&](int w, uint32_t c, int32_t g, int qbuf) {
                const uint32_t aq = sbase + OFF_Q + (uint32_t)(2 * w + qbuf) * QBYTES;
                const uint32_t ak = sbase + OFF_KV + ((uint32_t)g % NSLOT) * 2 * CBYTES;
                const uint32_t sb = (uint32_t)(c % NSB);
                const uint32_t dS = tmem + 256u * w + COL_S + sb * KC;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        mma_ss(dS, dbase | ((aq + kk * 32) >> 4), dbase | ((ak + kk * 32) >> 4), idS, kk > 0);
                    mma_commit(bar(bars, B_SFULL + NSB * w + (int)sb));
                }
                __syncwarp();
                TRACE2(6 + w, g);
            };
            auto issue_PV = [&](int w, int32_t j) {
                const uint32_t c = cw[w] + (uint32_t)j;
                const int32_t g = P.F[w] + j;
                const uint32_t sb = (uint32_t)(c % NSB);
                mbar_wait(bar(bars, B_PFULL + NSB * w + (int)sb), (uint32_t)((c / NSB) & 1));
                TRACE2(3 + w, g);
                fence_after();
                const int gi = (int)(g - P.lo), sl = (int)((uint32_t)g % NSLOT);
                const uint32_t av = sbase + OFF_KV + (uint32_t)sl * 2 * CBYTES + CBYTES;
#if GA_WTC_SEPP
                const uint32_t tP = tmem + 256u * w + COL_P + (c & 1u) * (KC / 2);
                const uint32_t tOacc = tmem + 256u * w + COL_O;
#else
                const uint32_t tP = tmem + 256u * w + COL_S + sb * KC;
                const uint32_t tOacc = tmem + 256u * w + COL_O + (uint32_t)qb[w] * D;
#endif
                readers -= 1u << (4 * gi);
                // this issuer's last reader of the chunk: release its slot unless the next item
                // keeps it (commit tracks every MMA this thread issued)
                const bool release = ((readers >> (4 * gi)) & 15u) == 0 && g < keep_from;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < KC / 16; ++kk) // 16 keys per MMA: 8 P columns, 16 V rows
                        mma_ts(tOacc, tP + kk * 8, dbase | ((av + kk * 16 * RB) >> 4), idO,
                               (j > 0 || kk > 0));
                    mma_commit(bar(bars, B_OFULL + 2 * w + (int)(c & 1)));
                    if (release) mma_commit(bar(bars, B_KVEMPTY + sl));
                }
                __syncwarp();
            };
            // S of the first NSB chunks of each tile (unless issued early); S_w(j + NSB) reuses
            // the buffer of chunk j, free once P V_w(j) has completed (waited below)
#pragma unroll
            for (int w = 0; w < 2; ++w)
                if (mine(w))
                    for (int32_t j = pre[w]; j < NSB && j < P.n[w]; ++j) {
                        chunk_ready(P.F[w] + j);
                        issue_S(w, cw[w] + j, P.F[w] + j, qb[w]);
                    }
            int npre[2] = {0, 0};
            bool nqw[2] = {false, false};
            auto prefetch = [&](int w, bool block) { // next tile's first S MMAs (resident chunks)
                for (int32_t jn = 0; jn < NSB && jn < N.n[w]; ++jn) {
                    const int32_t g = N.F[w] + jn;
                    if (g > P.hi || !((ready >> (int)(g - P.lo)) & 1u)) break;
                    if (!nqw[w]) {
                        const uint32_t qf = bar(bars, B_QFULL + 2 * w + (nq[w] & 1));
                        const uint32_t ph = (nq[w] >> 1) & 1;
                        if (block) mbar_wait(qf, ph);
                        else if (!mbar_test(qf, ph)) return;
                        ++nq[w];
                        nqw[w] = true;
                        fence_after();
                    }
                    issue_S(w, cw[w] + P.n[w] + jn, g, (nq[w] - 1) & 1);
                    ++npre[w];
                }
            };
            const int32_t jmax = max(mine0 ? P.n[0] : 0, mine1 ? P.n[1] : 0);
            for (int32_t j = 0; j < jmax; ++j) {
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    if (!mine(w) || j >= P.n[w]) continue;
                    issue_PV(w, j);
                    if (j + NSB < P.n[w]) {
#if !defined(GA_WTC_NO_WAR_WAIT) && !GA_WTC_SEPP
                        // S_w(j + NSB) overwrites the TMEM columns P V_w(j) reads (P over S): wait
                        // for P V_w(j) to complete — issue order alone did not keep the A-operand
                        // reads ahead of a later MMA's accumulator writes in the LongNet kernel
                        // (tools/lnet_stress.py); costs ~1-2% here (tools/ab_war.sh)
                        { const uint32_t cc = cw[w] + j; mbar_wait(bar(bars, B_OFULL + 2 * w + (int)(cc & 1)), (uint32_t)((cc >> 1) & 1)); fence_after(); }
#endif
                        chunk_ready(P.F[w] + j + NSB);
                        issue_S(w, cw[w] + j + NSB, P.F[w] + j + NSB, qb[w]);
                    } else if (j == P.n[w] - 1 && next_cont && N.valid[w]) {
                        prefetch(w, false); // only if the next Q tile already landed
                    }
                }
            }
            if (NISSUE == 2)
                for (int32_t g = max(re, P.lo); g <= P.hi && g < keep_from; ++g) release_unread(g);
#pragma unroll
            for (int w = 0; w < 2; ++w)
                if (mine(w) && next_cont && N.valid[w] && npre[w] == 0) prefetch(w, true);
            cw[0] += P.n[0];
            cw[1] += P.n[1];
            pre[0] = npre[0];
            pre[1] = npre[1];
            preq[0] = nqw[0];
            preq[1] = nqw[1];
            prev_stream = P.stream;
            prev_u = P.u;
            prev_lo = P.lo;
            waited = ready;
        }
    } else {
        // ============================ softmax warpgroups ============================
        // A tile's epilogue (O from TMEM, normalise, store) is deferred to the first chunk of the
        // warpgroup's next tile: O is double-buffered in TMEM (tile k accumulates in O[k & 1]), so
        // the softmax never waits for the last P V of a tile.
        const int w = warp >> 2, q = warp & 3;
        const uint32_t tl = tmem + 256u * w + ((uint32_t)(q * 32) << 16); // this warp's TMEM lanes
        const float sl2 = p.scale_log2;
        constexpr float kTau = 8.f;
        uint32_t cnt = 0; // running chunk counter (matches the MMA issuer's cw[w])
        auto wait_O = [&](uint32_t c) {
            mbar_wait(bar(bars, B_OFULL + 2 * w + (int)(c & 1)), (c >> 1) & 1);
            fence_after();
        };
        uint32_t ntile = 0; // tiles of this warpgroup (Q / O staging buffer and O buffer = index & 1)
        // deferred epilogue of the previous tile
        bool pend_epi = false, pend_rel = false;
        int32_t p_it = 0; // previous tile's item (its geometry is recomputed: fewer live registers)
        float l_prev = 0.f, m_prev = -INFINITY;
        uint32_t cnt_prev = 0, tix_prev = 0;
        auto release = [&]() { // the previous tile's O store has read its Q buffer: hand it back
            if (lane == 0) {
                tma::store_wait_read();
                mbar_arrive(bar(bars, B_QEMPTY + 2 * w + (int)(tix_prev & 1)));
            }
            __syncwarp();
            pend_rel = false;
        };
        // carried-state epilogue (ga_opts.state): this row's (m, l, o~) in the
        // log2 domain, written or (+)-combined into the caller's fp32 buffers (m is the row's
        // softmax reference: its running max, or within 2^kTau of it after a lazy rescale —
        // any reference combines exactly); with p.out also the normalised row
        auto state_epilogue = [&](uint32_t tO, int32_t c, int32_t h, int32_t x, int32_t alo, int32_t ahi) {
            const bool valid = x >= alo && x < ahi;
            const int64_t t = (int64_t)c + (int64_t)x * r - p.q_begin; // local query row
            const size_t rh = valid ? (size_t)t * H + h : 0;
            float mm = m_prev, ll = l_prev, a = 1.f, b = 0.f;
            bool mix = false;
            if (valid && p.state_mode == GA_STATE_ACCUMULATE) {
                const float l2 = p.state.l[rh];
                if (l2 > 0.f) { // l == 0 marks an empty state (its m is ignored)
                    const float m2 = p.state.m[rh];
                    const float mn = ll > 0.f ? fmaxf(mm, m2) : m2;
                    a = ll > 0.f ? ex2(mm - mn) : 0.f;
                    b = ex2(m2 - mn);
                    ll = ll * a + l2 * b;
                    mm = mn;
                    mix = true;
                }
            }
            const float inv = ll > 0.f ? 1.f / ll : 0.f;
            float4 *so = reinterpret_cast<float4 *>(p.state.o + rh * D);
            char *orow = p.out ? reinterpret_cast<char *>(p.out) + (size_t)t * row_bytes + (size_t)h * D * sizeof(T)
                               : nullptr;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                float o[32];
                tmem_ld32(tO + 32 * half, o); // warp-collective: every lane
                tmem_wait_ld();
                if (!valid) continue;
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) {
                    float4 v = make_float4(o[4 * qq], o[4 * qq + 1], o[4 * qq + 2], o[4 * qq + 3]);
                    if (mix) {
                        const float4 u = so[8 * half + qq];
                        v.x = v.x * a + u.x * b;
                        v.y = v.y * a + u.y * b;
                        v.z = v.z * a + u.z * b;
                        v.w = v.w * a + u.w * b;
                    }
                    so[8 * half + qq] = v;
                    o[4 * qq] = v.x * inv;
                    o[4 * qq + 1] = v.y * inv;
                    o[4 * qq + 2] = v.z * inv;
                    o[4 * qq + 3] = v.w * inv;
                }
                if (orow) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) stg16(orow + (4 * half + qq) * 16, pack<T>(o + 8 * qq));
                }
            }
            if (valid) {
                p.state.m[rh] = mm;
                p.state.l[rh] = ll;
            }
        };
        auto epilogue = [&]() {
            pend_epi = false;
            // P V of the tile's last chunk completed.  The O barriers alternate per chunk and a
            // parity wait is exact only if the barrier's previous phase completed: P V(e-2)'s
            // predecessor P V(e-4) ran before S(e-1) (observed), and P V(e-2) completing implies
            // P V(e-3), the predecessor of P V(e-1)
            if (cnt_prev >= 2) wait_O(cnt_prev - 2);
            wait_O(cnt_prev - 1);
            TRACE2(18 + w, 0);
#if GA_WTC_SEPP
            const uint32_t tO = tl + COL_O;
#else
            const uint32_t tO = tl + COL_O + (tix_prev & 1) * D;
#endif
            const float inv = l_prev > 0.f ? 1.f / l_prev : 0.f;
            const Tile Tq = tile_geo(tp, p_it, w);
            const int32_t p_c = Tq.c, p_h = Tq.h, p_a0 = Tq.a0, p_alo = Tq.a_lo, p_ahi = Tq.a_hi;
            const int32_t xr0 = p_a0 + 32 * q, x = xr0 + lane;
            const bool cut = !(p_a0 >= p_alo && p_a0 + ROWS <= p_ahi);
            // full tile: stage this warp's 32 rows in the tile's Q buffer (the tile's S MMAs
            // completed) in the TMA layout and store them with one 32-row box, released to the
            // loader later; tile cut by the query range / sequence end: plain stores of valid rows
            if (p.state.m) { // carried state (ga_state): fp32 (m, l, o~) per row, plain stores
                state_epilogue(tO, p_c, p_h, x, p_alo, p_ahi);
                if (lane == 0) mbar_arrive(bar(bars, B_QEMPTY + 2 * w + (int)(tix_prev & 1)));
                __syncwarp();
                return;
            }
            const uint32_t sO = sbase + OFF_Q + (uint32_t)(2 * w + (tix_prev & 1)) * QBYTES;
            char *orow = nullptr;
            if (cut && x >= p_alo && x < p_ahi)
                orow = reinterpret_cast<char *>(p.out) + (size_t)((int64_t)p_c + (int64_t)x * r - p.q_begin) * row_bytes +
                       (size_t)p_h * D * sizeof(T);
#pragma unroll
            for (int half = 0; half < 2; ++half) { // 32 columns at a time (register pressure)
                float o[32];
                tmem_ld32(tO + 32 * half, o);
                tmem_wait_ld();
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    float r8[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) r8[e] = o[8 * qq + e] * inv;
                    const uint4 v = pack<T>(r8);
                    if (!cut)
                        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sO + swz<D>(32 * q + lane, 4 * half + qq)),
                                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                                     : "memory");
                    else if (orow)
                        stg16(orow + (4 * half + qq) * 16, v);
                }
            }
            if (cut) {
                if (lane == 0) mbar_arrive(bar(bars, B_QEMPTY + 2 * w + (int)(tix_prev & 1)));
                __syncwarp();
                return;
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                const int tok = (int)((int64_t)p_c + (int64_t)xr0 * r - p.q_begin);
                tma::store_3d(&tp.tmO, 0, p_h, tok, sO + (uint32_t)q * (32 * RB));
                tma::store_commit();
            }
            pend_rel = true;
        };
        const int32_t mi = (int32_t)m;
        for (int32_t it = it_begin; it < it_end; ++it) {
            const Tile Tt = tile_geo(tp, it, w);
            if (!Tt.valid) continue;
            const int32_t xr0 = Tt.a0 + 32 * q, x = xr0 + lane;
#if GA_WTC_SEPP
            const uint32_t tO = tl + COL_O; // this tile's O accumulator
#else
            const uint32_t tO = tl + COL_O + (ntile & 1) * D; // this tile's O accumulator
#endif
            // keys of this warp's rows: union [ulo, uhi], every row: [ilo, ihi]; this row: [klo, khi]
            const int32_t ulo = max(xr0 - mi, 0), uhi = min(xr0 + 31 + mi, Tt.Nc - 1);
            const int32_t ilo = max(xr0 + 31 - mi, 0), ihi = min(xr0 + mi, Tt.Nc - 1);
            const int32_t klo = max(x - mi, 0), khi = min(x + mi, Tt.Nc - 1);
            float m_run = -INFINITY, l_run = 0.f;
            const int32_t n = Tt.n;
            for (int32_t j = 0; j < n; ++j) {
                const uint32_t c = cnt + (uint32_t)j, sb = c % NSB, sph = (c / NSB) & 1;
                const int32_t kmin = (Tt.F + j) * KC;
                const uint32_t tS = tl + COL_S + sb * KC; // S of chunk c; P is written over it
                // S_c is waited for even when skipped: every phase of the S barriers is then
                // observed in order (a parity wait cannot tell phase k from phase k + 2)
                TRACE(10 + w);
                mbar_wait(bar(bars, B_SFULL + NSB * w + (int)sb), sph);
                fence_after();
                TRACE(12 + w);
#if GA_WTC_SEPP
                const uint32_t tPw = tl + COL_P + (c & 1u) * (KC / 2); // P_c (written after P V_{c-2} read it)
#else
                const uint32_t tPw = tS;
#endif
                if (kmin > uhi || kmin + KC - 1 < ulo) { // no row of this warp reaches the chunk
                    uint32_t z[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) z[i] = 0u;
#if GA_WTC_SEPP
                    if (c >= 2) wait_O(c - 2);
#endif
                    tmem_st32(tPw, z);
                    tmem_wait_st();
                    if (pend_epi) epilogue(); // see below
                    fence_before();
                    mbar_arrive(bar(bars, B_PFULL + NSB * w + (int)sb));
                } else {
                    float sv[KC];
                    tmem_ld32(tS, sv);
                    tmem_ld32(tS + 32, sv + 32);
                    tmem_wait_ld();
                    if (!(kmin >= ilo && kmin + KC - 1 <= ihi)) { // partial: keep only this row's band
                        const int il = max(klo - kmin, -1), ih = min(khi - kmin, KC);
                        if (__any_sync(0xffffffffu, il > 0)) { // left edge of the band inside the chunk
#pragma unroll
                            for (int i = 0; i < KC; ++i) sv[i] = i >= il ? sv[i] : -INFINITY;
                        }
                        if (__any_sync(0xffffffffu, ih < KC - 1)) { // right edge
#pragma unroll
                            for (int i = 0; i < KC; ++i) sv[i] = i <= ih ? sv[i] : -INFINITY;
                        }
                    }
                    uint32_t pk[KC / 2];
                    auto exps = [&]() -> float { // pk = P (input type); returns the row's chunk sum
                        const float m_use = m_run == -INFINITY ? 0.f : m_run;
                        float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}; // packed partial sums
#pragma unroll
                        for (int i = 0; i < KC / 2; ++i) {
                            float x0 = sv[2 * i], x1 = sv[2 * i + 1];
                            ffma2_sm(x0, x1, sl2, -m_use);
                            x0 = ex2(x0);
                            x1 = ex2(x1);
                            fadd2_acc(ls[i & 1], x0, x1);
                            pk[i] = pack2<T>(x0, x1);
                        }
                        return (ls[0].x + ls[1].x) + (ls[0].y + ls[1].y);
                    };
                    // fast path once every row of the warp holds a reference max: weights against
                    // it first; a rescale is needed iff some weight exceeds 2^kTau, which a chunk
                    // sum <= 2^kTau rules out (then the chunk max is never computed); otherwise the
                    // careful path repeats the chunk exactly as before (bit-identical results)
                    bool fast = false;
                    if (__all_sync(0xffffffffu, m_run != -INFINITY)) {
                        const float lsum = exps();
                        if (!__any_sync(0xffffffffu, !(lsum <= 256.f))) { // 2^kTau; NaN/inf -> careful
                            l_run += lsum;
                            fast = true;
                        }
                    }
                    if (!fast) {
                        float lmx[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) lmx[i] = sv[i];
#pragma unroll
                        for (int i = 8; i < KC; ++i) lmx[i & 7] = fmaxf(lmx[i & 7], sv[i]);
                        const float lm = fmaxf(fmaxf(fmaxf(lmx[0], lmx[1]), fmaxf(lmx[2], lmx[3])),
                                               fmaxf(fmaxf(lmx[4], lmx[5]), fmaxf(lmx[6], lmx[7])));
                        // lazy rescale: a row moves its reference max only when the chunk's max exceeds
                        // it by more than kTau (weights stay <= 2^kTau); O needs rescaling only for rows
                        // that already hold weight (a row with m = -inf has O = 0 and l = 0)
                        const float lm2 = lm * sl2;
                        const bool need = lm2 > m_run + kTau;
                        const float a = (need && m_run != -INFINITY) ? ex2(m_run - lm2) : 1.f;
                        if (__any_sync(0xffffffffu, a != 1.f) && j > 0) {
                            wait_O(c - 1); // O stable: P V of the previous chunk completed
                            float ov[32];
#pragma unroll
                            for (int qq = 0; qq < D / 32; ++qq) {
                                tmem_ld32(tO + 32 * qq, ov);
                                tmem_wait_ld();
                                uint32_t ob[32];
#pragma unroll
                                for (int i = 0; i < 32; ++i) ob[i] = __float_as_uint(ov[i] * a);
                                tmem_st32(tO + 32 * qq, ob);
                            }
                            tmem_wait_st();
                        }
                        if (need) {
                            l_run *= a;
                            m_run = lm2;
                        }
                        l_run += exps();
                    }
#if GA_WTC_SEPP
                    if (c >= 2) wait_O(c - 2);
#endif
                    tmem_st32(tPw, pk);
                    tmem_wait_st();
                    // the previous tile's epilogue with this tile's first chunk (its last P V has
                    // long completed), BEFORE P of this chunk is released: P V of this chunk could
                    // otherwise complete a second phase of the O barrier the epilogue waits on
                    if (pend_epi) epilogue();
                    fence_before();
                    mbar_arrive(bar(bars, B_PFULL + NSB * w + (int)sb));
                    TRACE(14 + w);
                }
                // the staging buffer goes back to the loader one chunk after the store
                if (pend_rel && j > 0) release();
            }
            if (pend_epi) epilogue(); // (n >= 1: not reached)
            if (pend_rel) release();  // one-chunk tile
            cnt += (uint32_t)n;
            pend_epi = true;
            p_it = it;
            l_prev = l_run;
            m_prev = m_run;
            cnt_prev = cnt;
            tix_prev = ntile;
            ++ntile;
#ifndef GA_WTC_DEFER_EPILOGUE
            // epilogue right away (measured faster than deferring it into the next tile, which
            // needs more registers); O is still double-buffered, so the next tile's first P V
            // never waits for these TMEM reads
            epilogue();
#endif
        }
        if (pend_epi) epilogue();
        if (pend_rel) release();
        if (lane == 0) tma::store_wait_all(); // bulk stores complete before the CTA exits
        __syncwarp();
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

template <typename T> static ga_status launch_t(const TcParams &tp, int64_t grid, cudaStream_t s)
{
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(window_tc_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        if (e != cudaSuccess) return cuda_fail(e, "window_tc_kernel: set smem");
        configured = true;
    }
    window_tc_kernel<T><<<(unsigned)grid, THREADS, SMEM_BYTES, s>>>(tp);
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
    const int64_t grid = imin(wtc::sm_count(), tp.items);
    return dt == GA_BF16 ? wtc::launch_t<__nv_bfloat16>(tp, grid, s) : wtc::launch_t<__half>(tp, grid, s);
}

} // namespace ga

// longnet_umma.cu — tcgen05 (5th-gen tensor core, TMEM accumulators) kernel for the large
// LongNet groups.
//
// Same decomposition as longnet_tc.cu: the rows of G(sigma0, s) share one neighbour set, so
// (128 group rows) x (their concatenated key pieces) is a fully dense block.  Here a CTA of
// 128 threads owns 128 rows — thread t = row t = TMEM lane t — and streams the keys in
// chunks of KC = 64 through a 4-stage cp.async ring:
//
//   S  = Q K_c^T      tcgen05.mma.cta_group::1.kind::f16, M=128 N=64 K=16 x d/16, A and B
//                     from 128B-swizzled shared memory, fp32 accumulator in TMEM
//   softmax           each thread tcgen05.ld's its row of S, online softmax in the exp2
//                     domain (lazy rescale, threshold 2^8), writes P (bf16/fp16 pairs) back
//                     into TMEM with tcgen05.st
//   O += P V_c        tcgen05.mma with A = P from TMEM, B = V_c (MN-major) from shared
//                     memory, fp32 accumulator in TMEM
//
// One elected thread issues the MMAs; completion is signalled through tcgen05.commit ->
// mbarrier.  Two CTAs per SM overlap one CTA's softmax with the other's MMAs.
//
// Small groups (high valuation s: few rows, many keys) would waste most of a 128-row tile,
// so the rows with s >= h0 ("high rows") are processed BLOCK-wise instead: the LongNet
// mask restricted to them is the disjoint union, over levels t and level-t segments sigma,
// of the dense blocks (SURVEY §8(a) strided-block decomposition)
//     B(t, sigma) = { i in sigma : alpha^max(t+1,h0) | i } x { j in sigma : nu(j) = t }     t < K
//     A(t, sigma) = { i in sigma : min(nu(i),K) = t }      x { j in sigma : alpha^t | j }   t >= h0
// (a high row with s = min(nu(i),K) meets B at levels 0..s-1 and A at level s: exactly its
// pieces of masks.cuh).  Every block has >= 128 rows at the cfg4 shape, so it runs on the
// same tcgen05 pipeline; each block writes a partial (m, l, o~) per row and level, and
// longnet_merge_kernel combines a row's s + 1 partials with the associative (+) (P:374's
// split-and-merge, as in csr_heavy.cu).
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "tc_common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace ga {
namespace lnet_umma {
using namespace tc;
using namespace umma;

// warps 0-3: softmax (thread = row = TMEM lane); warp 4: loader (cp.async ring); warp 5: MMA
#ifndef GA_LNET_STAGES
#define GA_LNET_STAGES 4 // K/V ring depth (5 fits twice per SM too; measured equal: the ring is fed at the L2 rate)
#endif
constexpr int ROWS = 128, SM_THREADS = 128, THREADS = SM_THREADS + 64, KC = 64, STAGES = GA_LNET_STAGES;
constexpr int MAX_ITEMS = 64, MAX_PIECES = 64;

constexpr int MAX_BLK = 128; // block-mode work entries (level, kind)
// of every GA_LNET_POLY_DEN exp2 pairs, GA_LNET_POLY run as a degree-3 polynomial on the FMA
// pipe (ex2_poly2, relative error ~1e-4, below P's bf16 rounding).  Round 1 (issue-bound
// softmax): 1/4 -> 27.15 ms vs 26.07.  Now MUFU is ~68% busy in the group kernel: 1/16 ->
// 18.71-18.82 ms vs 18.88-18.90 (same box), 1/8 equal, 1/4 19.6.
#ifndef GA_LNET_POLY_DEN
#define GA_LNET_POLY_DEN 16
#endif
#ifndef GA_LNET_POLY
#define GA_LNET_POLY 1
#endif
constexpr int MAX_LAT = 24;  // TMA lattice levels (alpha = 2): 2^23 row pitch

struct UParams {
    AttnParams p;
    // group mode: items (s, tile) over the level-0 segments seg0 .. seg0 + n_seg
    int64_t seg0, n_seg;
    int32_t n_items;
    int16_t item_s[MAX_ITEMS];
    int16_t item_tile[MAX_ITEMS];
    // block mode (blocked = 1): entry e covers CTAs [blk_start[e], blk_start[e+1]) =
    // blk_nseg[e] level-t segments from blk_seg0[e] x blk_tiles[e] row tiles x H
    int32_t blocked, n_blk, h0;
    int16_t blk_t[MAX_BLK], blk_kind[MAX_BLK]; // kind 0 = B (nu(j) = t keys), 1 = A (last piece)
    int32_t blk_tiles[MAX_BLK];
    int64_t blk_seg0[MAX_BLK], blk_nseg[MAX_BLK], blk_start[MAX_BLK + 1];
    // partial slots: level t of high row i -> slot_off[t] + i / alpha^max(t,h0) - slot_first[t]
    int64_t slot_off[MAX_PIECES], slot_first[MAX_PIECES];
    float *partials; // [slots][H][D + 4]: m, l, (2 pad), o~ — 16-byte aligned o~
    // TMA lattice maps (alpha = 2, local K/V with kv_begin = 0; n_lat = 0: cp.async loader):
    // level t, kind 0 = odd multiples of 2^t (pieces t < s, nu(j) = t), kind 1 = all multiples
    // (the last piece); 64-row boxes of one head
    int32_t n_lat;
    CUtensorMap tmK[2 * MAX_LAT], tmV[2 * MAX_LAT];
};

template <int D> __host__ __device__ constexpr uint32_t smem_bytes()
{
    return 1024 /* alignment slack */ + ROWS * 2 * D /* Q */ + STAGES * 2 * KC * 2 * D /* K,V */ + ROWS * 8 /* rows */ +
           256 /* mbarriers, tmem base */;
}

// TMEM columns: S ring of NSB buffers at b KC (P_c, 16-bit pairs, is written over the first
// KC/2 columns of its S buffer), O at NSB KC: S0 S1 S2 | O = 256 columns at d = 64.  Three S
// buffers let S_{c+3} be issued as soon as P V_c is (P_c read), so S_{c+1} is ready well
// before the softmax of chunk c ends.
#ifndef GA_LNET_SEPP
#define GA_LNET_SEPP 1 // P in its own TMEM columns (S0 S1 | P0 P1 | O) instead of over its S buffer
#endif
#if GA_LNET_SEPP
constexpr int NSB = 2, NPB = 2;
constexpr uint32_t COL_S = 0, COL_P = NSB * KC, COL_O = COL_P + NPB * KC / 2;
#else
constexpr int NSB = 3;
constexpr uint32_t COL_S = 0, COL_O = NSB * KC;
#endif

#ifdef GA_LNET_TRACE
// debug timeline of one group-mode CTA (blockIdx.x == LNET_TRACE_CTA): per warp, lane 0
// records (val << 56 | event << 48 | warp << 40 | clock - t0)
constexpr int LT_N = 8192, LT_PER = LT_N / 8, LNET_TRACE_CTA = 2853; // item 3 (an s = 0 tile) of segment 150 at w0 = 2048, H = 1
__device__ unsigned long long g_ltrace[LT_N];
#define LTRACE(ev, val) do { if (lt_on && (threadIdx.x & 31) == 0 && lt_cnt < LT_PER) { \
    g_ltrace[(threadIdx.x >> 5) * LT_PER + lt_cnt++] = ((unsigned long long)((val) & 0xff) << 56) | \
        ((unsigned long long)(ev) << 48) | ((unsigned long long)(threadIdx.x >> 5) << 40) | \
        (unsigned long long)((clock64() - lt_t0) & 0xffffffffffull); } } while (0)
#else
#define LTRACE(ev, val)
#endif

template <typename T, int D>
__global__ void __launch_bounds__(THREADS, 2) longnet_umma_kernel(const __grid_constant__ UParams up)
{
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned base for the 128B-swizzled operand tiles
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    unsigned char *sgen = smem_raw + (sbase - raw);
    constexpr int RB = 2 * D;
    const uint32_t sQ = sbase;
    const uint32_t sK0 = sQ + ROWS * RB;                  // stage st: sK0 + st*KC*RB
    const uint32_t sV0 = sK0 + STAGES * KC * RB;
    int64_t *rows = reinterpret_cast<int64_t *>(sgen + ROWS * RB + 2 * STAGES * KC * RB);
    uint64_t *mbars = reinterpret_cast<uint64_t *>(rows + ROWS);
    uint32_t *tmem_base_smem = reinterpret_cast<uint32_t *>(mbars + 9 + 2 * STAGES);
    const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(mbars);
    // S_c complete (tcgen05.commit) for buffer b = c % NSB: mbS0 + 8 b; P V_c complete: mbO0 +
    // 8 (c & 1); P_c written by the 128 softmax threads: mbP0 + 8 b (addresses, not arrays:
    // dynamically indexed arrays would live in local memory)
    const uint32_t mbS0 = mb0, mbO0 = mb0 + 8 * NSB, mbP0 = mbO0 + 16;
    const uint32_t mbQ = mb0 + 64;                // Q tile landed (32 loader lanes)
    const uint32_t mbFull0 = mb0 + 72;            // stage st landed: mbFull0 + 8 st (32 lanes)
    const uint32_t mbEmpty0 = mbFull0 + 8 * STAGES; // stage st consumed (P V commit)

    const AttnParams &p = up.p;
    const DevMask &M = p.mask;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int H = p.H;
#ifdef GA_LNET_TRACE
    const bool lt_on = !up.blocked && blockIdx.x == LNET_TRACE_CTA;
    const long long lt_t0 = clock64();
    int lt_cnt = 0;
    LTRACE(0, 0);
#endif

    // ---- work item -> (segment [S0, S1), row progression, key pieces)
    int64_t S0, S1, seg_len, row_step; // rows: candidates (f0 + q) * row_step in [lo, hi)
    int s, tile, h, np, t_first;      // pieces t_first .. t_first + np - 1 of the rows
    bool skip_res;                    // drop the candidates whose q has residue rx mod alpha
    if (!up.blocked) {
        // 32-bit divisions (blockIdx.x < 2^31): a 64-bit one costs ~100 instructions per thread
        const uint32_t IH = (uint32_t)up.n_items * (uint32_t)H, bx = blockIdx.x;
        const uint32_t segl = bx / IH;
        const uint32_t rem = bx - segl * IH;
        const uint32_t item = rem / (uint32_t)H;
        h = (int)(rem - item * (uint32_t)H);
        s = up.item_s[item];
        tile = up.item_tile[item];
        seg_len = M.w0;
        S0 = (up.seg0 + segl) * M.w0;
        row_step = 1;
        for (int t = 0; t < s; ++t) row_step *= M.alpha;
        skip_res = s != (int)M.K;
        np = s + 1;
        t_first = 0;
    } else {
        int e = 0;
        while (e + 1 < up.n_blk && up.blk_start[e + 1] <= (int64_t)blockIdx.x) ++e;
        const uint32_t rel = (uint32_t)((int64_t)blockIdx.x - up.blk_start[e]);
        const uint32_t TH = (uint32_t)up.blk_tiles[e] * (uint32_t)H;
        const uint32_t segl = rel / TH, rem = rel - segl * TH;
        tile = (int)(rem / (uint32_t)H);
        h = (int)(rem - (uint32_t)tile * (uint32_t)H);
        const int t = up.blk_t[e];
        seg_len = M.w0;
        for (int u = 0; u < t; ++u) seg_len *= M.alpha;
        S0 = (up.blk_seg0[e] + segl) * seg_len;
        const int ex = up.blk_kind[e] == 0 ? (t + 1 > up.h0 ? t + 1 : up.h0) : t;
        row_step = 1;
        for (int u = 0; u < ex; ++u) row_step *= M.alpha;
        skip_res = up.blk_kind[e] == 1 && t != (int)M.K; // A rows: valuation exactly t
        s = t;
        np = 1;
        t_first = t;
    }
    S1 = imin(M.L, S0 + seg_len);
    const int64_t q_end = p.q_begin + p.q_rows;

    // ---- rows (closed form, see longnet_tc.cu): candidates (f0 + q) * row_step in [lo, hi);
    // skip_res drops q with residue rx mod alpha (those have a higher valuation)
    const int64_t step = row_step;
    const int64_t lo = imax(S0, p.q_begin), hi = imin(S1, q_end);
    const bool a2 = M.alpha == 2; // the common alpha: step = 2^ls, divisions by shifts
    const int ls = a2 ? __ffsll((unsigned long long)step) - 1 : 0;
    const int64_t f0 = a2 ? (lo + step - 1) >> ls : (lo + step - 1) / step;
    const int64_t nq = lo < hi && f0 * step < hi ? (a2 ? (hi - 1) >> ls : (hi - 1) / step) - f0 + 1 : 0;
    const int64_t rx = a2 ? (2 - (f0 & 1)) & 1 : (M.alpha - f0 % M.alpha) % M.alpha;
    const int64_t count = !skip_res ? nq : nq - (nq > rx ? (a2 ? (nq - 1 - rx) >> 1 : (nq - 1 - rx) / M.alpha) + 1 : 0);
    const int nrows = (int)imin(ROWS, count - (int64_t)tile * ROWS);
    if (nrows <= 0) return;
    if (tid < nrows) {
        const int64_t r = (int64_t)tile * ROWS + tid;
        int64_t q = r;
        if (skip_res) {
            if (a2) { // a1 = 1: idx = 0
                q = r * 2 + (0 < rx ? 0 : 1);
            } else {
                const int64_t a1 = M.alpha - 1, idx = r % a1;
                q = (r / a1) * M.alpha + (idx < rx ? idx : idx + 1);
            }
        }
        rows[tid] = (f0 + q) * step;
    }
    // ---- TMEM (warp 0) and mbarriers (thread 0)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(tmem_base_smem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int b = 0; b < NSB; ++b) {
            mbar_init(mbS0 + 8 * b, 1);
            mbar_init(mbP0 + 8 * b, SM_THREADS);
        }
        for (int b = 0; b < 2; ++b) mbar_init(mbO0 + 8 * b, 1);
        mbar_init(mbQ, SM_THREADS); // every softmax thread loads its own Q row
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(mbFull0 + 8 * st, 32);
            mbar_init(mbEmpty0 + 8 * st, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_base_smem;

    __shared__ Piece spiece[MAX_PIECES];
    __shared__ int pstart[MAX_PIECES + 1];
    if (tid < np) spiece[tid] = get_piece(M, rows[0], t_first + tid);
    __syncthreads();
    if (tid == 0) {
        pstart[0] = 0;
        for (int t = 0; t < np; ++t) pstart[t + 1] = pstart[t] + (int)spiece[t].count;
    }
    __syncthreads();
    const int nkeys = pstart[np];
    const int nblk = nkeys / 16;  // the tensor cores take whole 16-key blocks; a ragged
    const int ragged = nkeys - nblk * 16; // tail (general w0) is finished on CUDA cores
    const int nchunks = (nblk * 16 + KC - 1) / KC;
    if (warp < 4) {
        // Q: thread t loads row t (8 x 16 bytes; pad rows zeroed: they join the rescale votes) —
        // 128 threads issue it at once instead of the loader warp lane by lane (~3k cycles)
        const char *qrow = tid < nrows ? reinterpret_cast<const char *>(p.Q) + (size_t)h * D * sizeof(T) +
                                             (size_t)(rows[tid] - p.q_begin) * ((size_t)H * D * sizeof(T))
                                       : nullptr;
#pragma unroll
        for (int cc = 0; cc < RB / 16; ++cc) {
            if (qrow) cp_async16(sQ + swz<D>(tid, cc), qrow + cc * 16);
            else sts_zero16(sQ + swz<D>(tid, cc));
        }
        fence_proxy_async();
        cp_async_mbar_arrive(mbQ);
    }

    const size_t row_bytes = (size_t)H * D * sizeof(T);
    const char *Qg = reinterpret_cast<const char *>(p.Q) + (size_t)h * D * sizeof(T);
    const size_t hoff = (size_t)h * D * sizeof(T);
    const uint32_t idS = idesc<T>(ROWS, KC, false), idO = idesc<T>(ROWS, D, true);

    if (warp == 4) {
        // =================== loader warp: Q tile, then the K/V ring ===================
        const int lane = tid & 31;
        // chunk c -> stage c % STAGES.  Lane l resolves the token rows of keys l and l + 32
        // (piece cursor + piece_at + kv_row, once per key); the copies then go 8 lanes per
        // 128-byte row, 4 rows per instruction (coalesced), the row addresses passed by shuffle.
        // Keys past the last whole 16-key block are zeroed (masked).
        static_assert(RB / 16 == 8 && KC == 64, "8 lanes per 128-byte row, 2 keys per lane");
        const int cc = lane & 7;
        const char *kloc = reinterpret_cast<const char *>(p.K) + hoff + cc * 16;
        const ptrdiff_t vdelta = reinterpret_cast<const char *>(p.V) - reinterpret_cast<const char *>(p.K);
        int cur_t = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int st = c % STAGES;
            if (c >= STAGES) mbar_wait(mbEmpty0 + 8 * st, ((c / STAGES) - 1) & 1);
            LTRACE(20, c);
            // whole chunk inside one piece of an alpha = 2 mask: the keys are KC consecutive
            // rows of a token lattice -> one TMA box for K and one for V (warp-uniform test)
            int lt = -1;
            int64_t u0 = 0;
            if (up.n_lat > 0 && (c + 1) * KC <= nblk * 16) {
                const int k0 = c * KC;
                while (cur_t + 1 < np && pstart[cur_t + 1] <= k0) ++cur_t;
                if (k0 + KC <= pstart[cur_t + 1]) {
                    const Piece &P = spiece[cur_t];
                    const int64_t j0 = piece_at(P, k0 - pstart[cur_t]);
                    const int lev = __ffsll((unsigned long long)P.step) - 1; // step = 2^lev
                    // the lattice maps cover the local K/V rows [kv_begin, kv_begin + kv_rows)
                    // (sharded runs: this rank's shard; a chunk reaching other ranks' rows
                    // takes the cp.async path below)
                    const int64_t jl = j0 - p.kv_begin;
                    const int64_t jlast = jl + (int64_t)(KC - 1) * (P.mode == P_SKIPMUL ? 2 * P.step : P.step);
                    if (lev < up.n_lat && jl >= 0 && jlast < p.kv_rows) {
                        // (step = 2^lev: shifts, not 64-bit divisions, on the loader's path)
                        if (P.mode == P_SKIPMUL) { lt = 2 * lev; u0 = ((jl >> lev) - 1) >> 1; }
                        else { lt = 2 * lev + 1; u0 = jl >> lev; }
                    }
                }
            }
            if (lt >= 0) {
                if (lane == 0) {
                    tma::expect_tx(mbFull0 + 8 * st, 2 * KC * RB);
                    tma::load_3d(sK0 + st * KC * RB, &up.tmK[lt], 0, h, (int)u0, mbFull0 + 8 * st);
                    tma::load_3d(sV0 + st * KC * RB, &up.tmV[lt], 0, h, (int)u0, mbFull0 + 8 * st);
                } else {
                    mbar_arrive(mbFull0 + 8 * st);
                }
                continue;
            }
            if (p.k_peer == nullptr && p.kv_rows < INT32_MAX) { // local K/V: pass the row index (one shuffle)
                int jr[2];
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int k = c * KC + lane + 32 * half;
                    jr[half] = -1;
                    if (k < nblk * 16) {
                        while (cur_t + 1 < np && pstart[cur_t + 1] <= k) ++cur_t;
                        jr[half] = (int)(piece_at(spiece[cur_t], k - pstart[cur_t]) - p.kv_begin);
                    }
                }
#pragma unroll
                for (int it = 0; it < KC / 4; ++it) {
                    const int kl = 4 * it + (lane >> 3); // half = it >= 8 (warp-uniform)
                    const int j = __shfl_sync(0xffffffffu, jr[it >= 8], kl & 31);
                    const uint32_t so = st * KC * RB + swz<D>(kl, cc);
                    if (j >= 0) {
                        const char *kr = kloc + (int64_t)j * (int64_t)row_bytes;
                        cp_async16(sK0 + so, kr);
                        cp_async16(sV0 + so, kr + vdelta);
                    } else {
                        sts_zero16(sK0 + so);
                        sts_zero16(sV0 + so);
                    }
                }
            } else { // sharded: rows may live in a peer's buffer (kv_row), pass both pointers
                const char *kr2[2], *vr2[2];
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int k = c * KC + lane + 32 * half;
                    kr2[half] = vr2[half] = nullptr;
                    if (k < nblk * 16) {
                        while (cur_t + 1 < np && pstart[cur_t + 1] <= k) ++cur_t;
                        kv_row(p, piece_at(spiece[cur_t], k - pstart[cur_t]), row_bytes, kr2[half], vr2[half]);
                    }
                }
#pragma unroll
                for (int it = 0; it < KC / 4; ++it) {
                    const int kl = 4 * it + (lane >> 3); // half = it >= 8 (warp-uniform)
                    const int src = kl & 31;
                    const char *kr = reinterpret_cast<const char *>(
                        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(kr2[it >= 8]), src));
                    const char *vr = reinterpret_cast<const char *>(
                        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(vr2[it >= 8]), src));
                    if (kr != nullptr) {
                        cp_async16(sK0 + st * KC * RB + swz<D>(kl, cc), kr + hoff + cc * 16);
                        cp_async16(sV0 + st * KC * RB + swz<D>(kl, cc), vr + hoff + cc * 16);
                    } else {
                        sts_zero16(sK0 + st * KC * RB + swz<D>(kl, cc));
                        sts_zero16(sV0 + st * KC * RB + swz<D>(kl, cc));
                    }
                }
            }
            fence_proxy_async();
            cp_async_mbar_arrive(mbFull0 + 8 * st);
        }
        cp_async_wait<0>();
    } else if (warp == 5) {
        // =================== MMA warp: S_c = Q K_c^T, then O += P_{c-1} V_{c-1} ===================
        const int lane = tid & 31;
        auto issue_PV = [&](int c) { // after P_c arrived (written over S buffer c % NSB)
            mbar_wait(mbP0 + 8 * (c % NSB), (c / NSB) & 1);
            LTRACE(3, c);
            if (lane == 0) {
                fence_after();
                const uint32_t bv = sV0 + (c % STAGES) * KC * RB;
#if GA_LNET_SEPP
                const uint32_t tp = tmem + COL_P + (c % NPB) * (KC / 2);
#else
                const uint32_t tp = tmem + COL_S + (c % NSB) * KC;
#endif
#pragma unroll
                for (int kk = 0; kk < KC / 16; ++kk) // 16 keys per MMA: 8 P columns, 16 V rows
                    mma_ts(tmem + COL_O, tp + kk * 8, sdesc_sw128(bv + kk * 16 * RB), idO, (c > 0 || kk > 0));
                mma_commit(mbO0 + 8 * (c & 1));
                // S_c and P V_c have read the stage — signalled only when the loader refills it
                // (an arrive nobody waits for could land after the CTA exited; synccheck)
                if (c + STAGES < nchunks) mma_commit(mbEmpty0 + 8 * (c % STAGES));
            }
            __syncwarp();
        };
        // S_c into buffer c % NSB once stage c landed; the buffer's previous tenant P_{c-NSB}
        // was read by P V_{c-NSB}, issued before (tcgen05 ops of one thread run in order)
        auto issue_S = [&](int c) {
            mbar_wait(mbFull0 + 8 * (c % STAGES), (c / STAGES) & 1);
            LTRACE(1, c);
            if (lane == 0) {
                fence_after();
                const uint32_t bk = sK0 + (c % STAGES) * KC * RB;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) // K = 16 per MMA: +32 B inside the swizzle atom
                    mma_ss(tmem + COL_S + (c % NSB) * KC, sdesc_sw128(sQ + kk * 32), sdesc_sw128(bk + kk * 32), idS,
                           kk > 0);
                mma_commit(mbS0 + 8 * (c % NSB));
            }
            __syncwarp();
        };
        if (nchunks > 0) mbar_wait(mbQ, 0);
        for (int c = 0; c < nchunks && c < NSB; ++c) issue_S(c);
#if GA_LNET_SEPP
        // S_{c+2} goes into S_c's buffer, free once the softmax has read it (P_c arrived: waited
        // in issue_PV); P lives in its own columns, so no MMA completion gates the S issue
        for (int c = 0; c < nchunks; ++c) {
            issue_PV(c);
            if (c + NSB < nchunks) issue_S(c + NSB);
        }
#else
        static_assert(NSB == 3, "S_{c+2} reuses the buffer of P_{c-1}");
        for (int c = 0; c < nchunks; ++c) {
            issue_PV(c);
            if (c >= 1 && c + 2 >= nchunks) {
                // tail: no S left to issue, but every phase of the two-phase P V barrier is
                // still observed before the barrier's next arrival (synccheck-clean)
                mbar_wait(mbO0 + 8 * ((c - 1) & 1), ((c - 1) >> 1) & 1);
            } else if (c >= 1) {
                // S_{c+2} overwrites the TMEM columns P V_{c-1} read (P_{c-1}): wait for P V_{c-1}
                // to complete first — issue order alone does not order an MMA's TMEM A-operand
                // reads before a later MMA's accumulator writes (measured: sporadic corrupted
                // 32-lane quarters without this wait).  Waiting for the PREVIOUS P V (issued an
                // iteration ago, normally complete) keeps the MMA warp off the P V latency
                // (tools/lnet_trace.py).  P V_{c+1} is not issued yet, so the two-phase mbO ring
                // cannot alias here.
                mbar_wait(mbO0 + 8 * ((c - 1) & 1), ((c - 1) >> 1) & 1);
                LTRACE(7, c);
                issue_S(c + 2);
            }
        }
#endif
    }

    // =================== softmax warps: thread = row = TMEM lane ===================
    const uint32_t tlane = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = p.scale_log2;
    constexpr float kTau = 8.f;
    float m_run = -INFINITY, l_run = 0.f;
    auto wait_O = [&](int c) { // P V_c complete
        mbar_wait(mbO0 + 8 * (c & 1), (c >> 1) & 1);
        fence_after();
    };
    if (warp < 4) {
        for (int c = 0; c < nchunks; ++c) {
            // S_c
            LTRACE(10, c);
            mbar_wait(mbS0 + 8 * (c % NSB), (c / NSB) & 1);
            LTRACE(12, c);
            fence_after();
            float sv[KC];
            tmem_ld32(tlane + COL_S + (c % NSB) * KC, sv);
            tmem_ld32(tlane + COL_S + (c % NSB) * KC + 32, sv + 32);
            tmem_wait_ld();
            const int valid = nblk * 16 - c * KC; // keys of this chunk (< KC only in the last one)
            if (valid < KC) {
#pragma unroll
                for (int i = 0; i < KC; ++i) sv[i] = i < valid ? sv[i] : -INFINITY;
            }
            // P_c over S_c (this thread has read its row of S_c)
            uint32_t pk[KC / 2];
            auto exps = [&]() -> float { // pk = P_c (input type), returns the row's chunk sum
                float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}; // packed partial sums
#pragma unroll
                for (int i = 0; i < KC / 2; ++i) {
                    float x0 = sv[2 * i], x1 = sv[2 * i + 1];
                    ffma2_sm(x0, x1, sl2, -m_run);
                    if ((i % GA_LNET_POLY_DEN) < GA_LNET_POLY) { // part of the exponentials on the FMA pipe
                        ex2_poly2(x0, x1);
                    } else {
                        x0 = ex2(x0);
                        x1 = ex2(x1);
                    }
                    fadd2_acc(ls[i & 1], x0, x1);
                    pk[i] = pack2<T>(x0, x1);
                }
                return (ls[0].x + ls[1].x) + (ls[0].y + ls[1].y);
            };
            // Fast path (c > 0, reference max set): exponentials against the current reference
            // first; the lazy rescale is needed iff some weight exceeds 2^kTau, which a chunk
            // sum <= 2^kTau rules out — then the chunk max is never computed.  Otherwise the
            // careful path below (max, vote, rescale, exponentials again) gives exactly the
            // result it always gave, so both paths are bit-identical to it.
            bool fast = false;
            if (c > 0) {
                const float lsum = exps();
                if (!__any_sync(0xffffffffu, !(lsum <= 256.f))) { // 2^kTau; NaN/inf -> careful
                    l_run += lsum;
                    fast = true;
                }
            }
            if (!fast) {
                float lmx[8]; // 8 independent max chains
#pragma unroll
                for (int j = 0; j < 8; ++j) lmx[j] = sv[j];
#pragma unroll
                for (int i = 8; i < KC; ++i) lmx[i & 7] = fmaxf(lmx[i & 7], sv[i]);
                const float lm = fmaxf(fmaxf(fmaxf(lmx[0], lmx[1]), fmaxf(lmx[2], lmx[3])),
                                       fmaxf(fmaxf(lmx[4], lmx[5]), fmaxf(lmx[6], lmx[7])));
                // lazy rescale, voted per warp (each warp owns its 32 TMEM lanes of O); O is
                // stable once P V_{c-1} completed (P V_c is not issued before our P_c arrives)
                const bool need = lm * sl2 > m_run + kTau;
                if (__any_sync(0xffffffffu, need)) {
                    if (c > 0) wait_O(c - 1);
                    const float mn = fmaxf(m_run, lm * sl2);
                    const float a = ex2(m_run - mn);
                    if (__any_sync(0xffffffffu, c > 0 && a != 1.f)) { // tcgen05.ld/st: warp-uniform
                        float ov[32];
#pragma unroll
                        for (int q = 0; q < D / 32; ++q) {
                            tmem_ld32(tlane + COL_O + 32 * q, ov);
                            tmem_wait_ld();
                            uint32_t ob[32];
#pragma unroll
                            for (int i = 0; i < 32; ++i) ob[i] = __float_as_uint(ov[i] * a);
                            tmem_st32(tlane + COL_O + 32 * q, ob);
                        }
                        tmem_wait_st();
                    }
                    l_run *= a;
                    m_run = mn;
                }
                l_run += exps();
            }
#if GA_LNET_SEPP
            // P buffer c % 2 is free: P V_{c-2} completed, since the MMA warp committed S_c (waited
            // above) after issuing P V_{c-2} and a commit tracks every prior MMA of the thread
            // (the same argument keeps the parity waits on mbO below exact)
            tmem_st32(tlane + COL_P + (c % NPB) * (KC / 2), pk);
#else
            tmem_st32(tlane + COL_S + (c % NSB) * KC, pk);
#endif
            tmem_wait_st();
            fence_before();
            mbar_arrive(mbP0 + 8 * (c % NSB));
            LTRACE(14, c);
        }
    }
    // ---- O row from TMEM (+ ragged tail on CUDA cores), normalise, store
    const bool row_ok = warp < 4 && tid < nrows;
    float o[D];
    if (warp < 4 && nchunks > 0) {
#if GA_LNET_SEPP
        if (nchunks >= 2) wait_O(nchunks - 2); // every P V phase observed (synccheck-clean)
#endif
        wait_O(nchunks - 1);
#pragma unroll
        for (int q = 0; q < D / 32; ++q) tmem_ld32(tlane + COL_O + 32 * q, o + 32 * q);
        tmem_wait_ld();
    } else {
#pragma unroll
        for (int e = 0; e < D; ++e) o[e] = 0.f;
    }
    if (ragged > 0 && row_ok) { // < 16 keys every row sees: plain fp32 updates from global
        const char *qrow = Qg + (size_t)(rows[tid] - p.q_begin) * row_bytes;
        float qf[D];
#pragma unroll
        for (int q = 0; q < D / 8; ++q) unpack<T>(ldg16(qrow + q * 16), qf + 8 * q);
        for (int t = 0; t < ragged; ++t) {
            const int k = nblk * 16 + t;
            int pt = 0;
            while (pt + 1 < np && pstart[pt + 1] <= k) ++pt;
            const char *kr, *vr;
            kv_row(p, piece_at(spiece[pt], k - pstart[pt]), row_bytes, kr, vr);
            kr += hoff;
            vr += hoff;
            float sdot = 0.f, kf[8];
#pragma unroll
            for (int q = 0; q < D / 8; ++q) {
                unpack<T>(ldg16(kr + q * 16), kf);
#pragma unroll
                for (int e = 0; e < 8; ++e) sdot = fmaf(qf[8 * q + e], kf[e], sdot);
            }
            const float sc = sdot * sl2;
            if (sc > m_run) {
                const float a = ex2(m_run - sc);
                l_run *= a;
#pragma unroll
                for (int e = 0; e < D; ++e) o[e] *= a;
                m_run = sc;
            }
            const float pr = ex2(sc - m_run);
            l_run += pr;
#pragma unroll
            for (int q = 0; q < D / 8; ++q) {
                unpack<T>(ldg16(vr + q * 16), kf);
#pragma unroll
                for (int e = 0; e < 8; ++e) o[8 * q + e] = fmaf(pr, kf[e], o[8 * q + e]);
            }
        }
    }
    if (row_ok && up.blocked) { // partial state of (row, level s) for the merge kernel
        const int ex = s > up.h0 ? s : up.h0; // row / alpha^max(s, h0)
        int64_t q;
        if (M.alpha == 2) {
            q = rows[tid] >> ex;
        } else {
            int64_t stp = 1;
            for (int u = 0; u < ex; ++u) stp *= M.alpha;
            q = rows[tid] / stp;
        }
        const int64_t slot = up.slot_off[s] + q - up.slot_first[s];
        float *dst = up.partials + ((size_t)slot * H + h) * (D + 4);
        *reinterpret_cast<float4 *>(dst) = make_float4(m_run, l_run, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < D / 4; ++q)
            *reinterpret_cast<float4 *>(dst + 4 + 4 * q) = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    } else if (row_ok) {
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        char *Og = reinterpret_cast<char *>(p.out) + (size_t)h * D * sizeof(T) + (size_t)(rows[tid] - p.q_begin) * row_bytes;
#pragma unroll
        for (int q = 0; q < D / 8; ++q) {
            float r8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) r8[e] = o[8 * q + e] * inv;
            stg16(Og + q * 16, pack<T>(r8));
        }
    }
    LTRACE(99, 0);
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
    }
}

// One warp per (high row, head): combine the row's partials of levels 0..s with the
// associative (m, l, o~) (+) and store o~ / l (empty -> 0).
template <typename T, int D>
__global__ void __launch_bounds__(256) longnet_merge_kernel(const UParams up, int64_t first, int64_t n_high,
                                                            int64_t step_h0)
{
    const AttnParams &p = up.p;
    const DevMask &M = p.mask;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int H = p.H;
    if (gw >= n_high * H) return;
    const int64_t r = H == 1 ? gw : gw / H;
    const int h = (int)(gw - r * H);
    const int64_t i = (first + r) * step_h0;
    int s = 0; // min(nu(i), K), nu(0) = K
    const bool pow2 = (M.alpha & (M.alpha - 1)) == 0; // alpha = 2^la: valuations and slots by shifts
    const int la = pow2 ? __ffsll((unsigned long long)M.alpha) - 1 : 0;
    if (i == 0) s = (int)M.K;
    else if (pow2) s = (int)imin((int64_t)((__ffsll((unsigned long long)i) - 1) / la), M.K);
    else for (int64_t x = i; s < (int)M.K && x % M.alpha == 0; x /= M.alpha) ++s;
    constexpr int PER = D / 32;
    // lane t < s+1 fetches level t's (m, l) and its partial's address; one warp max and one
    // sum replace the sequential (+) chain, and the o~ loads of all levels are independent
    // (the exact (+) of a7 with the common reference max: o = sum_t 2^(m_t - M) o_t)
    const float *src = nullptr;
    float mt = -INFINITY, lt = 0.f;
    if (lane <= s) {
        const int ex = lane > up.h0 ? lane : up.h0; // alpha^max(t, h0)
        int64_t q;
        if (pow2) {
            q = i >> (ex * la);
        } else {
            int64_t stp = 1;
            for (int u = 0; u < ex; ++u) stp *= M.alpha;
            q = i / stp;
        }
        src = up.partials + ((size_t)(up.slot_off[lane] + q - up.slot_first[lane]) * H + h) * (D + 4);
        mt = src[0];
        lt = src[1];
    }
    float mx = mt;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float bt = (mt == -INFINITY) ? 0.f : ex2(mt - mx);
    float l = bt * lt;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    float o[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) o[e] = 0.f;
    const unsigned long long sp = reinterpret_cast<unsigned long long>(src);
#pragma unroll 4
    for (int t = 0; t <= s; ++t) {
        const float b = __shfl_sync(0xffffffffu, bt, t);
        const float *st = reinterpret_cast<const float *>(__shfl_sync(0xffffffffu, sp, t));
#pragma unroll
        for (int e = 0; e < PER; ++e) o[e] = fmaf(st[4 + lane + 32 * e], b, o[e]);
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T *Op = reinterpret_cast<T *>(p.out) + ((size_t)(i - p.q_begin) * H + h) * D;
#pragma unroll
    for (int e = 0; e < PER; ++e) Op[lane + 32 * e] = (T)(o[e] * inv);
}

template <typename T, int D> static ga_status launch_t(const UParams &up, int64_t blocks, cudaStream_t s)
{
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(longnet_umma_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem_bytes<D>());
        if (e != cudaSuccess) return cuda_fail(e, "longnet_umma_kernel: set smem");
        configured = true;
    }
    if (blocks == 0) return GA_OK;
    if (blocks > (int64_t)INT32_MAX) { set_error("LongNet tcgen05 grid too large"); return GA_ERR_UNSUPPORTED; }
    longnet_umma_kernel<T, D><<<(unsigned)blocks, THREADS, smem_bytes<D>(), s>>>(up);
    GA_CHECK_LAUNCH("longnet_umma_kernel");
    return GA_OK;
}

static int64_t ipow(int64_t a, int e)
{
    int64_t r = 1;
    while (e-- > 0) r *= a;
    return r;
}

// multiples of q in [a, b): first index ceil(a/q) and count
static void multiples(int64_t a, int64_t b, int64_t q, int64_t &first, int64_t &n)
{
    first = (a + q - 1) / q;
    n = b > a && first * q < b ? (b - 1) / q - first + 1 : 0;
}

// Block-mode plan for the high rows (s >= h0) of the query range: work entries and the
// partial-slot layout.  Returns the number of partial slots.
static int64_t plan_blocks(const AttnParams &p, int h0, UParams &up, int64_t &blocks)
{
    const DevMask &M = p.mask;
    const int K = (int)M.K;
    const int64_t qb = p.q_begin, qe = p.q_begin + p.q_rows;
    int64_t slots = 0;
    for (int t = 0; t <= K; ++t) {
        int64_t f, n;
        multiples(qb, qe, ipow(M.alpha, t > h0 ? t : h0), f, n);
        up.slot_off[t] = slots;
        up.slot_first[t] = f;
        slots += n;
    }
    up.blocked = 1;
    up.h0 = h0;
    int e = 0;
    blocks = 0;
    for (int t = 0; t <= K; ++t) {
        const int64_t W = M.w0 * ipow(M.alpha, t);
        const int64_t seg_lo = qb / W, seg_hi = (qe + W - 1) / W;
        for (int kind = 0; kind < 2; ++kind) {
            if (kind == 0 && t >= K) continue; // B: t < K
            if (kind == 1 && t < h0) continue; // A: levels of the high rows' last piece
            const int ex = kind == 0 ? (t + 1 > h0 ? t + 1 : h0) : t;
            const int64_t qs = ipow(M.alpha, ex);
            // most rows per level-t segment: multiples of alpha^ex in W tokens; A rows (kind 1,
            // t < K) have valuation exactly t, which for whole segments with alpha^(t+1) | W is
            // exactly W/alpha^t - W/alpha^(t+1) (no empty tiles)
            const bool whole = M.L % W == 0 && qb % W == 0 && qe % W == 0;
            const int64_t rows_max = (kind == 1 && t < K && whole && W % (qs * M.alpha) == 0)
                                         ? W / qs - W / (qs * M.alpha)
                                         : (W + qs - 1) / qs;
            if (e >= MAX_BLK) return -1;
            up.blk_t[e] = (int16_t)t;
            up.blk_kind[e] = (int16_t)kind;
            up.blk_tiles[e] = (int32_t)((rows_max + ROWS - 1) / ROWS);
            up.blk_seg0[e] = seg_lo;
            up.blk_nseg[e] = seg_hi - seg_lo;
            up.blk_start[e] = blocks;
            blocks += (int64_t)up.blk_tiles[e] * up.blk_nseg[e] * p.H;
            ++e;
        }
    }
    up.n_blk = e;
    up.blk_start[e] = blocks;
    return slots;
}

} // namespace lnet_umma

size_t longnet_umma_workspace(const AttnParams &p, int h0)
{
    lnet_umma::UParams up{};
    int64_t blocks = 0;
    const int64_t slots = lnet_umma::plan_blocks(p, h0, up, blocks);
    return slots < 0 ? 0 : (size_t)slots * p.H * (p.d + 4) * sizeof(float) + 256;
}

// Launch the tcgen05 kernel on the groups s = 0..s_max (those that fill 128-row tiles);
// with `partials` (workspace of longnet_umma_workspace bytes) the rows with s > s_max run
// block-wise on tcgen05 too and are merged; otherwise the caller runs them elsewhere.
#ifdef GA_LNET_TRACE
extern "C" int ga_lnet_trace_read(unsigned long long *out, int n)
{
    if (n < lnet_umma::LT_N) return -1;
    cudaMemcpyFromSymbol(out, lnet_umma::g_ltrace, sizeof(unsigned long long) * lnet_umma::LT_N);
    static unsigned long long z[lnet_umma::LT_N];
    cudaMemcpyToSymbol(lnet_umma::g_ltrace, z, sizeof(z));
    return lnet_umma::LT_N;
}
#endif

namespace lnet_umma {
// TMA lattice maps for alpha = 2 with local K/V starting at token 0: level t, odd multiples of
// 2^t (kind 0) and all multiples (kind 1).  Encoding ~4(K+1) maps is host work, so the set of
// the last (K, V, shape) is cached.
static void set_lattice(UParams &up, const AttnParams &p)
{
    up.n_lat = 0;
    const DevMask &M = p.mask;
    if (M.alpha != 2 || p.d != 64 || getenv("GA_LNET_CPASYNC")) return;
    // level t needs the local rows to start on the lattice: kv_begin a multiple of 2^(t+1)
    // (0 on one GPU; a shard boundary of a sharded run)
    int lat_max = MAX_LAT;
    if (p.kv_begin != 0) {
        lat_max = 0;
        while (lat_max < MAX_LAT && p.kv_begin % ((int64_t)2 << lat_max) == 0) ++lat_max;
    }
    struct Cache {
        const void *K, *V;
        int64_t rows;
        int H, n, lmax;
        CUtensorMap k[2 * MAX_LAT], v[2 * MAX_LAT];
    };
    static Cache c{};
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    int levels = (int)(M.K + 1 < MAX_LAT ? M.K + 1 : MAX_LAT);
    if (levels > lat_max) levels = lat_max;
    if (levels <= 0) return;
    if (!(c.K == p.K && c.V == p.V && c.rows == p.kv_rows && c.H == p.H && c.lmax == levels)) {
        c.n = 0;
        const size_t rb = (size_t)p.H * p.d * 2;
        for (int t = 0; t < levels; ++t) {
            const int64_t stp = (int64_t)1 << t;
            const int64_t n_all = (p.kv_rows + stp - 1) >> t, n_odd = n_all / 2;
            const char *Kc = reinterpret_cast<const char *>(p.K), *Vc = reinterpret_cast<const char *>(p.V);
            const bool ok = n_odd > 0 &&
                            tma::encode_lattice(&c.k[2 * t], Kc + stp * rb, n_odd, p.H, p.d, 2 * stp, KC) &&
                            tma::encode_lattice(&c.v[2 * t], Vc + stp * rb, n_odd, p.H, p.d, 2 * stp, KC) &&
                            tma::encode_lattice(&c.k[2 * t + 1], Kc, n_all, p.H, p.d, stp, KC) &&
                            tma::encode_lattice(&c.v[2 * t + 1], Vc, n_all, p.H, p.d, stp, KC);
            if (!ok) break;
            c.n = t + 1;
        }
        c.K = p.K;
        c.V = p.V;
        c.rows = p.kv_rows;
        c.H = p.H;
        c.lmax = levels;
        if (c.n != levels) c.n = 0; // all levels or none
    }
    up.n_lat = c.n;
    for (int i = 0; i < 2 * c.n; ++i) {
        up.tmK[i] = c.k[i];
        up.tmV[i] = c.v[i];
    }
}
} // namespace lnet_umma

ga_status launch_longnet_umma(const AttnParams &p, ga_dtype dt, int64_t seg0, int64_t n_seg, int s_max,
                              float *partials, cudaStream_t s)
{
    if (!(p.d == 64 && (dt == GA_BF16 || dt == GA_F16))) {
        set_error("LongNet tcgen05 kernel: unsupported d/dtype");
        return GA_ERR_UNSUPPORTED;
    }
    auto launch = [&](const lnet_umma::UParams &up, int64_t blocks) {
        return dt == GA_BF16 ? lnet_umma::launch_t<__nv_bfloat16, 64>(up, blocks, s)
                             : lnet_umma::launch_t<__half, 64>(up, blocks, s);
    };
    const DevMask &M = p.mask;
    if (s_max >= 0) { // group mode
        lnet_umma::UParams up{};
        up.p = p;
        lnet_umma::set_lattice(up, p);
        up.seg0 = seg0;
        up.n_seg = n_seg;
        int n = 0;
        int64_t stp = 1;
        for (int t = 0; t <= s_max; ++t) {
            // most rows with min(nu(i), K) == t in a w0 segment: multiples of a^t (at most
            // ceil(w0/a^t)) minus those of a^(t+1) (at least floor(w0/a^(t+1))) for t < K;
            // +1 covers a shorter range (last segment, shard cut), whose ceil can round up once
            // exact when every segment is whole and alpha^(t+1) | w0 (then no tile is empty)
            const bool whole = M.L % M.w0 == 0 && p.q_begin % M.w0 == 0 && (p.q_begin + p.q_rows) % M.w0 == 0;
            const int64_t cnt = (whole && t < (int)M.K && M.w0 % (stp * M.alpha) == 0)
                                    ? M.w0 / stp - M.w0 / (stp * M.alpha)
                                    : (M.w0 + stp - 1) / stp - (t < (int)M.K ? M.w0 / (stp * M.alpha) : 0) + 1;
            const int64_t tiles = (cnt + lnet_umma::ROWS - 1) / lnet_umma::ROWS;
            for (int64_t k = 0; k < tiles; ++k) {
                if (n >= lnet_umma::MAX_ITEMS) { set_error("LongNet tcgen05: too many items"); return GA_ERR_UNSUPPORTED; }
                up.item_s[n] = (int16_t)t;
                up.item_tile[n] = (int16_t)k;
                ++n;
            }
            stp *= M.alpha;
        }
        up.n_items = n;
        ga_status st = launch(up, (int64_t)n * n_seg * p.H);
        if (st != GA_OK) return st;
    }
    if (!partials || s_max >= (int)M.K) return GA_OK;
    // block mode for the high rows + merge
    lnet_umma::UParams ub{};
    ub.p = p;
    lnet_umma::set_lattice(ub, p);
    ub.partials = partials;
    int64_t blocks = 0;
    if (lnet_umma::plan_blocks(p, s_max + 1, ub, blocks) < 0) { set_error("LongNet: too many levels"); return GA_ERR_UNSUPPORTED; }
    ga_status st = launch(ub, blocks);
    if (st != GA_OK) return st;
    int64_t first, n_high;
    const int64_t step_h0 = lnet_umma::ipow(M.alpha, s_max + 1);
    lnet_umma::multiples(p.q_begin, p.q_begin + p.q_rows, step_h0, first, n_high);
    const int64_t warps = n_high * p.H;
    if (warps == 0) return GA_OK;
    const int64_t mblocks = (warps + 7) / 8;
    if (dt == GA_BF16)
        lnet_umma::longnet_merge_kernel<__nv_bfloat16, 64><<<(unsigned)mblocks, 256, 0, s>>>(ub, first, n_high, step_h0);
    else
        lnet_umma::longnet_merge_kernel<__half, 64><<<(unsigned)mblocks, 256, 0, s>>>(ub, first, n_high, step_h0);
    GA_CHECK_LAUNCH("longnet_merge_kernel");
    return GA_OK;
}

} // namespace ga

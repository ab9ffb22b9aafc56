// masks.cuh — neighbour enumeration Get_Neighbors(G, i, P_a) (Algorithm 1,
// PAPER.md:256, :271) for every mask family, as O(1) index arithmetic per neighbour.
//
// N(i) is delivered as a short list of "pieces"; each piece is an index progression the
// kernel walks with lane-group strides, so no neighbour list is ever materialised:
//   AFFINE   j = base + k*step                          (window, block-dilated, LongNet top level)
//   SKIPMUL  j = base + step*u(k), u(k) = k-th positive integer that is not a multiple of
//            alpha, i.e. u = (k/(alpha-1))*alpha + k%(alpha-1) + 1  (LongNet lower levels)
//   CSR      j = col_idx[base + k]
//
// Families (readings R1-R3, R11 in DESIGN.md):
//   WINDOW(w,r)  one AFFINE piece: j = i - lo*r + k*r, lo = min(i/r, m), hi = min((L-1-i)/r, m),
//                m = (w-1)/r, count = lo+hi+1.  (|i-j| < w and r | |i-j|)
//   BLOCK_DILATED(seg,r) one AFFINE piece over the segment's multiples of r, or none when
//                (i mod seg) mod r != 0.
//   LONGNET(w0,alpha) s+1 disjoint pieces with s = min(nu_alpha(i), K) (nu(0) = K):
//                for t < s the level-t segment's members whose valuation is exactly t
//                (SKIPMUL, step alpha^t); for t = s all multiples of alpha^s in the level-s
//                segment (AFFINE).  This is the disjoint decomposition of the union of
//                BlockDilated(w0 alpha^k, alpha^k) levels: (i,j) is an edge iff
//                floor(i/w_t) == floor(j/w_t) with t = min(nu(i), nu(j), K).
//   CSR          one CSR piece.
//
// Compiled as CUDA (__device__) and as plain C++ (tests/enum_host.cpp builds it with g++
// to check the enumerator against the oracle on the CPU).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GA_HD __host__ __device__ __forceinline__
#else
#define GA_HD inline
#endif

namespace ga {

enum MaskKind { K_CSR = 0, K_WINDOW = 1, K_LONGNET = 2, K_BIGBIRD = 3, K_BLOCK_DILATED = 4 };
enum PieceMode { P_AFFINE = 0, P_SKIPMUL = 1, P_CSR = 2 };

struct DevMask {
    int32_t kind;
    int32_t parts;        // BigBird components: bit 0 window, 1 global minus window, 2 random (0 = all);
                          // LongNet: GA_LONGNET_MULTISET = every level's block, duplicates kept
    int64_t L;
    const int64_t *row_ptr;
    const int32_t *col_idx;
    int64_t nnz;          // CSR edge count
    int64_t w, r, m;      // window: m = (w-1)/r
    int64_t w0, alpha, K; // LongNet: K = max{k: w0 alpha^k <= L}
    int64_t seg;          // block dilated
    const int64_t *gidx;  // BigBird globals (device) or nullptr = evenly spaced
    int64_t ng, nrand;
    uint64_t seed;
};

struct Piece {
    int64_t base, step, count;
    int32_t mode;
    int32_t alpha; // SKIPMUL: u ranges over the integers with u mod alpha != rexcl
    int32_t rexcl;
    int32_t pad;
    const int32_t *cols;
};

GA_HD int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
GA_HD int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

// alpha-adic valuation capped at K; nu(0) = K.
// trailing zero bits of x != 0 (the 2-adic valuation)
GA_HD int ctz64(int64_t x)
{
#if defined(__CUDA_ARCH__)
    return __ffsll((long long)x) - 1;
#else
    return __builtin_ctzll((unsigned long long)x);
#endif
}

GA_HD int64_t valuation(int64_t x, int64_t alpha, int64_t K)
{
    if (x == 0) return K;
    if (alpha == 2) return imin((int64_t)ctz64(x), K); // the common alpha: no 64-bit divisions
    int64_t v = 0;
    while (v < K && x % alpha == 0) { x /= alpha; ++v; }
    return v;
}

GA_HD int64_t ipow(int64_t a, int64_t e)
{
    int64_t r = 1;
    for (int64_t t = 0; t < e; ++t) r *= a;
    return r;
}

GA_HD int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// LongNet variants (DevMask.parts bits): 1 = multiset mixture (reading R11b), 2 = per-head
// offsets (reading R11c): head h keeps, at level t, the positions congruent
// to h modulo alpha^t instead of 0 — LongNet's s_j = j mod r.  Since alpha^t divides the
// level's segment length, that is (i - h) mod alpha^t == 0, so the disjoint decomposition of
// the set union carries over with every valuation taken of (i - h): s = min(nu(|i - h|), K).
enum { LN_MULTISET = 1, LN_HEAD_OFFSETS = 2 };

// Number of pieces of row i (head h: only LongNet with per-head offsets depends on it).
GA_HD int num_pieces_h(const DevMask &M, int64_t i, int h)
{
    switch (M.kind) {
    case K_WINDOW:
    case K_CSR: return 1;
    case K_BLOCK_DILATED: return ((i % M.seg) % M.r == 0) ? 1 : 0;
    case K_LONGNET: {
        const int64_t x = (M.parts & LN_HEAD_OFFSETS) ? i - h : i;
        return (int)valuation(x < 0 ? -x : x, M.alpha, M.K) + 1;
    }
    default: return 0;
    }
}

GA_HD int num_pieces(const DevMask &M, int64_t i) { return num_pieces_h(M, i, 0); }

GA_HD Piece get_piece_h(const DevMask &M, int64_t i, int pc, int h);

// Piece pc of row i.  For LongNet pc = level t in [0, s].
GA_HD Piece get_piece(const DevMask &M, int64_t i, int pc) { return get_piece_h(M, i, pc, 0); }

GA_HD Piece get_piece_h(const DevMask &M, int64_t i, int pc, int h)
{
    Piece P;
    P.mode = P_AFFINE;
    P.alpha = 0;
    P.rexcl = 0;
    P.pad = 0;
    P.cols = nullptr;
    switch (M.kind) {
    case K_WINDOW: {
        int64_t lo = imin(i / M.r, M.m), hi = imin((M.L - 1 - i) / M.r, M.m);
        P.base = i - lo * M.r;
        P.step = M.r;
        P.count = lo + hi + 1;
        return P;
    }
    case K_CSR: {
        int64_t b = M.row_ptr[i];
        P.mode = P_CSR;
        P.cols = M.col_idx;
        P.base = b;
        P.step = 1;
        P.count = M.row_ptr[i + 1] - b;
        return P;
    }
    case K_BLOCK_DILATED: {
        int64_t s0 = (i / M.seg) * M.seg, s1 = imin(M.L, s0 + M.seg);
        P.base = s0;
        P.step = M.r;
        P.count = ceil_div(s1 - s0, M.r);
        return P;
    }
    case K_LONGNET: {
        const int64_t hoff = (M.parts & LN_HEAD_OFFSETS) ? h : 0;
        const int64_t x = i - hoff;
        int64_t s = valuation(x < 0 ? -x : x, M.alpha, M.K);
        if (M.alpha == 2 && M.w0 > 0 && (M.w0 & (M.w0 - 1)) == 0) {
            // alpha = 2 and w0 = 2^lw: the same quantities by shifts and masks (exact)
            const int t = pc, lseg = ctz64(M.w0) + pc;
            const int64_t stp = (int64_t)1 << t;
            const int64_t s0 = (i >> lseg) << lseg, s1 = imin(M.L, s0 + ((int64_t)1 << lseg));
            const int64_t b = s0 + (hoff & (stp - 1));
            const int64_t U = b < s1 ? (s1 - b + stp - 1) >> t : 0;
            P.base = b;
            P.step = stp;
            if (pc < s && !(M.parts & LN_MULTISET)) {
                const int64_t rx = ((b - hoff) >> t) & 1; // (a^t divides b - hoff)
                P.mode = P_SKIPMUL;
                P.alpha = 2;
                P.rexcl = (int32_t)rx;
                P.count = U - (U > rx ? ((U - 1 - rx) >> 1) + 1 : 0);
            } else {
                P.count = U;
            }
            return P;
        }
        int64_t stp = ipow(M.alpha, pc);
        int64_t segw = M.w0 * stp;
        int64_t s0 = (i / segw) * segw, s1 = imin(M.L, s0 + segw);
        const int64_t b = s0 + hoff % stp; // first position == h (mod a^t): a^t divides s0
        int64_t U = b < s1 ? ceil_div(s1 - b, stp) : 0; // such positions in the segment
        P.base = b;
        P.step = stp;
        if (pc < s && !(M.parts & LN_MULTISET)) { // multiset: every level keeps all of them
            // keep j = b + a^t u with nu(j - h) == t exactly, i.e. ((b - h)/a^t + u) mod a != 0:
            // exclude the residue u == -((b - h)/a^t) (mod a)  (b - h is a multiple of a^t)
            const int64_t q0 = (b - hoff) / stp;
            const int64_t c0 = ((q0 % M.alpha) + M.alpha) % M.alpha;
            const int64_t rx = (M.alpha - c0) % M.alpha;
            P.mode = P_SKIPMUL;
            P.alpha = (int32_t)M.alpha;
            P.rexcl = (int32_t)rx;
            P.count = U - (U > rx ? (U - 1 - rx) / M.alpha + 1 : 0);
        } else {
            P.count = U;
        }
        return P;
    }
    default: P.base = 0; P.step = 1; P.count = 0; return P;
    }
}

GA_HD int64_t piece_at(const Piece &P, int64_t k)
{
    if (P.mode == P_AFFINE) return P.base + k * P.step;
    if (P.mode == P_CSR) return (int64_t)P.cols[P.base + k];
    if (P.alpha == 2) return P.base + P.step * (2 * k + (P.rexcl == 0 ? 1 : 0)); // the common alpha
    const int64_t a1 = P.alpha - 1;
    const int64_t idx = k % a1;
    const int64_t u = (k / a1) * P.alpha + (idx < P.rexcl ? idx : idx + 1);
    return P.base + P.step * u;
}

// Degree |N(i)| (closed form per family; SURVEY §8(c) "Per-row degrees").
GA_HD int64_t degree(const DevMask &M, int64_t i)
{
    int n = num_pieces(M, i);
    int64_t d = 0;
    for (int pc = 0; pc < n; ++pc) d += get_piece(M, i, pc).count;
    return d;
}

// SplitMix64 output function of state x + gamma (reading R22 / R10).
GA_HD uint64_t splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ---- BigBird helpers (used by the CSR generator; readings R8-R10) ----------------
GA_HD int64_t bb_global_at(const DevMask &M, int64_t k)
{
    if (M.gidx) return M.gidx[k];
    return (int64_t)((k * M.L) / M.ng); // k < 2^20 and L < 2^43 keep this in int64
}

// number of globals with value < x (G sorted ascending)
GA_HD int64_t bb_count_below(const DevMask &M, int64_t x)
{
    int64_t lo = 0, hi = M.ng;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (bb_global_at(M, mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

GA_HD bool bb_is_global(const DevMask &M, int64_t j)
{
    int64_t k = bb_count_below(M, j);
    return k < M.ng && bb_global_at(M, k) == j;
}

GA_HD void bb_window(const DevMask &M, int64_t i, int64_t &lo, int64_t &hi)
{
    lo = imax(0, i - M.w + 1);
    hi = imin(M.L - 1, i + M.w - 1);
}

// the BigBird window predicate: WINDOW(w, r) (r = 1 unless dilated)
GA_HD bool bb_in_window(const DevMask &M, int64_t i, int64_t j)
{
    const int64_t d = i > j ? i - j : j - i;
    return d < M.w && d % M.r == 0;
}

// |W_i| in closed form (the window rows inside [0, L))
GA_HD int64_t bb_wsize(const DevMask &M, int64_t i)
{
    return 1 + imin(i, M.w - 1) / M.r + imin(M.L - 1 - i, M.w - 1) / M.r;
}

// globals inside W_i
GA_HD int64_t bb_globals_in_window(const DevMask &M, int64_t i)
{
    int64_t lo, hi;
    bb_window(M, i, lo, hi);
    const int64_t a = bb_count_below(M, lo), b = bb_count_below(M, hi + 1);
    if (M.r == 1) return b - a;
    int64_t n = 0;
    for (int64_t k = a; k < b; ++k) n += bb_in_window(M, i, bb_global_at(M, k)) ? 1 : 0;
    return n;
}

// |W_i U G| for a non-global row
GA_HD int64_t bb_wg(const DevMask &M, int64_t i) { return bb_wsize(M, i) + (M.ng - bb_globals_in_window(M, i)); }

// degree of row i restricted to the selected components (window | global \ window | random)
GA_HD int64_t bb_degree(const DevMask &M, int64_t i)
{
    const int parts = M.parts ? M.parts : 7;
    const int64_t nw = bb_wsize(M, i);
    if (bb_is_global(M, i)) return ((parts & 1) ? nw : 0) + ((parts & 2) ? M.L - nw : 0);
    const int64_t gout = M.ng - bb_globals_in_window(M, i);
    const int64_t comp = M.L - (nw + gout);
    return ((parts & 1) ? nw : 0) + ((parts & 2) ? gout : 0) + ((parts & 4) ? imin(comp, M.nrand) : 0);
}

// candidate t of row i: floor((splitmix64(splitmix64(seed) ^ (i*2^20 + t)) >> 32) * L / 2^32)
GA_HD int64_t bb_candidate(const DevMask &M, uint64_t base, int64_t i, uint64_t t)
{
    uint64_t h = splitmix64(base ^ ((uint64_t)i * (1ULL << 20) + t));
    uint64_t hi32 = h >> 32;
#if defined(__CUDA_ARCH__)
    return (int64_t)__umul64hi(hi32 << 32, (uint64_t)M.L);
#else
    return (int64_t)(((unsigned __int128)hi32 * (uint64_t)M.L) >> 32);
#endif
}

} // namespace ga

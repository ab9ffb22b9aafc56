// window_tiled.cu — tensor-core band kernel for Window(w, r) masks (bf16 / fp16).
//
// Residue class c of a dilated window is a pure band: class rows a (token c + a*r) see class
// rows b with |a - b| <= m, m = floor((w-1)/r) (readings R1/R2).  A CTA takes
// ROWS = 112 consecutive class rows of one (class, head) and stages the Q tile and the K/V
// band they reach in shared memory (cp.async 16-byte chunks, XOR swizzle so ldmatrix and
// per-lane row reads are bank-conflict free).  Each warp owns 16 rows; the keys they reach
// split into
//
//   F  = keys every one of the 16 rows sees      -> 16-key blocks on the tensor cores
//        (mma.sync m16n8k16: S = Q K^T, online softmax in registers, O += P V)
//   U\F plus F's ragged tail (< 16 keys)        -> CUDA cores, ONLY the valid pairs,
//        with FHFMA (bf16 x bf16 + f32) so no per-element conversion is needed
//
// so no masked-out product is computed (work optimality) and the tensor
// cores only see dense contractions.  For interior warps U\F is two 16x15 triangles; the
// pairing "row x takes its 15-x left keys and x right keys" gives every lane exactly 15
// edges (no idle lanes).  Warps whose band is clipped by the sequence ends, or whose tile
// is cut by the query range, use a predicated general loop for U\F.  The CUDA-core state
// seeds the MMA phase's running (m, l, O) through a per-warp shared-memory hand-off.
#include "tc_common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace ga {
namespace band {

#ifdef GA_BAND_PROF
__device__ unsigned long long g_prof[8];
#define PROF_T(var) const long long var = clock64()
#define PROF_ADD(k, a, b) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_prof[k], (unsigned long long)((b) - (a))); } while (0)
#else
#define PROF_T(var)
#define PROF_ADD(k, a, b)
#endif

constexpr int WARPS = 7; // 112 rows: two CTAs (28 KB Q + 94 KB band each) fit one SM at m=127
constexpr int ROWS = 16 * WARPS;
constexpr int THREADS = 32 * WARPS;
constexpr int MAX_GEN = 48; // keys of U\F (+ tail) a clipped warp may have: <= 15 + 15 + 15

using tc::Geo;
using tc::ldsm_x4;
using tc::ldsm_x4_t;
using tc::lds16;
using tc::swz;
using tc::cp_async16;

constexpr int QBOX = 56; // rows per TMA box of the Q tile (2 boxes)
// TMA boxes of the K/V band: 64 rows (box * r <= 256 tokens up to r = 4; 32 rows beyond).
// Few large boxes issue fastest (8- and 16-row boxes measured slower at cfg2; 128 rows no
// faster than 64)
__host__ __device__ constexpr int band_box_rows(int64_t r) { return r <= 4 ? 64 : 32; }

struct BandParams {
    CUtensorMap tmQ, tmK, tmV; // TMA maps of one residue class x head (element stride r)
    AttnParams p;
    int64_t m;          // band half-width in class rows
    int64_t r;          // dilation = number of classes
    int64_t tiles;      // tiles per (class, head) (max over classes)
    int64_t edge_tiles; // tiles at each end whose band may be clipped (scheduled first)
    uint32_t smem_bytes;
    int32_t tma;        // 1: tiles whose band is local load through the tensor maps
    int32_t bbox;       // rows per TMA box of the band (band_box_rows(r))
};

// band rows allocated: ROWS + 2m rounded up to whole TMA boxes (multiples of 16 rows, so the
// V band starts on a swizzle period: 1024 B at d = 64, 512 B at d = 32)
__host__ __device__ constexpr int64_t band_alloc_rows(int64_t m, int64_t r)
{
    return (ROWS + 2 * m + band_box_rows(r) - 1) / band_box_rows(r) * band_box_rows(r);
}

template <int D> __host__ __device__ constexpr uint32_t band_smem(int64_t m, int64_t r)
{
    return (uint32_t)(1024                                           // alignment slack
                      + ROWS * Geo<D>::RB                            // Q tile (hand-off + output staging)
                      + 2 * band_alloc_rows(m, r) * Geo<D>::RB + 64); // K and V band, 2 mbarriers
}

// One CUDA-core edge: score of (q half, key half) -> full score via the lane pair.
template <typename T, int D>
__device__ __forceinline__ float half_dot(const uint32_t *qv, uint32_t rowaddr, int key, int hf)
{
    constexpr int HC = Geo<D>::HC;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f; // four independent FHFMA chains
#pragma unroll
    for (int k = 0; k < HC; ++k) {
        const uint4 u = lds16(rowaddr + swz<D>(key, hf * HC + k));
        s0 = fma2h<T>(qv[4 * k], u.x, s0);
        s1 = fma2h<T>(qv[4 * k + 1], u.y, s1);
        s2 = fma2h<T>(qv[4 * k + 2], u.z, s2);
        s3 = fma2h<T>(qv[4 * k + 3], u.w, s3);
    }
    float s = (s0 + s1) + (s2 + s3);
    return s + __shfl_xor_sync(0xffffffffu, s, 1);
}

template <typename T, int D>
__device__ __forceinline__ void half_axpy(float *oc, float pr, uint32_t vaddr, int key, int hf)
{
    constexpr int HC = Geo<D>::HC;
    const uint32_t p2 = pack2<T>(pr, pr);
#pragma unroll
    for (int k = 0; k < HC; ++k) {
        const uint4 u = lds16(vaddr + swz<D>(key, hf * HC + k));
        axpy2h<T>(p2, u.x, oc[8 * k + 0], oc[8 * k + 1]);
        axpy2h<T>(p2, u.y, oc[8 * k + 2], oc[8 * k + 3]);
        axpy2h<T>(p2, u.z, oc[8 * k + 4], oc[8 * k + 5]);
        axpy2h<T>(p2, u.w, oc[8 * k + 6], oc[8 * k + 7]);
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(THREADS, (D <= 64 ? 2 : 1)) band_kernel(const __grid_constant__ BandParams bp)
{
    using G = Geo<D>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const AttnParams &p = bp.p;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int H = p.H;
    const int64_t r = bp.r, m = bp.m, L = p.mask.L;

    // CTA geometry (32-bit divisions: the grid and r*H fit in 32 bits; 64-bit only for
    // sequences beyond 2^31 tokens)
    PROF_T(t_start);
    const uint32_t rH = (uint32_t)(r * H), bid = blockIdx.x;
    const uint32_t ch = bid % rH;
    // tile order: the tiles at both sequence ends (clipped bands, predicated paths) run first
    const int64_t ord = bid / rH;
    const int64_t nb = imin(bp.edge_tiles, bp.tiles / 2);
    const int64_t tile = ord < nb ? ord : ord < 2 * nb ? bp.tiles - 1 - (ord - nb) : ord - nb;
    const int64_t c = ch / (uint32_t)H;
    const int h = (int)(ch - (uint32_t)c * (uint32_t)H);
    if (c >= L) return;
    const int64_t q_end = p.q_begin + p.q_rows;
    auto cdiv = [&](int64_t a) -> int64_t { // ceil(a / r) for a >= 0
        if (a < (int64_t)0x7fffffff) return (int64_t)(((uint32_t)a + (uint32_t)r - 1u) / (uint32_t)r);
        return (a + r - 1) / r;
    };
    const int64_t Nc = cdiv(L - c); // class rows in [0, L)
    const int64_t a_lo = p.q_begin > c ? cdiv(p.q_begin - c) : 0;
    const int64_t a_hi = q_end > c ? imin(cdiv(q_end - c), Nc) : 0;
    // tiles are anchored at absolute class-row multiples of ROWS, so a query-range shard
    // aligned to ROWS*r tokens computes every row exactly as the unsharded launch does
    const int64_t a0 = (a_lo / ROWS) * ROWS + tile * ROWS;
    if (a0 >= a_hi) return;
    const int64_t v_lo = imax(a0, a_lo), v_hi = imin(a0 + ROWS, a_hi); // valid rows [v_lo, v_hi)
    const bool interior = v_lo == a0 && v_hi == a0 + ROWS && a0 - m >= 0 && a0 + ROWS - 1 + m <= Nc - 1;

    const int64_t NB = ROWS + 2 * m; // band rows; band-local 0 = class row a0 - m
    const int64_t NBA = band_alloc_rows(m, r);
    const int BBOX = bp.bbox;
    // 1024-byte aligned base: the 128B swizzle of TMA follows the address bits, tc::swz the row
    const uint32_t sraw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbase = (sraw + 1023u) & ~1023u;
    const uint32_t sQ = sbase, sK = sQ + ROWS * G::RB, sV = sK + (uint32_t)(NBA * G::RB);
    const uint32_t mb0 = sV + (uint32_t)(NBA * G::RB), mb1 = mb0 + 8; // TMA stage barriers

    // ---- per-warp key geometry (band-local indices; abs = a0 - m + local)
    const int w16 = warp * 16;
    const int64_t x0 = a0 + w16; // first absolute class row of this warp
    const int64_t wv_lo = imax(x0, v_lo), wv_hi = imin(x0 + 16, v_hi);
    const bool warp_live = wv_lo < wv_hi;
    const int64_t base = a0 - m;
    const int Ulo = (int)(imax(0, x0 - m) - base), Uhi = (int)(imin(Nc - 1, x0 + 15 + m) - base);
    const int Flo = (int)(imax(0, x0 + 15 - m) - base), Fhi = (int)(imin(Nc - 1, x0 + m) - base);
    const int nF = Fhi - Flo + 1;            // >= 2m - 14 - clipping > 0 for m >= 15
    const int q16 = nF > 0 ? nF / 16 : 0;    // dense 16-key blocks (tensor cores)
    const int rem = nF > 0 ? nF % 16 : 0;    // ragged dense tail (CUDA cores)

    // ---- stage Q rows and the K/V band rows the valid rows reach (16-byte cp.async)
    const size_t row_bytes = (size_t)H * D * sizeof(T);
    const char *Qg = reinterpret_cast<const char *>(p.Q) + (size_t)h * D * sizeof(T);
    const char *Kg = reinterpret_cast<const char *>(p.K) + (size_t)h * D * sizeof(T);
    const char *Vg = reinterpret_cast<const char *>(p.V) + (size_t)h * D * sizeof(T);
    const int ld_lo = (int)(imax(0, v_lo - m) - base), ld_hi = (int)(imin(Nc - 1, v_hi - 1 + m) - base) + 1;
    // band row `row` (class row base+row, token c + (base+row)*r) starts at band0 + row*rstride;
    // the pointers are formed for in-range rows only (base may be negative for clipped tiles)
    const uint32_t rstride = (uint32_t)(r * row_bytes); // < 4 GB: one 32x32->64 multiply per row
    const int64_t band_tok0 = c + base * r - p.kv_begin;
    // sharded runs: a tile at a shard edge reaches rows owned by the neighbour ranks and
    // reads them from their memory (kv_row); every other tile takes the strided fast path
    const bool band_local = p.k_peer == nullptr ||
                            (band_tok0 + ld_lo * r >= 0 && band_tok0 + (int64_t)(ld_hi - 1) * r < p.kv_rows);
    const size_t hoff = (size_t)h * D * sizeof(T);
    auto load_band = [&](int r0, int r1) {
        r0 = max(r0, ld_lo);
        r1 = min(r1, ld_hi);
        if (band_local) {
            for (int idx = r0 * G::NC + tid; idx < r1 * G::NC; idx += THREADS) {
                const int row = idx / G::NC, cc = idx % G::NC;
                const int64_t off =
                    band_tok0 * (int64_t)row_bytes + (int64_t)((uint64_t)(uint32_t)row * rstride) + cc * 16;
                cp_async16(sK + swz<D>(row, cc), Kg + off);
                cp_async16(sV + swz<D>(row, cc), Vg + off);
            }
        } else {
            for (int idx = r0 * G::NC + tid; idx < r1 * G::NC; idx += THREADS) {
                const int row = idx / G::NC, cc = idx % G::NC;
                const char *kr, *vr;
                kv_row(p, c + (base + row) * r, row_bytes, kr, vr);
                cp_async16(sK + swz<D>(row, cc), kr + hoff + cc * 16);
                cp_async16(sV + swz<D>(row, cc), vr + hoff + cc * 16);
            }
        }
    };
    // stage 0: rows the CUDA-core phase reads (ends of the band); stage 1: the dense middle,
    // which lands while the CUDA-core phase runs
    const int mid0 = ROWS - 1, mid1 = max(mid0, (int)(2 * m + 1) - 16);
    const bool use_tma = bp.tma && band_local;
    if (use_tma) {
        // TMA: warp 0 issues the boxes (Q tile and band ends -> barrier 0; band middle ->
        // barrier 1).  Rows outside the sequence / query range come back as zeros, which
        // also defines the pad rows of clipped tiles (they join the rescale votes).
        const int s0 = (mid0 + BBOX - 1) / BBOX, s1 = max(s0, mid1 / BBOX); // stage-1 boxes [s0, s1)
        const int nbox = (int)(NBA / BBOX);
        if (tid == 0) {
            umma::mbar_init(mb0, 1);
            umma::mbar_init(mb1, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (warp == 0) {
            constexpr uint32_t QB = QBOX * G::RB;
            const uint32_t BB = (uint32_t)BBOX * G::RB;
            if (lane == 0) {
                tma::expect_tx(mb0, (uint32_t)(ROWS / QBOX) * QB + 2u * (uint32_t)(nbox - (s1 - s0)) * BB);
                tma::expect_tx(mb1, 2u * (uint32_t)(s1 - s0) * BB);
            }
            __syncwarp();
            const int qtok0 = (int)(c + a0 * r - p.q_begin), ktok0 = (int)(c + base * r - p.kv_begin);
            if (lane < ROWS / QBOX)
                tma::load_3d(sQ + lane * QB, &bp.tmQ, 0, h, qtok0 + lane * QBOX * (int)r, mb0);
            if (lane < nbox) {
                const uint32_t mb = (lane >= s0 && lane < s1) ? mb1 : mb0;
                tma::load_3d(sK + lane * BB, &bp.tmK, 0, h, ktok0 + lane * BBOX * (int)r, mb);
                tma::load_3d(sV + lane * BB, &bp.tmV, 0, h, ktok0 + lane * BBOX * (int)r, mb);
            }
        }
        umma::mbar_wait(mb0, 0);
        if (!interior) umma::mbar_wait(mb1, 0); // clipped: CUDA keys may be anywhere
    } else {
        const char *Qt = Qg + (c + a0 * r - p.q_begin) * (int64_t)row_bytes;
        const int q_lo = (int)(v_lo - a0), q_hi = (int)(v_hi - a0);
        for (int idx = q_lo * G::NC + tid; idx < q_hi * G::NC; idx += THREADS) {
            const int row = idx / G::NC, cc = idx % G::NC;
            cp_async16(sQ + swz<D>(row, cc), Qt + (int64_t)((uint64_t)(uint32_t)row * rstride) + cc * 16);
        }
        if (!interior) { // pad rows of a clipped tile join the rescale votes: make them defined
            for (int idx = tid; idx < ROWS * G::NC; idx += THREADS) {
                const int row = idx / G::NC;
                if (row < q_lo || row >= q_hi) tc::sts_zero16(sQ + swz<D>(row, idx % G::NC));
            }
        }
        load_band(0, mid0);
        load_band(mid1, (int)NB);
        asm volatile("cp.async.commit_group;" ::: "memory");
        load_band(mid0, mid1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (interior) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory"); // clipped: CUDA keys may be anywhere
        __syncthreads();
    }

    PROF_T(t_loaded);
    PROF_ADD(0, t_start, t_loaded);
    const float sl2 = p.scale_log2;

    // A fragments of Q for the tensor-core phase, taken before the Q rows are reused
    const int g = lane >> 2, t4 = lane & 3;
    tc::MmaRows<T, D> rs; // running (m, l, O) of the warp's 16 rows in the mma layout
    auto &qa = rs.qa;
    auto &o = rs.o;
    auto &mr = rs.mr;
    auto &lr = rs.lr;
    if (warp_live) {
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) {
            const int row = w16 + (lane & 7) + ((lane >> 3) & 1) * 8;
            const int chk = 2 * kk + (lane >> 4);
            ldsm_x4(sQ + swz<D>(row, chk), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
        }
    }

    // ================= CUDA-core phase: U\F and F's ragged tail =================
    if (warp_live) {
        const int x = lane >> 1, hf = lane & 1;
        uint32_t qv[G::HC * 4];
#pragma unroll
        for (int k = 0; k < G::HC; ++k) {
            const uint4 u = lds16(sQ + swz<D>(w16 + x, hf * G::HC + k));
            qv[4 * k] = u.x; qv[4 * k + 1] = u.y; qv[4 * k + 2] = u.z; qv[4 * k + 3] = u.w;
        }
        float mc = -INFINITY, lc = 0.f, oc[D / 2];
#pragma unroll
        for (int e = 0; e < D / 2; ++e) oc[e] = 0.f;
        if (interior) {
            // exact triangles: row x takes left keys Ulo+x..Ulo+14 and right keys
            // Fhi+1..Fhi+x, then the ragged tail Flo+16*q16 ..; 15 + rem steps, all lanes busy
            const int steps = 15 + rem; // <= 30
            auto key_of = [&](int t) {
                if (t < 15) return (t < 15 - x) ? (Ulo + x + t) : (Fhi + 1 + (t - 15 + x));
                return Flo + 16 * q16 + (t - 15);
            };
            float sc[30]; // pass 1: scores and their exact max (no rescaling needed)
#pragma unroll
            for (int t = 0; t < 30; ++t) {
                if (t >= steps) break;
                sc[t] = half_dot<T, D>(qv, sK, key_of(t), hf) * sl2;
                mc = fmaxf(mc, sc[t]);
            }
#pragma unroll
            for (int t = 0; t < 30; ++t) { // pass 2: weights, weighted sum of V
                if (t >= steps) break;
                const float pr = ex2(sc[t] - mc);
                lc += pr;
                half_axpy<T, D>(oc, pr, sV, key_of(t), hf);
            }
        } else {
            // clipped / cut warp: candidates [Ulo,Flo) U [Flo+16*q16, Fhi] U (Fhi, Uhi],
            // each pair predicated on |row - key| <= m and the row being valid
            const int64_t xa = x0 + x;
            const bool row_ok = xa >= wv_lo && xa < wv_hi;
            const int n_left = Flo - Ulo, n_tail = rem, n_right = Uhi - Fhi;
            const int n_all = n_left + n_tail + n_right;
            for (int t = 0; t < n_all; ++t) {
                const int key = t < n_left ? Ulo + t : t < n_left + n_tail ? Flo + 16 * q16 + (t - n_left)
                                                                             : Fhi + 1 + (t - n_left - n_tail);
                const int64_t ka = base + key;
                const bool ok = row_ok && ka >= xa - m && ka <= xa + m;
                if (!__any_sync(0xffffffffu, ok)) continue;
                const float s = half_dot<T, D>(qv, sK, key, hf) * sl2;
                if (ok) {
                    if (s > mc) { // online update with rescale (rare path)
                        const float a = ex2(mc - s);
                        lc *= a;
#pragma unroll
                        for (int e = 0; e < D / 2; ++e) oc[e] *= a;
                        mc = s;
                    }
                    const float pr = ex2(s - mc);
                    lc += pr;
                    half_axpy<T, D>(oc, pr, sV, key, hf);
                }
            }
        }
        // ---- hand-off into the MMA layout (lane (g,t4): rows g, g+8; dims 8j+2t4, +1):
        // m and l by shuffles, o through this warp's 16 Q rows (one half-row per round;
        // a half-row of fp32 is exactly one Q row of bytes)
        __syncwarp(); // every lane has finished reading its Q rows
        mr[0] = __shfl_sync(0xffffffffu, mc, 2 * g);
        mr[1] = __shfl_sync(0xffffffffu, mc, 2 * (g + 8));
        const float l0 = __shfl_sync(0xffffffffu, lc, 2 * g), l1 = __shfl_sync(0xffffffffu, lc, 2 * (g + 8));
        lr[0] = t4 == 0 ? l0 : 0.f;
        lr[1] = t4 == 0 ? l1 : 0.f;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            if (hf == hh) {
#pragma unroll
                for (int k = 0; k < G::NC; ++k)
                    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(sQ + swz<D>(w16 + x, k)),
                                 "f"(oc[4 * k]), "f"(oc[4 * k + 1]), "f"(oc[4 * k + 2]), "f"(oc[4 * k + 3]));
            }
            __syncwarp();
#pragma unroll
            for (int jl = 0; jl < G::NB8 / 2; ++jl) {
                const int j = hh * (G::NB8 / 2) + jl, chunk = 2 * jl + (t4 >> 1);
                float2 v0, v1;
                asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v0.x), "=f"(v0.y)
                             : "r"(sQ + swz<D>(w16 + g, chunk) + (t4 & 1) * 8));
                asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v1.x), "=f"(v1.y)
                             : "r"(sQ + swz<D>(w16 + g + 8, chunk) + (t4 & 1) * 8));
                o[j][0] = v0.x;
                o[j][1] = v0.y;
                o[j][2] = v1.x;
                o[j][3] = v1.y;
            }
            __syncwarp();
        }
    }
    PROF_T(t_cuda);
    PROF_ADD(1, t_loaded, t_cuda);
    if (use_tma) {
        umma::mbar_wait(mb1, 0); // dense rows landed
    } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads(); // dense rows landed
    }
    PROF_T(t_dense);
    PROF_ADD(2, t_cuda, t_dense);
    if (!warp_live) return; // no further CTA-wide barriers

    // ================= tensor-core phase: dense 16x16 blocks of F =================
    // per-lane ldmatrix row offsets are block-invariant up to +16*b*RB
    // per-lane ldmatrix addresses of block 0; block b adds 16*b rows (the swizzle phase
    // repeats every 8 rows, so the offset is a plain add)
    uint32_t kaddr[G::KS], vaddr[G::NB8 / 2];
    {
        const int krow = Flo + (lane & 7) + (lane >> 4) * 8;       // K (non-trans) rows
        const int vrow = Flo + (lane & 7) + ((lane >> 3) & 1) * 8; // V (trans) rows
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) kaddr[kk] = sK + swz<D>(krow, 2 * kk + ((lane >> 3) & 1));
#pragma unroll
        for (int jj = 0; jj < G::NB8 / 2; ++jj) vaddr[jj] = sV + swz<D>(vrow, 2 * jj + (lane >> 4));
    }
    {
        tc::MmaRows<T, D> &st = rs;
        int b = 0;
        for (; b + 1 < q16; b += 2) // pairs: both S tiles, one vote, both P V updates
            st.block16x2(kaddr, vaddr, (uint32_t)(b * 16 * G::RB), (uint32_t)((b + 1) * 16 * G::RB), sl2);
        if (b < q16) st.block16(kaddr, vaddr, (uint32_t)(b * 16 * G::RB), sl2);
    }
    PROF_T(t_mma);
    PROF_ADD(3, t_dense, t_mma);
    // ---- finalise: l = quad sum, normalise, stage through this warp's Q rows, store
    rs.reduce_l();
    const float inv0 = lr[0] > 0.f ? 1.f / lr[0] : 0.f, inv1 = lr[1] > 0.f ? 1.f / lr[1] : 0.f;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < G::NB8; ++j) {
        const uint32_t w0 = pack2<T>(o[j][0] * inv0, o[j][1] * inv0);
        const uint32_t w1 = pack2<T>(o[j][2] * inv1, o[j][3] * inv1);
        // element (row, col 8j + 2t4) sits in chunk j, byte 4*t4
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sQ + swz<D>(w16 + g, j) + 4 * t4), "r"(w0));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sQ + swz<D>(w16 + g + 8, j) + 4 * t4), "r"(w1));
    }
    __syncwarp();
    char *Og = reinterpret_cast<char *>(p.out) + (size_t)h * D * sizeof(T);
#pragma unroll
    for (int idx = lane; idx < 16 * G::NC; idx += 32) {
        const int row = idx / G::NC, cc = idx % G::NC;
        const int64_t xa = x0 + row;
        if (xa < wv_lo || xa >= wv_hi) continue;
        const int64_t i = c + xa * r;
        stg16(Og + (size_t)(i - p.q_begin) * row_bytes + cc * 16, lds16(sQ + swz<D>(w16 + row, cc)));
    }
    PROF_T(t_end);
    PROF_ADD(4, t_mma, t_end);
    PROF_ADD(5, t_start, t_end);
}

static constexpr uint32_t kMaxSmem = 227 * 1024;

template <typename T, int D> static ga_status launch_t(const BandParams &bp, cudaStream_t s)
{
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(band_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
        if (e != cudaSuccess) return cuda_fail(e, "band_kernel: set smem");
        configured = true;
    }
    const int64_t blocks = bp.tiles * bp.r * bp.p.H;
    if (blocks == 0) return GA_OK;
    band_kernel<T, D><<<(unsigned)blocks, THREADS, bp.smem_bytes, s>>>(bp);
    GA_CHECK_LAUNCH("band_kernel");
    return GA_OK;
}

} // namespace band

#ifdef GA_BAND_PROF
extern "C" void ga_band_prof_read(unsigned long long *out)
{
    cudaMemcpyFromSymbol(out, band::g_prof, sizeof(unsigned long long) * 8);
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(band::g_prof, z, sizeof(z));
}
#endif

static uint32_t band_smem_for(int d, int64_t m, int64_t r)
{
    switch (d) {
    case 32: return band::band_smem<32>(m, r);
    case 64: return band::band_smem<64>(m, r);
    default: return band::band_smem<128>(m, r);
    }
}

int64_t band_tile_rows() { return band::ROWS; }

bool window_tiled_supported(const AttnParams &p, ga_dtype dt)
{
    if (p.mask.kind != K_WINDOW || (dt != GA_BF16 && dt != GA_F16)) return false;
    if (p.mask.m < 15) return false;
    return band_smem_for(p.d, p.mask.m, p.mask.r) <= band::kMaxSmem;
}

ga_status launch_window_tiled(const AttnParams &p, ga_dtype dt, cudaStream_t s)
{
    band::BandParams bp;
    bp.p = p;
    bp.m = p.mask.m;
    bp.r = p.mask.r;
    // class rows of the query range per class: at most ceil(q_rows / r) + 1
    const int64_t per_class = (p.q_rows + bp.r - 1) / bp.r + 1;
    bp.tiles = (per_class + band::ROWS - 1) / band::ROWS + 1; // +1: grid anchored at ROWS multiples
    bp.edge_tiles = (bp.m + band::ROWS - 1) / band::ROWS + 2;
    bp.smem_bytes = band_smem_for(p.d, bp.m, bp.r);
    bp.bbox = band::band_box_rows(bp.r);
    // TMA maps of Q (query rows) and K/V (key rows) with element stride r; d = 128 rows
    // (256 B) exceed one swizzle span and dilations above 8 exceed the traversal stride,
    // those keep the cp.async path
    bp.tma = p.d <= 64 && (int64_t)bp.bbox * bp.r <= 256 && band::QBOX * bp.r <= 256 &&
             band::band_alloc_rows(bp.m, bp.r) / bp.bbox <= 32 &&
             tma::encode_rows(&bp.tmQ, p.Q, p.q_rows, p.H, p.d, (int)bp.r, band::QBOX) &&
             tma::encode_rows(&bp.tmK, p.K, p.kv_rows, p.H, p.d, (int)bp.r, bp.bbox) &&
             tma::encode_rows(&bp.tmV, p.V, p.kv_rows, p.H, p.d, (int)bp.r, bp.bbox);
    if (bp.r * p.H * bp.tiles > (int64_t)INT32_MAX) {
        set_error("band kernel grid too large");
        return GA_ERR_UNSUPPORTED;
    }
    if (dt == GA_BF16) {
        switch (p.d) {
        case 32: return band::launch_t<__nv_bfloat16, 32>(bp, s);
        case 64: return band::launch_t<__nv_bfloat16, 64>(bp, s);
        case 128: return band::launch_t<__nv_bfloat16, 128>(bp, s);
        }
    } else {
        switch (p.d) {
        case 32: return band::launch_t<__half, 32>(bp, s);
        case 64: return band::launch_t<__half, 64>(bp, s);
        case 128: return band::launch_t<__half, 128>(bp, s);
        }
    }
    set_error("band kernel: unsupported d");
    return GA_ERR_UNSUPPORTED;
}

} // namespace ga

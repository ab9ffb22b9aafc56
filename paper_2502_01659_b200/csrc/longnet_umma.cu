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
// mbarrier.  Two CTAs per SM overlap one CTA's softmax with the other's MMAs.  Groups with
// fewer than 128 rows stay on the mma.sync kernel (longnet_tc.cu).
#include <type_traits>

#include "tc_common.cuh"
#include "umma.cuh"

namespace ga {
namespace lnet_umma {
using namespace tc;
using namespace umma;

constexpr int ROWS = 128, THREADS = 128, KC = 64, STAGES = 4;
constexpr int MAX_ITEMS = 64, MAX_PIECES = 64;

struct UParams {
    AttnParams p;
    int64_t seg0, n_seg;
    int32_t n_items;
    int16_t item_s[MAX_ITEMS];
    int16_t item_tile[MAX_ITEMS];
};

template <int D> __host__ __device__ constexpr uint32_t smem_bytes()
{
    return 1024 /* alignment slack */ + ROWS * 2 * D /* Q */ + STAGES * 2 * KC * 2 * D /* K,V */ + ROWS * 8 /* rows */ +
           64 /* mbarriers, tmem base */;
}

// TMEM columns: S[2] at 0 and KC, P[2] (16-bit pairs) at 2KC and 2KC + KC/2, O at 3KC
constexpr uint32_t COL_S = 0, COL_P = 2 * KC, COL_O = 3 * KC; // S0 S1 | P0 P1 | O  (256 columns at d=64)

template <typename T, int D>
__global__ void __launch_bounds__(THREADS, 2) longnet_umma_kernel(const UParams up)
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
    uint32_t *tmem_base_smem = reinterpret_cast<uint32_t *>(mbars + 4);
    const uint32_t mbS[2] = {(uint32_t)__cvta_generic_to_shared(&mbars[0]), (uint32_t)__cvta_generic_to_shared(&mbars[1])};
    const uint32_t mbO[2] = {(uint32_t)__cvta_generic_to_shared(&mbars[2]), (uint32_t)__cvta_generic_to_shared(&mbars[3])};

    const AttnParams &p = up.p;
    const DevMask &M = p.mask;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int H = p.H;

    const int64_t IH = (int64_t)up.n_items * H;
    const int64_t segl = (int64_t)blockIdx.x / IH;
    const int64_t rem = (int64_t)blockIdx.x - segl * IH;
    const int64_t item = rem / H;
    const int h = (int)(rem - item * H);
    const int64_t seg = up.seg0 + segl;
    const int s = up.item_s[item], tile = up.item_tile[item];
    const int64_t S0 = seg * M.w0, S1 = imin(M.L, S0 + M.w0);
    const int64_t q_end = p.q_begin + p.q_rows;

    // ---- group rows (closed form, see longnet_tc.cu)
    int64_t step = 1;
    for (int t = 0; t < s; ++t) step *= M.alpha;
    const int64_t lo = imax(S0, p.q_begin), hi = imin(S1, q_end);
    const int64_t f0 = (lo + step - 1) / step;
    const int64_t nq = lo < hi && f0 * step < hi ? (hi - 1) / step - f0 + 1 : 0;
    const bool top = s == (int)M.K;
    const int64_t rx = (M.alpha - f0 % M.alpha) % M.alpha;
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
    // ---- TMEM (warp 0) and mbarriers (thread 0)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(tmem_base_smem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(mbS[b], 1);
            mbar_init(mbO[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_base_smem;

    __shared__ Piece spiece[MAX_PIECES];
    __shared__ int pstart[MAX_PIECES + 1];
    const int np = s + 1;
    if (tid < np) spiece[tid] = get_piece(M, rows[0], tid);
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

    const size_t row_bytes = (size_t)H * D * sizeof(T);
    const char *Qg = reinterpret_cast<const char *>(p.Q) + (size_t)h * D * sizeof(T);
    const size_t hoff = (size_t)h * D * sizeof(T);

    int cur_t = 0;
    auto load_chunk = [&](int c) {
        const int st = c % STAGES;
        const int kl = tid >> 1, hf = tid & 1; // 2 threads per key
        const int k = c * KC + kl;
        if (k < nblk * 16) {
            while (cur_t + 1 < np && pstart[cur_t + 1] <= k) ++cur_t;
            const char *kr, *vr;
            kv_row(p, piece_at(spiece[cur_t], k - pstart[cur_t]), row_bytes, kr, vr);
#pragma unroll
            for (int q = 0; q < D / 16; ++q) {
                const int cc = hf * (D / 16) + q;
                cp_async16(sK0 + st * KC * RB + swz<D>(kl, cc), kr + hoff + cc * 16);
                cp_async16(sV0 + st * KC * RB + swz<D>(kl, cc), vr + hoff + cc * 16);
            }
        } else if (c < nchunks) { // keys past the last whole block in the final chunk: zero
            // K/V rows (the stage holds an older chunk's keys), their scores are masked below
#pragma unroll
            for (int q = 0; q < D / 16; ++q) {
                const int cc = hf * (D / 16) + q;
                sts_zero16(sK0 + st * KC * RB + swz<D>(kl, cc));
                sts_zero16(sV0 + st * KC * RB + swz<D>(kl, cc));
            }
        }
        cp_async_commit();
    };
    // pad rows (>= nrows) are zeroed: they join the warp-uniform rescale vote
    for (int idx = tid; idx < ROWS * (RB / 16); idx += THREADS) {
        const int r = idx / (RB / 16), cc = idx % (RB / 16);
        if (r < nrows)
            cp_async16(sQ + swz<D>(r, cc), Qg + (size_t)(rows[r] - p.q_begin) * row_bytes + cc * 16);
        else
            sts_zero16(sQ + swz<D>(r, cc));
    }
#pragma unroll
    for (int c = 0; c < STAGES - 1; ++c) load_chunk(c); // stages 0..S-2 (empty groups are fine)

    // thread = row = TMEM lane; warp w reads lanes [32w, 32w+32)
    const uint32_t tlane = tmem + ((uint32_t)(warp * 32) << 16);
    const float sl2 = p.scale_log2;
    constexpr float kTau = 8.f;
    float m_run = -INFINITY, l_run = 0.f;
    const uint32_t idS = idesc<T>(ROWS, KC, false), idO = idesc<T>(ROWS, D, true);
    // Software pipeline: S_{c+1} runs on the tensor core while chunk c's softmax runs.
    // S_c -> TMEM S[c&1] (mbarrier mbS[c&1]); P_c -> P[c&1]; P V_c -> O (mbO[c&1]).  The
    // k-th use of a double-buffer slot completes its mbarrier phase with parity k & 1.
    auto issue_S = [&](int c) {
        if (tid == 0) {
            fence_after();
            const uint32_t bk = sK0 + (c % STAGES) * KC * RB;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) // K = 16 per MMA: +32 B inside the swizzle atom
                mma_ss(tmem + COL_S + (c & 1) * KC, sdesc_sw128(sQ + kk * 32), sdesc_sw128(bk + kk * 32), idS,
                       kk > 0);
            mma_commit(mbS[c & 1]);
        }
    };
    auto wait_O = [&](int c) { // P V_c complete
        mbar_wait(mbO[c & 1], (c >> 1) & 1);
        fence_after();
    };
    if (nchunks > 0) { // prologue: chunk 0 (and Q) landed -> S_0
        cp_async_wait<STAGES - 2>();
        fence_proxy_async();
        __syncthreads();
        issue_S(0);
    }
    for (int c = 0; c < nchunks; ++c) {
        const int st = c % STAGES;
        // 1. S_{c+1} (chunks 0..c+2 committed; c+1 must have landed)
        if (c + 1 < nchunks) {
            cp_async_wait<STAGES - 3>();
            fence_proxy_async();
            fence_before(); // the reads of S[(c+1)&1] (chunk c-1) are complete
            __syncthreads();
            issue_S(c + 1);
        }
        // 2. S_c
        mbar_wait(mbS[c & 1], (c >> 1) & 1);
        fence_after();
        float sv[KC];
        tmem_ld32(tlane + COL_S + (c & 1) * KC, sv);
        tmem_ld32(tlane + COL_S + (c & 1) * KC + 32, sv + 32);
        tmem_wait_ld();
        const int valid = nblk * 16 - c * KC; // keys of this chunk (< KC only in the last one)
        if (valid < KC) {
#pragma unroll
            for (int i = 0; i < KC; ++i) sv[i] = i < valid ? sv[i] : -INFINITY;
        }
        float lmx[8]; // 8 independent max chains (a 63-deep serial chain is latency-bound)
#pragma unroll
        for (int j = 0; j < 8; ++j) lmx[j] = sv[j];
#pragma unroll
        for (int i = 8; i < KC; ++i) lmx[i & 7] = fmaxf(lmx[i & 7], sv[i]);
        const float lm = fmaxf(fmaxf(fmaxf(lmx[0], lmx[1]), fmaxf(lmx[2], lmx[3])),
                               fmaxf(fmaxf(lmx[4], lmx[5]), fmaxf(lmx[6], lmx[7])));
        // 3. lazy rescale (O must be stable: the last issued P V is P V_{c-1})
        const bool need = lm * sl2 > m_run + kTau;
        if (__syncthreads_or(need)) {
            if (c > 0) wait_O(c - 1);
            const float mn = fmaxf(m_run, lm * sl2);
            const float a = ex2(m_run - mn);
            // tcgen05.ld/st are .sync.aligned: the whole warp takes the branch (a = 1 rows
            // multiply by one)
            if (__any_sync(0xffffffffu, c > 0 && a != 1.f)) { // rescale the rows of O in TMEM
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
        // 4. P_c into P[c&1] (last read by P V_{c-2})
        if (c >= 2) wait_O(c - 2);
        uint32_t pk[KC / 2];
        float ls[4] = {0.f, 0.f, 0.f, 0.f}; // independent partial sums
#pragma unroll
        for (int i = 0; i < KC / 2; ++i) {
            const float p0 = ex2(fmaf(sv[2 * i], sl2, -m_run)), p1 = ex2(fmaf(sv[2 * i + 1], sl2, -m_run));
            ls[i & 3] += p0 + p1;
            pk[i] = pack2<T>(p0, p1);
        }
        l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        tmem_st32(tlane + COL_P + (c & 1) * (KC / 2), pk);
        tmem_wait_st();
        fence_before();
        __syncthreads();
        if (tid == 0) {
            fence_after();
            const uint32_t bv = sV0 + st * KC * RB;
#pragma unroll
            for (int kk = 0; kk < KC / 16; ++kk) // 16 keys per MMA: 8 P columns, 16 V rows
                mma_ts(tmem + COL_O, tmem + COL_P + (c & 1) * (KC / 2) + kk * 8, sdesc_sw128(bv + kk * 16 * RB), idO,
                       (c > 0 || kk > 0));
            mma_commit(mbO[c & 1]);
        }
        // 5. refill the stage of chunk c-1 (free once P V_{c-1} is done) with chunk c+3
        if (c >= 1) wait_O(c - 1);
        load_chunk(c + STAGES - 1 < nchunks ? c + STAGES - 1 : nchunks + STAGES); // no-op past the end
    }
    cp_async_wait<0>();
    if (nchunks > 0) wait_O(nchunks - 1);
    // ---- O row from TMEM (+ ragged tail on CUDA cores), normalise, store
    const bool row_ok = tid < nrows;
    float o[D];
    if (nchunks > 0) {
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
    if (row_ok) {
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
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
    }
}

template <typename T, int D> static ga_status launch_t(const UParams &up, cudaStream_t s)
{
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(longnet_umma_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem_bytes<D>());
        if (e != cudaSuccess) return cuda_fail(e, "longnet_umma_kernel: set smem");
        configured = true;
    }
    const int64_t blocks = (int64_t)up.n_items * up.n_seg * up.p.H;
    if (blocks == 0) return GA_OK;
    longnet_umma_kernel<T, D><<<(unsigned)blocks, THREADS, smem_bytes<D>(), s>>>(up);
    GA_CHECK_LAUNCH("longnet_umma_kernel");
    return GA_OK;
}

} // namespace lnet_umma

// Launch the tcgen05 kernel on the groups s = 0..s_max (those that fill 128-row tiles);
// the caller runs the remaining groups on the mma.sync kernel.
ga_status launch_longnet_umma(const AttnParams &p, ga_dtype dt, int64_t seg0, int64_t n_seg, int s_max,
                              cudaStream_t s)
{
    lnet_umma::UParams up;
    up.p = p;
    up.seg0 = seg0;
    up.n_seg = n_seg;
    const DevMask &M = p.mask;
    int n = 0;
    int64_t stp = 1;
    for (int t = 0; t <= s_max; ++t) {
        const int64_t cnt = M.w0 / stp + 1;
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
    if (p.d == 64 && dt == GA_BF16) return lnet_umma::launch_t<__nv_bfloat16, 64>(up, s);
    if (p.d == 64 && dt == GA_F16) return lnet_umma::launch_t<__half, 64>(up, s);
    set_error("LongNet tcgen05 kernel: unsupported d/dtype");
    return GA_ERR_UNSUPPORTED;
}

} // namespace ga

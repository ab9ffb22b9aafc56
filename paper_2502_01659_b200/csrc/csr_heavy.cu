// csr_heavy.cu — heavy-row split + state merge for explicit CSR masks.
//
// The paper's global kernel "can only be as fast as its slowest block" because global
// rows are dense.  BigBird rows of global tokens have L edges (2^20 in
// cfg3) against ~383 for the rest, so a row with more than C edges is cut into chunks of
// C edges.  Each chunk is one warp task producing a partial online-softmax state
// (m, l, o~) per head; a merge pass combines a row's partials with the associative
// operator (+): m = max(m1,m2), l = l1 e^{m1-m} + l2 e^{m2-m}, o~ likewise (identity
// (-inf, 0, 0)), then normalises.  The light rows run in the generic edge kernel, which
// skips rows above C.
//
// Plan (deterministic, no atomics):  cnt[i] = deg(i) > C ? ceil(deg/C) : 0  ->  exclusive
// scan -> item table (row, chunk) -> chunk kernel -> merge kernel.  bf16/fp16 chunks run
// on the mma.sync edge blocks of csr_mma.cuh, fp32 on the edge kernel's lane groups.
//
// Full rows (bf16/fp16, L % 16 == 0): a heavy row with deg(i) == L holds every column (a
// valid CSR row is sorted and unique), so all such rows share their neighbour set — the
// global rows of BigBird / Longformer.  They leave the item table and run
// as dense tiles: 64 full rows x a 4096-key chunk per CTA on mma.sync with the keys staged
// once in shared memory (K/V read once per 64 rows instead of once per row), partial states
// per (row, chunk), then the same (+) merge.  The count packs both prefix sums into one
// int64 scan: chunks in bits 0-39, full rows in bits 40-63.
//
// Workspace layout (csr_heavy_workspace):  cnt int64 [L+1] | item_row int64 [I] |
// item_chunk int32 [I] | partials f32 [I * H * (d+2)] | full_row int64 [F] |
// full partials f32 [F * NCH * H * (d+2)],  I = 2*nnz/C + 2 >= sum of chunks,
// F = min(rows, nnz / L) >= number of full rows, NCH = ceil(L / 4096).
#include "csr_mma.cuh"
#include "edge_core.cuh"

namespace ga {

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static int64_t max_items(int64_t nnz, int64_t C) { return 2 * (nnz / C) + 2; }

constexpr int64_t kChunkMask = (int64_t(1) << 40) - 1; // packed count: chunks | full rows << 40
constexpr int FULL_KCH = 4096;                          // keys per full-row CTA
constexpr int FULL_ROWS = 64, FULL_KC = 64, FULL_THREADS = 128;

static int64_t max_full(int64_t rows, int64_t Lm, int64_t nnz) { return Lm > 0 ? imin(rows, nnz / Lm) : 0; }
__host__ __device__ static inline int64_t full_chunks(int64_t Lm) { return (Lm + FULL_KCH - 1) / FULL_KCH; }

size_t csr_heavy_workspace(int64_t rows, int64_t Lm, int64_t nnz, int32_t H, int32_t d, int64_t C)
{
    const int64_t I = max_items(nnz, C);
    const int64_t F = max_full(rows, Lm, nnz);
    return align256(sizeof(int64_t) * (rows + 1)) + align256(sizeof(int64_t) * I) + align256(sizeof(int32_t) * I) +
           align256(sizeof(float) * (size_t)I * H * (d + 2)) + align256(sizeof(int64_t) * F) +
           align256(sizeof(float) * (size_t)F * full_chunks(Lm) * H * (d + 2));
}

__global__ void heavy_count_kernel(const int64_t *row_ptr, int64_t row0, int64_t rows, int64_t C, int64_t Lfull,
                                   int64_t *cnt)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > rows) return;
    if (t == rows) { cnt[rows] = 0; return; }
    const int64_t deg = row_ptr[row0 + t + 1] - row_ptr[row0 + t];
    if (deg > C && deg == Lfull) cnt[t] = int64_t(1) << 40; // full row: dense tiles
    else cnt[t] = deg > C ? (deg + C - 1) / C : 0;
}

__global__ void heavy_items_kernel(const int64_t *cnt_scanned, int64_t rows, int64_t *item_row, int32_t *item_chunk,
                                   int64_t *full_row)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t c0 = cnt_scanned[t], c1 = cnt_scanned[t + 1];
    if ((c1 >> 40) != (c0 >> 40)) full_row[c0 >> 40] = t;
    const int64_t b = c0 & kChunkMask, n = (c1 & kChunkMask) - b;
    for (int64_t c = 0; c < n; ++c) {
        item_row[b + c] = t;
        item_chunk[b + c] = (int32_t)c;
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(256) heavy_chunk_kernel(AttnParams p, const int64_t *cnt_scanned, const int64_t *item_row,
                                                          const int32_t *item_chunk, float *partials)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int H = p.H;
    const int64_t n_items = cnt_scanned[p.q_rows] & kChunkMask;
    if (gw >= n_items * H) return;
    const int64_t it = gw / H;
    const int h = (int)(gw - it * H);
    const int64_t t = item_row[it];
    const int64_t c = item_chunk[it];
    const int64_t i = p.q_begin + t;

    if constexpr (sizeof(T) == 2) { // mma.sync edge blocks (csr_mma.cuh)
        const int64_t rb = p.mask.row_ptr[i], deg = p.mask.row_ptr[i + 1] - rb;
        const int64_t kb = c * p.heavy_threshold;
        const int64_t ke = imin(kb + p.heavy_threshold, deg);
        csrmma::RowAcc<T, D> ra;
        ra.init(p, t, h, lane);
        ra.run(p, p.mask.col_idx + rb + kb, ke - kb, h, lane);
        float r[2 * csrmma::RowAcc<T, D>::KS];
        const float l = ra.finish(r);
        const int g = lane >> 2;
        float *dst = partials + ((size_t)it * H + h) * (D + 2);
        if (lane == 0) { dst[0] = ra.m; dst[1] = l; }
        if ((lane & 3) == 0) {
#pragma unroll
            for (int x = 0; x < 2 * csrmma::RowAcc<T, D>::KS; ++x) dst[2 + g * (D / 8) + x] = r[x];
        }
        return;
    }
    EdgeAcc<T, D, false> acc;
    acc.init(p, t, h, lane);
    const Piece P = get_piece(p.mask, i, 0);
    const int64_t kb = c * p.heavy_threshold;
    const int64_t ke = kb + p.heavy_threshold < P.count ? kb + p.heavy_threshold : P.count;
    acc.template run_csr<csr_depth<T, D>()>(P.cols + P.base, kb, ke);
    acc.merge_groups();
    if (acc.g == 0) {
        constexpr int PER = EdgeAcc<T, D, false>::PER;
        float *dst = partials + ((size_t)it * H + h) * (D + 2);
        if (acc.sub == 0) { dst[0] = acc.m; dst[1] = acc.l; }
#pragma unroll
        for (int e = 0; e < PER; ++e) dst[2 + acc.sub * PER + e] = acc.o[e];
    }
}

// one warp per (heavy row, head): lanes own d/32.. elements; combine chunk partials.
template <typename T, int D>
__global__ void __launch_bounds__(256) heavy_merge_kernel(AttnParams p, const int64_t *cnt_scanned, const int64_t *item_row,
                                                          const int32_t *item_chunk, const float *partials)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int H = p.H;
    const int64_t n_items = cnt_scanned[p.q_rows] & kChunkMask;
    if (gw >= n_items * H) return;
    const int64_t it0 = gw / H;
    const int h = (int)(gw - it0 * H);
    if (item_chunk[it0] != 0) return; // the row's first chunk owns the merge
    const int64_t t = item_row[it0];
    const int64_t nch = (cnt_scanned[t + 1] & kChunkMask) - (cnt_scanned[t] & kChunkMask);
    constexpr int PER = (D + 31) / 32;
    float m = -INFINITY, l = 0.f, o[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) o[e] = 0.f;
    for (int64_t c = 0; c < nch; ++c) {
        const float *src = partials + ((size_t)(it0 + c) * H + h) * (D + 2);
        const float m2 = src[0], l2 = src[1];
        const float mn = fmaxf(m, m2);
        const float a = (m == -INFINITY) ? 0.f : ex2(m - mn);
        const float b = (m2 == -INFINITY) ? 0.f : ex2(m2 - mn);
        l = l * a + l2 * b;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int col = lane + 32 * e;
            if (col < D) o[e] = o[e] * a + src[2 + col] * b;
        }
        m = mn;
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T *Op = reinterpret_cast<T *>(p.out) + ((size_t)t * H + h) * D;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
        const int col = lane + 32 * e;
        if (col < D) Op[col] = (T)(o[e] * inv);
    }
}

// Full rows: CTA = (64-row tile of the full-row list, 4096-key chunk, head); 4 warps x 16
// rows on mma.sync (tc::MmaRows), keys in 64-key cp.async stages (double-buffered).  Writes
// the partial (m, l, o~) of each (row, chunk) in natural dim order.
template <typename T, int D>
__global__ void __launch_bounds__(FULL_THREADS) full_rows_kernel(const __grid_constant__ AttnParams p,
                                                                 const int64_t *nfull_packed, const int64_t *full_row,
                                                                 int64_t ntiles, float *fpart)
{
    using G = tc::Geo<D>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int H = p.H;
    const int64_t nfull = *nfull_packed >> 40;
    const int64_t ch = blockIdx.x; // one CTA per (key chunk, head) walks the tiles of full rows
    const int h = (int)(blockIdx.y);
    (void)ntiles;
    // (a grid sized by the host's bound on the full-row count would launch mostly empty CTAs)
    for (int64_t tile = 0; tile * FULL_ROWS < nfull; ++tile) {
    const int nrows = (int)imin(FULL_ROWS, nfull - tile * FULL_ROWS);
    if (tile > 0) __syncthreads(); // the previous tile's shared buffers are free
    const int64_t NCH = full_chunks(p.mask.L);
    const int64_t k0 = ch * FULL_KCH, nkeys = imin((int64_t)FULL_KCH, p.mask.L - k0); // multiple of 16

    const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sK0 = sQ + FULL_ROWS * G::RB, sV0 = sK0 + 2 * FULL_KC * G::RB;
    const size_t row_bytes = (size_t)H * D * sizeof(T), hoff = (size_t)h * D * sizeof(T);

    for (int idx = tid; idx < FULL_ROWS * G::NC; idx += FULL_THREADS) {
        const int r = idx / G::NC, cc = idx % G::NC;
        if (r < nrows)
            tc::cp_async16(sQ + tc::swz<D>(r, cc), reinterpret_cast<const char *>(p.Q) +
                                                       (size_t)full_row[tile * FULL_ROWS + r] * row_bytes + hoff + cc * 16);
        else
            tc::sts_zero16(sQ + tc::swz<D>(r, cc)); // pad rows take part in the rescale vote
    }
    const int64_t nst = (nkeys + FULL_KC - 1) / FULL_KC;
    auto load_stage = [&](int64_t c, int st) {
        for (int idx = tid; idx < FULL_KC * G::NC; idx += FULL_THREADS) {
            const int kl = idx / G::NC, cc = idx % G::NC;
            const int64_t k = c * FULL_KC + kl;
            if (k < nkeys) {
                const char *kr, *vr;
                kv_row(p, k0 + k, row_bytes, kr, vr);
                tc::cp_async16(sK0 + st * FULL_KC * G::RB + tc::swz<D>(kl, cc), kr + hoff + cc * 16);
                tc::cp_async16(sV0 + st * FULL_KC * G::RB + tc::swz<D>(kl, cc), vr + hoff + cc * 16);
            }
        }
    };
    load_stage(0, 0);
    tc::cp_async_commit();
    if (nst > 1) load_stage(1, 1);
    tc::cp_async_commit();

    tc::MmaRows<T, D> st;
    st.init_empty();
    tc::cp_async_wait<1>();
    __syncthreads();
    st.load_q(sQ, warp * 16, lane);
    uint32_t kaddr[G::KS], vaddr[G::NB8 / 2];
    {
        const int krow = (lane & 7) + (lane >> 4) * 8, vrow = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int kk = 0; kk < G::KS; ++kk) kaddr[kk] = sK0 + tc::swz<D>(krow, 2 * kk + ((lane >> 3) & 1));
#pragma unroll
        for (int jj = 0; jj < G::NB8 / 2; ++jj) vaddr[jj] = sV0 + tc::swz<D>(vrow, 2 * jj + (lane >> 4));
    }
    const float sl2 = p.scale_log2;
    for (int64_t c = 0; c < nst; ++c) {
        const int stg = (int)(c & 1);
        if (c > 0) {
            tc::cp_async_wait<1>();
            __syncthreads();
        }
        const int blocks_here = (int)imin(FULL_KC / 16, (nkeys - c * FULL_KC) / 16);
        const uint32_t soff = (uint32_t)(stg * FULL_KC * G::RB);
        int b = 0;
        for (; b + 1 < blocks_here; b += 2) st.block16x2(kaddr, vaddr, soff + b * 16 * G::RB, soff + (b + 1) * 16 * G::RB, sl2);
        if (b < blocks_here) st.block16(kaddr, vaddr, soff + b * 16 * G::RB, sl2);
        __syncthreads();
        if (c + 2 < nst) load_stage(c + 2, stg);
        tc::cp_async_commit();
    }
    tc::cp_async_wait<0>();
    st.reduce_l();
    const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int r = warp * 16 + g + 8 * hr;
        if (r >= nrows) continue;
        float *dst = fpart + (((size_t)(tile * FULL_ROWS + r) * NCH + ch) * H + h) * (D + 2);
        if (t4 == 0) { dst[0] = st.mr[hr]; dst[1] = st.lr[hr]; }
#pragma unroll
        for (int j = 0; j < G::NB8; ++j) {
            dst[2 + 8 * j + 2 * t4] = st.o[j][2 * hr];
            dst[2 + 8 * j + 2 * t4 + 1] = st.o[j][2 * hr + 1];
        }
    }
    }
}

// one warp per (full row, head): (+)-merge its NCH chunk partials, normalise, store
template <typename T, int D>
__global__ void __launch_bounds__(256) full_merge_kernel(const __grid_constant__ AttnParams p,
                                                         const int64_t *nfull_packed, const int64_t *full_row,
                                                         const float *fpart)
{
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int H = p.H;
    const int64_t nfull = *nfull_packed >> 40;
    if (gw >= nfull * H) return;
    const int64_t f = gw / H;
    const int h = (int)(gw - f * H);
    const int64_t NCH = full_chunks(p.mask.L);
    constexpr int PER = (D + 31) / 32;
    float m = -INFINITY, l = 0.f, o[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) o[e] = 0.f;
    for (int64_t c = 0; c < NCH; ++c) {
        const float *src = fpart + (((size_t)f * NCH + c) * H + h) * (D + 2);
        const float m2 = src[0], l2 = src[1];
        const float mn = fmaxf(m, m2);
        const float a = (m == -INFINITY) ? 0.f : ex2(m - mn);
        const float b = (m2 == -INFINITY) ? 0.f : ex2(m2 - mn);
        l = l * a + l2 * b;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int col = lane + 32 * e;
            if (col < D) o[e] = o[e] * a + src[2 + col] * b;
        }
        m = mn;
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T *Op = reinterpret_cast<T *>(p.out) + ((size_t)full_row[f] * H + h) * D;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
        const int col = lane + 32 * e;
        if (col < D) Op[col] = (T)(o[e] * inv);
    }
}

// nfull_packed: DEVICE int64 whose bits 40-63 hold the number of full rows (the last entry of
// the scanned heavy-row counts, or a count written by the BigBird prep kernel); full_row:
// their local query rows; F: a host upper bound on that number
template <typename T, int D>
static ga_status launch_full_t(const AttnParams &p, const int64_t *nfull_packed, const int64_t *full_row, float *fpart,
                               int64_t F, cudaStream_t s)
{
    if (F == 0) return GA_OK;
    using G = tc::Geo<D>;
    const int64_t ntiles = (F + FULL_ROWS - 1) / FULL_ROWS, NCH = full_chunks(p.mask.L);
    const uint32_t smem = FULL_ROWS * G::RB + 4 * FULL_KC * G::RB;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(full_rows_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    full_rows_kernel<T, D><<<dim3((unsigned)NCH, (unsigned)p.H), FULL_THREADS, smem, s>>>(p, nfull_packed, full_row,
                                                                                          ntiles, fpart);
    GA_CHECK_LAUNCH("full_rows_kernel");
    full_merge_kernel<T, D><<<(unsigned)((F * p.H + 7) / 8), 256, 0, s>>>(p, nfull_packed, full_row, fpart);
    GA_CHECK_LAUNCH("full_merge_kernel");
    return GA_OK;
}

template <typename T, int D>
static ga_status launch_heavy_t(const AttnParams &p, int64_t *cnt, int64_t *item_row, int32_t *item_chunk,
                                float *partials, int64_t I, const int64_t *full_row, float *fpart, int64_t F,
                                cudaStream_t s)
{
    if constexpr (sizeof(T) == 2) {
        const ga_status st = launch_full_t<T, D>(p, cnt + p.q_rows, full_row, fpart, F, s);
        if (st != GA_OK) return st;
    }
    const int64_t warps = I * p.H;
    const int64_t blocks = (warps + 7) / 8;
    heavy_chunk_kernel<T, D><<<(unsigned)blocks, 256, 0, s>>>(p, cnt, item_row, item_chunk, partials);
    GA_CHECK_LAUNCH("heavy_chunk_kernel");
    heavy_merge_kernel<T, D><<<(unsigned)blocks, 256, 0, s>>>(p, cnt, item_row, item_chunk, partials);
    GA_CHECK_LAUNCH("heavy_merge_kernel");
    return GA_OK;
}

template <typename T>
static ga_status launch_heavy_d(const AttnParams &p, int64_t *cnt, int64_t *ir, int32_t *ic, float *part, int64_t I,
                                const int64_t *fr, float *fp, int64_t F, cudaStream_t s)
{
    switch (p.d) {
    case 32: return launch_heavy_t<T, 32>(p, cnt, ir, ic, part, I, fr, fp, F, s);
    case 64: return launch_heavy_t<T, 64>(p, cnt, ir, ic, part, I, fr, fp, F, s);
    case 128: return launch_heavy_t<T, 128>(p, cnt, ir, ic, part, I, fr, fp, F, s);
    }
    set_error("d=%d unsupported", p.d);
    return GA_ERR_UNSUPPORTED;
}

size_t full_rows_partials_bytes(int64_t F, int64_t Lm, int32_t H, int32_t d)
{
    return sizeof(float) * (size_t)F * full_chunks(Lm) * H * (d + 2);
}

ga_status launch_full_rows(const AttnParams &p, ga_dtype dt, const int64_t *nfull_packed, const int64_t *full_row,
                           float *fpart, int64_t F, cudaStream_t s)
{
    if (dt == GA_F32 || p.mask.L % 16 != 0) {
        set_error("full-row tiles need bf16/fp16 and L %% 16 == 0");
        return GA_ERR_UNSUPPORTED;
    }
    switch (p.d) {
    case 32: return dt == GA_BF16 ? launch_full_t<__nv_bfloat16, 32>(p, nfull_packed, full_row, fpart, F, s)
                                  : launch_full_t<__half, 32>(p, nfull_packed, full_row, fpart, F, s);
    case 64: return dt == GA_BF16 ? launch_full_t<__nv_bfloat16, 64>(p, nfull_packed, full_row, fpart, F, s)
                                  : launch_full_t<__half, 64>(p, nfull_packed, full_row, fpart, F, s);
    case 128: return dt == GA_BF16 ? launch_full_t<__nv_bfloat16, 128>(p, nfull_packed, full_row, fpart, F, s)
                                   : launch_full_t<__half, 128>(p, nfull_packed, full_row, fpart, F, s);
    }
    set_error("d=%d unsupported", p.d);
    return GA_ERR_UNSUPPORTED;
}

ga_status launch_csr_heavy(const AttnParams &p, ga_dtype dt, void *ws, size_t ws_bytes, cudaStream_t s)
{
    const int64_t C = p.heavy_threshold;
    const int64_t rows = p.q_rows;
    const int64_t I = max_items(p.nnz, C);
    const int64_t Lm = p.mask.L;
    const size_t need = csr_heavy_workspace(rows, Lm, p.nnz, p.H, p.d, C);
    if (ws == nullptr || ws_bytes < need) {
        set_error("CSR heavy-row split needs %zu workspace bytes (got %zu); see ga_workspace_size", need, ws_bytes);
        return GA_ERR_OOM;
    }
    char *w = reinterpret_cast<char *>(ws);
    int64_t *cnt = reinterpret_cast<int64_t *>(w);
    w += align256(sizeof(int64_t) * (rows + 1));
    int64_t *item_row = reinterpret_cast<int64_t *>(w);
    w += align256(sizeof(int64_t) * I);
    int32_t *item_chunk = reinterpret_cast<int32_t *>(w);
    w += align256(sizeof(int32_t) * I);
    float *partials = reinterpret_cast<float *>(w);
    w += align256(sizeof(float) * (size_t)I * p.H * (p.d + 2));
    int64_t *full_row = reinterpret_cast<int64_t *>(w);
    const int64_t F = max_full(rows, Lm, p.nnz);
    w += align256(sizeof(int64_t) * F);
    float *fpart = reinterpret_cast<float *>(w);
    // dense full-row tiles: bf16/fp16 with whole 16-key blocks
    const bool full = dt != GA_F32 && Lm % 16 == 0 && F > 0;

    heavy_count_kernel<<<(unsigned)((rows + 1 + 255) / 256), 256, 0, s>>>(p.mask.row_ptr, p.q_begin, rows, C,
                                                                          full ? Lm : -1, cnt);
    GA_CHECK_LAUNCH("heavy_count_kernel");
    ga_status st = scan_exclusive_i64(cnt, rows + 1, s);
    if (st != GA_OK) return st;
    heavy_items_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(cnt, rows, item_row, item_chunk, full_row);
    GA_CHECK_LAUNCH("heavy_items_kernel");
    switch (dt) {
    case GA_F32: return launch_heavy_d<float>(p, cnt, item_row, item_chunk, partials, I, nullptr, nullptr, 0, s);
    case GA_BF16:
        return launch_heavy_d<__nv_bfloat16>(p, cnt, item_row, item_chunk, partials, I, full_row, fpart, full ? F : 0, s);
    case GA_F16: return launch_heavy_d<__half>(p, cnt, item_row, item_chunk, partials, I, full_row, fpart, full ? F : 0, s);
    }
    set_error("unknown dtype");
    return GA_ERR_INVALID_ARG;
}

} // namespace ga

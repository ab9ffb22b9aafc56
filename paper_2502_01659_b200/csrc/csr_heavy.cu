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
// scan -> item table (row, chunk) -> chunk kernel -> merge kernel.
//
// Workspace layout (csr_heavy_workspace):  cnt int64 [L+1] | item_row int64 [I] |
// item_chunk int32 [I] | partials f32 [I * H * (d+2)],  I = 2*nnz/C + 1 >= sum of chunks.
#include "edge_core.cuh"

namespace ga {

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static int64_t max_items(int64_t nnz, int64_t C) { return 2 * (nnz / C) + 2; }

size_t csr_heavy_workspace(int64_t L, int64_t nnz, int32_t H, int32_t d, int64_t C)
{
    const int64_t I = max_items(nnz, C);
    return align256(sizeof(int64_t) * (L + 1)) + align256(sizeof(int64_t) * I) + align256(sizeof(int32_t) * I) +
           align256(sizeof(float) * (size_t)I * H * (d + 2));
}

__global__ void heavy_count_kernel(const int64_t *row_ptr, int64_t row0, int64_t rows, int64_t C, int64_t *cnt)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > rows) return;
    if (t == rows) { cnt[rows] = 0; return; }
    const int64_t deg = row_ptr[row0 + t + 1] - row_ptr[row0 + t];
    cnt[t] = deg > C ? (deg + C - 1) / C : 0;
}

__global__ void heavy_items_kernel(const int64_t *cnt_scanned, int64_t rows, int64_t *item_row, int32_t *item_chunk)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows) return;
    const int64_t b = cnt_scanned[t], n = cnt_scanned[t + 1] - b;
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
    const int64_t n_items = cnt_scanned[p.q_rows];
    if (gw >= n_items * H) return;
    const int64_t it = gw / H;
    const int h = (int)(gw - it * H);
    const int64_t t = item_row[it];
    const int64_t c = item_chunk[it];
    const int64_t i = p.q_begin + t;

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
    const int64_t n_items = cnt_scanned[p.q_rows];
    if (gw >= n_items * H) return;
    const int64_t it0 = gw / H;
    const int h = (int)(gw - it0 * H);
    if (item_chunk[it0] != 0) return; // the row's first chunk owns the merge
    const int64_t t = item_row[it0];
    const int64_t nch = cnt_scanned[t + 1] - cnt_scanned[t];
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

template <typename T, int D>
static ga_status launch_heavy_t(const AttnParams &p, int64_t *cnt, int64_t *item_row, int32_t *item_chunk,
                                float *partials, int64_t I, cudaStream_t s)
{
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
                                cudaStream_t s)
{
    switch (p.d) {
    case 32: return launch_heavy_t<T, 32>(p, cnt, ir, ic, part, I, s);
    case 64: return launch_heavy_t<T, 64>(p, cnt, ir, ic, part, I, s);
    case 128: return launch_heavy_t<T, 128>(p, cnt, ir, ic, part, I, s);
    }
    set_error("d=%d unsupported", p.d);
    return GA_ERR_UNSUPPORTED;
}

ga_status launch_csr_heavy(const AttnParams &p, ga_dtype dt, void *ws, size_t ws_bytes, cudaStream_t s)
{
    const int64_t C = p.heavy_threshold;
    const int64_t rows = p.q_rows;
    const int64_t I = max_items(p.nnz, C);
    const size_t need = csr_heavy_workspace(rows, p.nnz, p.H, p.d, C);
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

    heavy_count_kernel<<<(unsigned)((rows + 1 + 255) / 256), 256, 0, s>>>(p.mask.row_ptr, p.q_begin, rows, C, cnt);
    GA_CHECK_LAUNCH("heavy_count_kernel");
    ga_status st = scan_exclusive_i64(cnt, rows + 1, s);
    if (st != GA_OK) return st;
    heavy_items_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(cnt, rows, item_row, item_chunk);
    GA_CHECK_LAUNCH("heavy_items_kernel");
    switch (dt) {
    case GA_F32: return launch_heavy_d<float>(p, cnt, item_row, item_chunk, partials, I, s);
    case GA_BF16: return launch_heavy_d<__nv_bfloat16>(p, cnt, item_row, item_chunk, partials, I, s);
    case GA_F16: return launch_heavy_d<__half>(p, cnt, item_row, item_chunk, partials, I, s);
    }
    set_error("unknown dtype");
    return GA_ERR_INVALID_ARG;
}

} // namespace ga

// maskgen.cu — mask/graph generator, CSR validation, int64 scan and
// the seeded input generator (a0).
//
// Pattern -> CSR in three device passes, the way the paper's verification converts a mask
// "into the desired sparse matrix representation":
//   1. degree:  row_ptr[i] = |N(i)| from the closed forms (masks.cuh), row_ptr[L] = 0
//   2. scan:    exclusive prefix sum in place -> row_ptr[L] = nnz
//   3. fill:    col_idx[row_ptr[i] ..] = N(i) ascending (binary CSR, reading R7)
// BigBird random columns follow the counter-hash rejection rule of reading R10 so the CPU
// oracle and this generator agree bit for bit.
#include "common.cuh"

namespace ga {

// ------------------------------------------------------------------ scan (3 phase)
static constexpr int SCAN_THREADS = 256;
static constexpr int SCAN_ITEMS = 8;
static constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t *total)
{
    __shared__ int64_t warp_sums[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t s = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += y;
        }
        if (lane < SCAN_THREADS / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    const int64_t warp_prefix = wid > 0 ? warp_sums[wid - 1] : 0;
    *total = warp_sums[SCAN_THREADS / 32 - 1];
    __syncthreads();
    return warp_prefix + x - v;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(const int64_t *data, int64_t n, int64_t *sums)
{
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
        if (base + k < n) s += data[base + k];
    int64_t total;
    block_exclusive_scan(s, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_sums_kernel(int64_t *sums, int64_t nb)
{
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += SCAN_TILE) {
        const int64_t base = b0 + threadIdx.x * SCAN_ITEMS;
        int64_t v[SCAN_ITEMS], s = 0;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            v[k] = base + k < nb ? sums[base + k] : 0;
            s += v[k];
        }
        int64_t total;
        int64_t ex = block_exclusive_scan(s, &total) + carry;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            if (base + k < nb) sums[base + k] = ex;
            ex += v[k];
        }
        carry += total;
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) scan_apply_kernel(int64_t *data, int64_t n, const int64_t *sums)
{
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS], s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        v[k] = base + k < n ? data[base + k] : 0;
        s += v[k];
    }
    int64_t total;
    int64_t ex = block_exclusive_scan(s, &total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if (base + k < n) data[base + k] = ex;
        ex += v[k];
    }
}

ga_status scan_exclusive_i64(int64_t *data, int64_t n, cudaStream_t s)
{
    if (n <= 0) return GA_OK;
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    int64_t *sums = nullptr;
    cudaError_t e = scratch_alloc((void **)&sums, sizeof(int64_t) * nb, s);
    if (e != cudaSuccess) return cuda_fail(e, "scan: scratch allocation");
    scan_reduce_kernel<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(data, n, sums);
    scan_sums_kernel<<<1, SCAN_THREADS, 0, s>>>(sums, nb);
    scan_apply_kernel<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(data, n, sums);
    e = scratch_free(sums, s);
    if (e != cudaSuccess) return cuda_fail(e, "scan: cudaFreeAsync");
    note_launches(2); // + 1 below: three scan kernels
    GA_CHECK_LAUNCH("scan kernels");
    return GA_OK;
}

// ------------------------------------------------------------------ degrees
__global__ void degree_kernel(DevMask M, int64_t *row_ptr)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > M.L) return;
    if (i == M.L) { row_ptr[M.L] = 0; return; }
    row_ptr[i] = M.kind == K_BIGBIRD ? bb_degree(M, i) : degree(M, i);
}

// ------------------------------------------------------------------ fill
// Window / block-dilated: one ascending piece; a warp per row writes it coalesced.
// LongNet: s+1 ascending pieces merged (k-way, small s) by lane 0.
static constexpr int MAX_PIECES = 64;

__global__ void fill_pieces_kernel(DevMask M, const int64_t *row_ptr, int32_t *col_idx)
{
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= M.L) return;
    int32_t *dst = col_idx + row_ptr[i];
    const int np = num_pieces(M, i);
    if (np == 1) {
        const Piece P = get_piece(M, i, 0);
        for (int64_t k = lane; k < P.count; k += 32) dst[k] = (int32_t)piece_at(P, k);
        return;
    }
    if (lane != 0 || np == 0) return;
    Piece P[MAX_PIECES];
    int64_t cur[MAX_PIECES];
    for (int pc = 0; pc < np; ++pc) { P[pc] = get_piece(M, i, pc); cur[pc] = 0; }
    int64_t n = 0;
    for (;;) {
        int best = -1;
        int64_t bj = 0;
        for (int pc = 0; pc < np; ++pc) {
            if (cur[pc] >= P[pc].count) continue;
            const int64_t j = piece_at(P[pc], cur[pc]);
            if (best < 0 || j < bj) { best = pc; bj = j; }
        }
        if (best < 0) break;
        dst[n++] = (int32_t)bj;
        cur[best]++;
    }
}

// BigBird: warp per row, columns ascending, restricted to the selected components
// (bit 0 window W_i, bit 1 global rows/cols minus W_i, bit 2 random; reading R8-R10).
// Global rows and rows whose complement of W_i U G is exhausted use a membership filter
// over all j, warp-compacted in order; the others merge window, globals outside W_i and the
// random columns drawn by lane 0 (reading R10), all ascending.
static constexpr int MAX_RANDOM = 320;

__global__ void fill_bigbird_kernel(DevMask M, const int64_t *row_ptr, int32_t *col_idx)
{
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= M.L) return;
    const int parts = M.parts ? M.parts : 7;
    int32_t *dst = col_idx + row_ptr[i];
    const bool glob = bb_is_global(M, i);
    const bool exhausted = !glob && M.L - bb_wg(M, i) <= M.nrand;
    if (glob || exhausted) {
        int64_t out = 0;
        for (int64_t j0 = 0; j0 < M.L; j0 += 32) {
            const int64_t j = j0 + lane;
            bool inc = false;
            if (j < M.L) {
                const bool w = bb_in_window(M, i, j);
                if (glob) inc = w ? (parts & 1) : (parts & 2);
                else inc = w ? (parts & 1) : bb_is_global(M, j) ? (parts & 2) : (parts & 4);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, inc);
            if (inc) dst[out + __popc(bal & ((1u << lane) - 1u))] = (int32_t)j;
            out += __popc(bal);
        }
        return;
    }
    if (lane != 0) return;
    int64_t R[MAX_RANDOM];
    int n = 0;
    if (parts & 4) {
        const uint64_t base = splitmix64(M.seed);
        for (uint64_t t = 0; n < M.nrand; ++t) {
            const int64_t c = bb_candidate(M, base, i, t);
            if (bb_in_window(M, i, c)) continue;
            if (bb_is_global(M, c)) continue;
            bool dup = false;
            for (int q = 0; q < n; ++q)
                if (R[q] == c) { dup = true; break; }
            if (dup) continue;
            // insertion keeps R sorted
            int q = n++;
            while (q > 0 && R[q - 1] > c) { R[q] = R[q - 1]; --q; }
            R[q] = c;
        }
    }
    // 3-way merge: window W_i (step r), globals outside W_i, random R
    int64_t wj = INT64_MAX, whi = -1;
    if (parts & 1) {
        wj = i - imin(i, M.w - 1) / M.r * M.r;
        whi = i + imin(M.L - 1 - i, M.w - 1) / M.r * M.r;
    }
    int64_t out = 0, gk = 0, rk = 0;
    auto next_g = [&](int64_t &k) -> int64_t {
        if (!(parts & 2)) return INT64_MAX;
        while (k < M.ng) {
            const int64_t gv = bb_global_at(M, k);
            if (!bb_in_window(M, i, gv)) return gv;
            ++k;
        }
        return INT64_MAX;
    };
    int64_t gv = next_g(gk);
    for (;;) {
        const int64_t a = wj <= whi ? wj : INT64_MAX;
        const int64_t r = rk < n ? R[rk] : INT64_MAX;
        int64_t v = a;
        if (gv < v) v = gv;
        if (r < v) v = r;
        if (v == INT64_MAX) break;
        dst[out++] = (int32_t)v;
        if (v == a) wj += M.r;
        else if (v == gv) { ++gk; gv = next_g(gk); }
        else ++rk;
    }
}

ga_status maskgen_to_csr(const DevMask &M, int64_t *row_ptr, int32_t *col_idx, cudaStream_t s)
{
    // a row draws min(n_random, L - |W_i U G|) columns and |W_i| >= w, so only patterns that
    // can draw more than MAX_RANDOM columns for some row are rejected
    if (M.kind == K_BIGBIRD && M.nrand > MAX_RANDOM && M.L - M.w > MAX_RANDOM) {
        set_error("n_random=%lld exceeds %d", (long long)M.nrand, MAX_RANDOM);
        return GA_ERR_UNSUPPORTED;
    }
    if (M.kind == K_LONGNET && M.K + 1 > MAX_PIECES) {
        set_error("LongNet with %lld levels exceeds %d", (long long)(M.K + 1), MAX_PIECES);
        return GA_ERR_UNSUPPORTED;
    }
    degree_kernel<<<(unsigned)((M.L + 1 + 255) / 256), 256, 0, s>>>(M, row_ptr);
    GA_CHECK_LAUNCH("degree_kernel");
    ga_status st = scan_exclusive_i64(row_ptr, M.L + 1, s);
    if (st != GA_OK) return st;
    if (col_idx == nullptr) return GA_OK;
    const unsigned blocks = (unsigned)((M.L * 32 + 255) / 256);
    if (M.kind == K_BIGBIRD)
        fill_bigbird_kernel<<<blocks, 256, 0, s>>>(M, row_ptr, col_idx);
    else
        fill_pieces_kernel<<<blocks, 256, 0, s>>>(M, row_ptr, col_idx);
    GA_CHECK_LAUNCH("fill kernel");
    return GA_OK;
}

// ------------------------------------------------------------------ validation
__global__ void validate_kernel(DevMask M, int *bad)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M.L) {
        if (i == M.L && (M.row_ptr[0] != 0 || M.row_ptr[M.L] != M.nnz)) atomicExch(bad, 1);
        return;
    }
    const int64_t b = M.row_ptr[i], e = M.row_ptr[i + 1];
    if (e < b || b < 0 || e > M.nnz) { atomicExch(bad, 1); return; }
    int64_t prev = -1;
    for (int64_t k = b; k < e; ++k) {
        const int64_t c = M.col_idx[k];
        if (c <= prev || c >= M.L) { atomicExch(bad, 1); return; }
        prev = c;
    }
}

ga_status mask_validate(const DevMask &M, cudaStream_t s, int *ok)
{
    int *bad = nullptr;
    cudaError_t e = scratch_alloc((void **)&bad, sizeof(int), s);
    if (e != cudaSuccess) return cuda_fail(e, "validate: scratch allocation");
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    validate_kernel<<<(unsigned)((M.L + 1 + 255) / 256), 256, 0, s>>>(M, bad);
    GA_CHECK_LAUNCH("validate_kernel");
    int h = 1;
    cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    scratch_free(bad, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "validate: sync");
    *ok = h == 0;
    if (h != 0) {
        set_error("CSR mask is malformed (row_ptr/col_idx invariants S:97-98)");
        return GA_ERR_MASK;
    }
    return GA_OK;
}

// ------------------------------------------------------------------ inputs (a0, R22)
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half from_f32<__half>(float x) { return __float2half_rn(x); }

template <typename T>
__global__ void fill_inputs_kernel(T *dst, int64_t n, uint64_t base, uint64_t e0, float shift)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const uint64_t u = splitmix64(base ^ (e0 + (uint64_t)t));
        const float x = (float)(u >> 40) * (1.0f / 16777216.0f) + shift;
        dst[t] = from_f32<T>(x);
    }
}

ga_status fill_inputs(void *dst, ga_dtype dt, int64_t n, uint64_t seed, int32_t tensor, int64_t e0, float shift,
                      cudaStream_t s)
{
    if (n <= 0) return GA_OK;
    const uint64_t base = splitmix64(seed + (uint64_t)tensor);
    const unsigned blocks = (unsigned)(n / 256 + 1 < 148 * 32 ? n / 256 + 1 : 148 * 32);
    switch (dt) {
    case GA_F32: fill_inputs_kernel<float><<<blocks, 256, 0, s>>>((float *)dst, n, base, (uint64_t)e0, shift); break;
    case GA_BF16:
        fill_inputs_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>((__nv_bfloat16 *)dst, n, base, (uint64_t)e0, shift);
        break;
    case GA_F16: fill_inputs_kernel<__half><<<blocks, 256, 0, s>>>((__half *)dst, n, base, (uint64_t)e0, shift); break;
    default: set_error("unknown dtype"); return GA_ERR_INVALID_ARG;
    }
    GA_CHECK_LAUNCH("fill_inputs_kernel");
    return GA_OK;
}

} // namespace ga

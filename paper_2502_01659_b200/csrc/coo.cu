// coo.cu — COO edge list -> binary CSR on the device (the
// paper's COO mask storage).  The paper's COO kernel searches each row's entries in the
// list (P:370's row search dominates); here COO is an input format only, converted once:
//
//   key[e] = row[e] * L + col[e]    (range-checked: 0 <= row, col < L, else GA_ERR_MASK)
//   radix sort of the keys (CUB), unique (a binary mask counts an edge once, reading R7)
//   col_idx[k] = ukey[k] mod L,  row_ptr[r] = lower_bound(ukey, r * L)
//
// The result is the unique sorted CSR of the edge set, so it equals the CPU conversion bit
// for bit regardless of the input order.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"

namespace ga {

__global__ void coo_keys_kernel(const int32_t *rows, const int32_t *cols, int64_t n, int64_t L, int64_t *keys,
                                int *bad)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rows[e], c = cols[e];
        if (r < 0 || r >= L || c < 0 || c >= L) {
            *bad = 1;
            keys[e] = 0;
        } else {
            keys[e] = r * L + c;
        }
    }
}

__global__ void coo_cols_kernel(const int64_t *ukeys, const int64_t *nsel, int64_t L, int32_t *col_idx)
{
    const int64_t n = *nsel;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        col_idx[e] = (int32_t)(ukeys[e] % L);
}

__global__ void coo_rowptr_kernel(const int64_t *ukeys, const int64_t *nsel, int64_t L, int64_t *row_ptr)
{
    const int64_t n = *nsel;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= L; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t key = r * L; // first key of row r
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ukeys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        row_ptr[r] = lo;
    }
}

} // namespace ga

using namespace ga;

extern "C" ga_status ga_coo_to_csr(int64_t L, const int32_t *rows, const int32_t *cols, int64_t n, int64_t *row_ptr,
                                   int32_t *col_idx, int64_t *nnz_out, void *stream)
{
    if (L <= 0 || L > INT32_MAX || n < 0 || !row_ptr || !nnz_out || (n > 0 && (!rows || !cols || !col_idx))) {
        set_error("ga_coo_to_csr: bad arguments (L=%lld, n=%lld)", (long long)L, (long long)n);
        return GA_ERR_INVALID_ARG;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n1 = n > 0 ? n : 1;
    // key bits: L*L - 1 < 2^end_bit
    int end_bit = 1;
    while (end_bit < 63 && ((uint64_t)1 << end_bit) < (uint64_t)L * (uint64_t)L) ++end_bit;
    size_t sort_bytes = 0, uniq_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (const int64_t *)nullptr, (int64_t *)nullptr, n1, 0, end_bit,
                                   s);
    cub::DeviceSelect::Unique(nullptr, uniq_bytes, (const int64_t *)nullptr, (int64_t *)nullptr, (int64_t *)nullptr,
                              n1, s);
    const size_t tmp_bytes = sort_bytes > uniq_bytes ? sort_bytes : uniq_bytes;
    char *buf = nullptr;
    const size_t kb = (size_t)n1 * sizeof(int64_t);
    cudaError_t e = scratch_alloc(reinterpret_cast<void **>(&buf), 2 * kb + 256 + tmp_bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "ga_coo_to_csr scratch");
    int64_t *keys = reinterpret_cast<int64_t *>(buf), *sorted = reinterpret_cast<int64_t *>(buf + kb);
    int64_t *nsel = reinterpret_cast<int64_t *>(buf + 2 * kb);
    int *bad = reinterpret_cast<int *>(buf + 2 * kb + 8);
    void *tmp = buf + 2 * kb + 256;
    ga_status st = GA_OK;
    int h_bad = 0;
    int64_t h_n = 0;
    do {
        if ((e = cudaMemsetAsync(buf + 2 * kb, 0, 16, s)) != cudaSuccess) { st = cuda_fail(e, "memset"); break; }
        if (n > 0) {
            const unsigned blocks = (unsigned)imin((n + 255) / 256, 148 * 32);
            coo_keys_kernel<<<blocks, 256, 0, s>>>(rows, cols, n, L, keys, bad);
            note_launches(1);
            size_t tb = tmp_bytes;
            if ((e = cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, n, 0, end_bit, s)) != cudaSuccess) {
                st = cuda_fail(e, "radix sort");
                break;
            }
            tb = tmp_bytes;
            if ((e = cub::DeviceSelect::Unique(tmp, tb, sorted, keys, nsel, n, s)) != cudaSuccess) {
                st = cuda_fail(e, "unique");
                break;
            }
            coo_cols_kernel<<<blocks, 256, 0, s>>>(keys, nsel, L, col_idx);
            note_launches(1);
        }
        coo_rowptr_kernel<<<(unsigned)imin((L + 256) / 256, 148 * 32), 256, 0, s>>>(keys, nsel, L, row_ptr);
        note_launches(1);
        if ((e = cudaPeekAtLastError()) != cudaSuccess) { st = cuda_fail(e, "coo kernels"); break; }
        if ((e = cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaMemcpyAsync(&h_n, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaStreamSynchronize(s)) != cudaSuccess) {
            st = cuda_fail(e, "coo readback");
            break;
        }
    } while (0);
    scratch_free(buf, s);
    if (st != GA_OK) return st;
    if (h_bad) {
        set_error("ga_coo_to_csr: an edge index lies outside [0, L)");
        return GA_ERR_MASK;
    }
    *nnz_out = h_n;
    return GA_OK;
}

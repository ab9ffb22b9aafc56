// tma.cu — host-side tensor-map encoding (driver entry point resolved through cudart, so
// libga.so needs no libcuda link).
#include <cuda_runtime.h>

#include <mutex>

#include "tma.cuh"

namespace ga {
namespace tma {

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encoder()
{
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    });
    return fn;
}

struct Key {
    const void *base;
    int64_t ntok;
    int H, D, r, box;
    bool operator==(const Key &o) const
    {
        return base == o.base && ntok == o.ntok && H == o.H && D == o.D && r == o.r && box == o.box;
    }
};

static bool encode_uncached(CUtensorMap *map, const void *base, int64_t ntok, int H, int D, int r, int box_rows);
static bool encode_gather_uncached(CUtensorMap *map, const void *base, int64_t ntok, int H, int D);

// Encoding is host work on every launch; a cache keyed by (buffer, shape, stride, box)
// serves the repeated launches of a training / serving loop.  64 entries: the host pipeline
// (8 chunks x Q/out maps + K/V) and a few device-path callers fit without evicting each other.
static const int kCache = 64;
bool encode_rows(CUtensorMap *map, const void *base, int64_t ntok, int H, int D, int r, int box_rows)
{
    static std::mutex mu;
    static Key keys[kCache];
    static CUtensorMap maps[kCache];
    static int n = 0, next = 0;
    const Key k{base, ntok, H, D, r, box_rows};
    {
        std::lock_guard<std::mutex> g(mu);
        for (int i = 0; i < n; ++i)
            if (keys[i] == k) { *map = maps[i]; return true; }
    }
    const bool ok = r == 0  ? encode_gather_uncached(map, base, ntok, H, D)
                    : r < 0 ? encode_lattice(map, base, ntok, H, D, 1, -r) // contiguous rows, box -r
                            : encode_uncached(map, base, ntok, H, D, r, box_rows);
    if (!ok) return false;
    std::lock_guard<std::mutex> g(mu);
    keys[next] = k;
    maps[next] = *map;
    next = (next + 1) % kCache;
    if (n < kCache) ++n;
    return true;
}

static bool encode_uncached(CUtensorMap *map, const void *base, int64_t ntok, int H, int D, int r, int box_rows)
{
    const int rb = D * 2;
    if ((rb != 128 && rb != 64) || r < 1 || r > 8 || box_rows * r > 256 || ntok <= 0 || ntok >= (int64_t)1 << 32)
        return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0) return false;
    EncodeTiled enc = encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)ntok};
    const cuuint64_t strides[2] = {(cuuint64_t)rb, (cuuint64_t)H * rb}; // bytes, dims 1 and 2
    const cuuint32_t box[3] = {(cuuint32_t)D, 1u, (cuuint32_t)(box_rows * r)};
    const cuuint32_t estr[3] = {1u, 1u, (cuuint32_t)r};
    const CUresult e = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return e == CUDA_SUCCESS;
}

} // namespace tma
} // namespace ga

namespace ga {
namespace tma {

// 2D view {H*D elements, ntok rows} with a {D, 1} box (one (token, head) row): the box of a
// tile::gather4 load, which fetches 4 such rows at arbitrary token coordinates
static bool encode_gather_uncached(CUtensorMap *map, const void *base, int64_t ntok, int H, int D)
{
    const int rb = D * 2;
    if (rb != 128 || ntok <= 0 || ntok >= (int64_t)1 << 31) return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0) return false;
    EncodeTiled enc = encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)H * D, (cuuint64_t)ntok};
    const cuuint64_t strides[1] = {(cuuint64_t)H * rb};
    const cuuint32_t box[2] = {(cuuint32_t)D, 1u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult e = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void *>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return e == CUDA_SUCCESS;
}

bool encode_gather(CUtensorMap *map, const void *base, int64_t ntok, int H, int D)
{
    return encode_rows(map, base, ntok, H, D, 0, 0);
}

bool encode_block(CUtensorMap *map, const void *base, int64_t ntok, int H, int D, int box_rows)
{
    return encode_rows(map, base, ntok, H, D, -box_rows, 0);
}

} // namespace tma
} // namespace ga

namespace ga {
namespace tma {

bool encode_lattice(CUtensorMap *map, const void *base, int64_t nrows, int H, int D, int64_t pitch, int box_rows)
{
    const int rb = D * 2;
    if (rb != 128 || nrows <= 0 || nrows >= (int64_t)1 << 32 || pitch < 1 || box_rows < 1 || box_rows > 256) return false;
    const uint64_t gstride = (uint64_t)pitch * H * rb;
    if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0 || gstride >= (uint64_t)1 << 40) return false;
    EncodeTiled enc = encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)nrows};
    const cuuint64_t strides[2] = {(cuuint64_t)rb, (cuuint64_t)gstride};
    const cuuint32_t box[3] = {(cuuint32_t)D, 1u, (cuuint32_t)box_rows};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

} // namespace tma
} // namespace ga

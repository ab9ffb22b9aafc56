// common.cuh — dtype traits, 16-byte vector conversion, fast exp2, error plumbing.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ga.h"
#include "masks.cuh"

namespace ga {

// ---------------------------------------------------------------- error plumbing
void set_error(const char *fmt, ...);
ga_status cuda_fail(cudaError_t e, const char *where);
void note_launches(int n); // telemetry: kernels launched by the library (ga_launch_count)
// stream-ordered scratch from libga's private per-device pool (freed blocks stay cached there)
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t s);
cudaError_t scratch_free(void *p, cudaStream_t s);

#define GA_CHECK_LAUNCH(where)                                                     \
    do {                                                                           \
        ::ga::note_launches(1);                                                    \
        cudaError_t _e = cudaPeekAtLastError();                                    \
        if (_e != cudaSuccess) return ::ga::cuda_fail(_e, where);                  \
    } while (0)

// task index / heads without a 64-bit division (~100 instructions each) in the common cases
__device__ __forceinline__ int64_t div_heads(int64_t g, int H)
{
    if (H == 1) return g;
    if (g < 0xffffffffLL) return (int64_t)((uint32_t)g / (uint32_t)H);
    return g / H;
}

// ---------------------------------------------------------------- math
__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp(float x) { return __frcp_rn(x); }

// ---------------------------------------------------------------- dtype traits
template <typename T> struct DT;
template <> struct DT<float> { static constexpr int VEC = 4; };
template <> struct DT<__nv_bfloat16> { static constexpr int VEC = 8; };
template <> struct DT<__half> { static constexpr int VEC = 8; };

__device__ __forceinline__ uint4 ldg16(const void *p)
{
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void stg16(void *p, uint4 v)
{
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

template <typename T> __device__ __forceinline__ void unpack(const uint4 &u, float *f);

template <> __device__ __forceinline__ void unpack<float>(const uint4 &u, float *f)
{
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
}

__device__ __forceinline__ void bf2_to_f(uint32_t w, float &lo, float &hi)
{
    lo = __uint_as_float(w << 16);
    hi = __uint_as_float(w & 0xffff0000u);
}

template <> __device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4 &u, float *f)
{
    bf2_to_f(u.x, f[0], f[1]);
    bf2_to_f(u.y, f[2], f[3]);
    bf2_to_f(u.z, f[4], f[5]);
    bf2_to_f(u.w, f[6], f[7]);
}

__device__ __forceinline__ void h2_to_f(uint32_t w, float &lo, float &hi)
{
    __half2 h = *reinterpret_cast<__half2 *>(&w);
    float2 f = __half22float2(h);
    lo = f.x;
    hi = f.y;
}

template <> __device__ __forceinline__ void unpack<__half>(const uint4 &u, float *f)
{
    h2_to_f(u.x, f[0], f[1]);
    h2_to_f(u.y, f[2], f[3]);
    h2_to_f(u.z, f[4], f[5]);
    h2_to_f(u.w, f[6], f[7]);
}

template <typename T> __device__ __forceinline__ uint4 pack(const float *f);

template <> __device__ __forceinline__ uint4 pack<float>(const float *f)
{
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
}

__device__ __forceinline__ uint32_t f2_to_bf2(float lo, float hi)
{
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&b);
}

template <> __device__ __forceinline__ uint4 pack<__nv_bfloat16>(const float *f)
{
    return make_uint4(f2_to_bf2(f[0], f[1]), f2_to_bf2(f[2], f[3]), f2_to_bf2(f[4], f[5]), f2_to_bf2(f[6], f[7]));
}

__device__ __forceinline__ uint32_t f2_to_h2(float lo, float hi)
{
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&h);
}

template <> __device__ __forceinline__ uint4 pack<__half>(const float *f)
{
    return make_uint4(f2_to_h2(f[0], f[1]), f2_to_h2(f[2], f[3]), f2_to_h2(f[4], f[5]), f2_to_h2(f[6], f[7]));
}

// ---------------------------------------------------------------- 16-bit pair helpers
template <typename T> __device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) { return f2_to_bf2(lo, hi); }
template <> __device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) { return f2_to_h2(lo, hi); }

// c + x.lo*y.lo + x.hi*y.hi with 16-bit inputs and f32 accumulation (FHFMA)
template <typename T> __device__ __forceinline__ float fma2h(uint32_t x, uint32_t y, float c);

template <> __device__ __forceinline__ float fma2h<__nv_bfloat16>(uint32_t x, uint32_t y, float c)
{
    float d;
    asm("{ .reg .b16 xl, xh, yl, yh; .reg .f32 t; mov.b32 {xl, xh}, %1; mov.b32 {yl, yh}, %2;\n\t"
        "fma.rn.f32.bf16 t, xl, yl, %3; fma.rn.f32.bf16 %0, xh, yh, t; }"
        : "=f"(d)
        : "r"(x), "r"(y), "f"(c));
    return d;
}

template <> __device__ __forceinline__ float fma2h<__half>(uint32_t x, uint32_t y, float c)
{
    float d;
    asm("{ .reg .b16 xl, xh, yl, yh; .reg .f32 t; mov.b32 {xl, xh}, %1; mov.b32 {yl, yh}, %2;\n\t"
        "fma.rn.f32.f16 t, xl, yl, %3; fma.rn.f32.f16 %0, xh, yh, t; }"
        : "=f"(d)
        : "r"(x), "r"(y), "f"(c));
    return d;
}

// (o0, o1) += p * (v.lo, v.hi), p held in the low half of a 16x2 register
template <typename T> __device__ __forceinline__ void axpy2h(uint32_t p16x2, uint32_t v, float &o0, float &o1);

template <> __device__ __forceinline__ void axpy2h<__nv_bfloat16>(uint32_t p, uint32_t v, float &o0, float &o1)
{
    asm("{ .reg .b16 pl, ph, vl, vh; mov.b32 {pl, ph}, %2; mov.b32 {vl, vh}, %3;\n\t"
        "fma.rn.f32.bf16 %0, pl, vl, %0; fma.rn.f32.bf16 %1, pl, vh, %1; }"
        : "+f"(o0), "+f"(o1)
        : "r"(p), "r"(v));
}

template <> __device__ __forceinline__ void axpy2h<__half>(uint32_t p, uint32_t v, float &o0, float &o1)
{
    asm("{ .reg .b16 pl, ph, vl, vh; mov.b32 {pl, ph}, %2; mov.b32 {vl, vh}, %3;\n\t"
        "fma.rn.f32.f16 %0, pl, vl, %0; fma.rn.f32.f16 %1, pl, vh, %1; }"
        : "+f"(o0), "+f"(o1)
        : "r"(p), "r"(v));
}

// ---------------------------------------------------------------- kernel parameters
struct AttnParams {
    const void *Q, *K, *V;
    void *out;
    DevMask mask;
    int64_t q_begin, q_rows, kv_begin, kv_rows;
    int32_t H, d;
    float scale_log2; // log2(e) / sqrt(d)
    int64_t nnz;             // CSR edge count (upper bound for the heavy-row plan)
    int64_t heavy_threshold; // CSR: rows above this are skipped by the light kernel (0 = none)
    unsigned long long *edge_counter;
    unsigned long long *row_fingerprint;
    unsigned long long *tensor_counter; // tcgen05 window kernel probe: MMA tile products
    // Sharded runs over peer memory (ga_attention_sharded): rank q holds K/V token rows
    // [q*shard_rows, (q+1)*shard_rows) at k_peer[q] / v_peer[q] (CUDA IPC mappings; the
    // local rank's own entry is its K/V).  Rows outside [kv_begin, kv_begin + kv_rows) are
    // read from their owner over NVLink.  NULL = single-buffer mode.
    const char *const *k_peer;
    const char *const *v_peer;
    int64_t shard_rows;
    // optional caller workspace (ga_opts): CSR heavy-row split, LongNet block partials
    void *workspace;
    size_t workspace_bytes;
    // carried (m, l, o) state (ga_opts.state; state.m == NULL: none)
    ga_state state;
    int32_t state_mode;
    // explicit CSR on the edge kernel: edges whose key lies outside [kv_begin, kv_begin +
    // kv_rows) are skipped (a row's sorted columns in that range are one contiguous slice,
    // found by binary search) — one key block of the ring exchange (ga_opts.exchange)
    int32_t kv_clip;
};

// Base address (head 0, element 0) of K and V token row j: the local buffer when j is in
// [kv_begin, kv_begin + kv_rows), else the owning peer's buffer (sharded runs).
__device__ __forceinline__ void kv_row(const AttnParams &p, int64_t j, size_t row_bytes, const char *&kr,
                                       const char *&vr)
{
    const int64_t lj = j - p.kv_begin;
    if (p.k_peer == nullptr || (uint64_t)lj < (uint64_t)p.kv_rows) {
        kr = reinterpret_cast<const char *>(p.K) + lj * (int64_t)row_bytes;
        vr = reinterpret_cast<const char *>(p.V) + lj * (int64_t)row_bytes;
        return;
    }
    const int64_t q = j / p.shard_rows;
    const int64_t off = (j - q * p.shard_rows) * (int64_t)row_bytes;
    kr = p.k_peer[q] + off;
    vr = p.v_peer[q] + off;
}

// launchers (defined in the kernel translation units)
ga_status launch_edge(const AttnParams &p, ga_dtype dt, cudaStream_t s);
ga_status launch_csr_heavy(const AttnParams &p, ga_dtype dt, void *ws, size_t ws_bytes, cudaStream_t s);
bool csr_mma_supported(const AttnParams &p, ga_dtype dt);
ga_status launch_csr_mma(const AttnParams &p, ga_dtype dt, cudaStream_t s);
size_t csr_heavy_workspace(int64_t rows, int64_t Lmask, int64_t nnz, int32_t H, int32_t d, int64_t C);
bool window_tiled_supported(const AttnParams &p, ga_dtype dt);
int64_t band_tile_rows(); // class rows per band-kernel tile
int64_t window_tc_tile_rows(); // class rows per tcgen05 window-kernel tile
ga_status launch_window_tiled(const AttnParams &p, ga_dtype dt, cudaStream_t s);
bool longnet_tc_supported(const AttnParams &p, ga_dtype dt);
ga_status launch_longnet_tc(const AttnParams &p, ga_dtype dt, cudaStream_t s, bool use_umma);
int longnet_umma_levels(const AttnParams &p, ga_dtype dt);
size_t longnet_umma_workspace(const AttnParams &p, int h0);
bool window_tc_supported(const AttnParams &p, ga_dtype dt);
ga_status launch_window_tc(const AttnParams &p, ga_dtype dt, cudaStream_t s);
size_t full_rows_partials_bytes(int64_t F, int64_t Lm, int32_t H, int32_t d);
ga_status launch_full_rows(const AttnParams &p, ga_dtype dt, const int64_t *nfull_packed, const int64_t *full_row,
                           float *fpart, int64_t F, cudaStream_t s);
ga_status bigbird_check(const AttnParams &p);
size_t bigbird_workspace(const AttnParams &p, ga_dtype dt);
ga_status launch_bigbird(const AttnParams &p, ga_dtype dt, cudaStream_t s);
ga_status attention_backward(const AttnParams &p, ga_dtype dt, const void *O, const void *dO, const float *lse_in,
                             float *dQ, float *dK, float *dV, cudaStream_t s);
bool backward_tc_supported(const AttnParams &p, ga_dtype dt);
ga_status launch_backward_tc(const AttnParams &p, ga_dtype dt, const void *O, const void *dO, const float *lse_in,
                             float *lse, float *Dv, float *dQ, float *dK, float *dV, cudaStream_t s);

ga_status maskgen_to_csr(const DevMask &M, int64_t *row_ptr, int32_t *col_idx, cudaStream_t s);
ga_status mask_validate(const DevMask &M, cudaStream_t s, int *ok);
ga_status scan_exclusive_i64(int64_t *data, int64_t n, cudaStream_t s);
ga_status fill_inputs(void *dst, ga_dtype dt, int64_t n, uint64_t seed, int32_t tensor, int64_t e0, float shift,
                      cudaStream_t s);
ga_status state_finalize(const ga_state &st, int64_t rows, int32_t H, int32_t d, ga_dtype dt, void *out,
                         cudaStream_t s);

} // namespace ga

// microbench.cu — B200 pipe throughputs that decide the window-kernel design:
// FFMA (3-register), FFMA2 (fma.rn.f32x2), legacy HMMA (mma.sync m16n8k16 bf16->f32),
// MUFU ex2, shared-memory LDS.128 (broadcast and conflict-free).
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_ffma(float *out, float a, float b)
{
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 0.001f + i;
    float x = a + threadIdx.x * 1e-7f, y = b - threadIdx.x * 1e-7f;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(x, acc[i], y);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float *out, float a, float b)
{
    float2 acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
    float2 x = make_float2(a + threadIdx.x * 1e-7f, a), y = make_float2(b, b - threadIdx.x * 1e-7f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(x, acc[i], y);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_hmma(float *out)
{
    unsigned a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = 7, a3 = 11, b0 = 5, b1 = threadIdx.x;
    float c[4][4] = {};
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                         "{%0,%1,%2,%3};"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2(float *out, float a)
{
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = a * i + threadIdx.x * 1e-6f;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(acc[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fhfma(float *out, unsigned a, unsigned b)
{
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 0.001f + i;
    unsigned x = a + threadIdx.x, y = b ^ threadIdx.x;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("{ .reg .b16 xl, xh, yl, yh; mov.b32 {xl, xh}, %1; mov.b32 {yl, yh}, %2; "
                         "fma.rn.f32.bf16 %0, xh, yl, %0; }" : "+f"(acc[i]) : "r"(x), "r"(y));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <bool BCAST>
__global__ void k_lds(float *out)
{
    __shared__ float4 sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = BCAST ? 0 : (threadIdx.x & 31);
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float4 v = sm[(idx + i * 32 + (it & 3) * 256) & 1023];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <typename F>
float timeit(F f)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 256;
    float *out;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    const double thr = (double)blocks * threads;
    float ms = timeit([&] { k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.5f); });
    printf("FFMA  : %.2f TFLOP/s (%.1f FMA/clk/SM at 1.965GHz)\n", thr * ITERS * 8 * 2 / ms / 1e9,
           thr * ITERS * 8 / (ms * 1e-3) / sms / 1.965e9);
    ms = timeit([&] { k_ffma2<<<blocks, threads>>>(out, 1.0001f, 0.5f); });
    printf("FFMA2 : %.2f TFLOP/s (%.1f FMA/clk/SM)\n", thr * ITERS * 16 * 2 / ms / 1e9,
           thr * ITERS * 16 / (ms * 1e-3) / sms / 1.965e9);
    ms = timeit([&] { k_fhfma<<<blocks, threads>>>(out, 0x3f803f80u, 0x3f813f81u); });
    printf("FHFMA : %.2f TFLOP/s (%.1f FMA/clk/SM)\n", thr * ITERS * 8 * 2 / ms / 1e9,
           thr * ITERS * 8 / (ms * 1e-3) / sms / 1.965e9);
    ms = timeit([&] { k_hmma<<<blocks, threads>>>(out); });
    printf("HMMA  : %.2f TFLOP/s (m16n8k16 bf16, f32 acc)\n", (thr / 32) * (ITERS / 4) * 4 * 16 * 8 * 16 * 2 / ms / 1e9);
    ms = timeit([&] { k_ex2<<<blocks, threads>>>(out, 0.3f); });
    printf("EX2   : %.2f Gop/s (%.1f /clk/SM)\n", thr * (ITERS / 4) * 8 / ms / 1e6,
           thr * (ITERS / 4) * 8 / (ms * 1e-3) / sms / 1.965e9);
    ms = timeit([&] { k_lds<true><<<blocks, threads>>>(out); });
    printf("LDS128 bcast : %.1f warp-instr/clk/SM\n", (thr / 32) * (ITERS / 4) * 8 / (ms * 1e-3) / sms / 1.965e9);
    ms = timeit([&] { k_lds<false><<<blocks, threads>>>(out); });
    printf("LDS128 lanes : %.1f warp-instr/clk/SM (%.0f B/clk/SM)\n",
           (thr / 32) * (ITERS / 4) * 8 / (ms * 1e-3) / sms / 1.965e9,
           (thr / 32) * (ITERS / 4) * 8 * 512 / (ms * 1e-3) / sms / 1.965e9);
    return 0;
}

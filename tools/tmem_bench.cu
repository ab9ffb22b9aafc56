// tmem_bench.cu — per-SM rates that bound the tcgen05 softmax chunk loop (d = 64):
//   * MUFU ex2 on f32, f16x2 and bf16x2 operands (elements / clk / SM)
//   * TMEM -> register reads (tcgen05.ld 32x32b.x32) with 4..16 warps per SM (bytes / clk / SM)
//   * both mixed as in the softmax (64 columns read, 64 exponentials) to see whether they overlap
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define ITERS 2048

__global__ void k_ex2_f32(float *out, float a)
{
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = a * i + threadIdx.x * 1e-6f;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(acc[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2_f16x2(float *out, float a)
{
    uint32_t acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        __half2 h = __floats2half2_rn(a * i - 0.5f, -a * i);
        acc[i] = *reinterpret_cast<uint32_t *>(&h) ^ (threadIdx.x & 1);
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(acc[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += (float)acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2_bf16x2(float *out, float a)
{
    uint32_t acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a * i - 0.5f, -a * i);
        acc[i] = *reinterpret_cast<uint32_t *>(&h) ^ (threadIdx.x & 1);
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(acc[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += (float)acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t *r)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void ld16x256(uint32_t taddr, uint32_t *r)
{
    // 16 lanes x 256 bits, .x8: 32 registers per thread as well (other access shape)
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t *r)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                 "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                 "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
                 : "memory");
}

// mode 0: TMEM reads only (64 columns per step); 1: reads + 64 ex2 (f32) per step (the softmax
// chunk); 2: ex2 only on register data (no TMEM); 3: reads with 16x256b shape; 4: reads + ex2 +
// 32-column P store (the whole softmax chunk traffic)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_tmem(float *out, int iters)
{
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    // warp w: lanes 32 (w % 4), its own 64-column window (warps of one lane quarter share columns
    // modulo 512)
    const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64 % 512);
    float acc = 0.f;
    uint32_t r[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) r[i] = 0x3f000000u + threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 1 || MODE == 4) {
            ld32(ta, r);
            ld32(ta + 32, r + 32);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else if (MODE == 3) {
            ld16x256(ta, r);
            ld16x256(ta + 32, r + 32);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        if (MODE == 1 || MODE == 2 || MODE == 4) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                float x0 = __uint_as_float(r[i]) * 0.01f - 1.f, x1 = __uint_as_float(r[i + 1]) * 0.01f - 1.f;
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
                s0 += x0;
                s1 += x1;
                if (MODE == 4) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
                    r[i / 2] = *reinterpret_cast<uint32_t *>(&h);
                }
            }
            acc += s0 + s1;
            if (MODE == 2) {
#pragma unroll
                for (int i = 0; i < 64; ++i) r[i] += 1u;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) acc += __uint_as_float(r[i]);
        }
        if (MODE == 4) {
            st32(ta + 256 % 512, r); // P columns (other half of the window set)
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

template <typename F> float timeit(F f)
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
    const double clk = 1.965e9;
    float *out;
    cudaMalloc(&out, sizeof(float) * sms * 4 * 512);
    {
        const int blocks = sms * 4, threads = 256;
        const double thr = (double)blocks * threads;
        float ms = timeit([&] { k_ex2_f32<<<blocks, threads>>>(out, 0.3f); });
        printf("ex2 f32     : %.1f elem/clk/SM\n", thr * ITERS * 8 / (ms * 1e-3) / sms / clk);
        ms = timeit([&] { k_ex2_f16x2<<<blocks, threads>>>(out, 0.3f); });
        printf("ex2 f16x2   : %.1f elem/clk/SM\n", thr * ITERS * 16 / (ms * 1e-3) / sms / clk);
        ms = timeit([&] { k_ex2_bf16x2<<<blocks, threads>>>(out, 0.3f); });
        printf("ex2 bf16x2  : %.1f elem/clk/SM\n", thr * ITERS * 16 / (ms * 1e-3) / sms / clk);
    }
    const int iters = 4096;
    const char *names[5] = {"ld 64 cols", "ld 64 + 64 ex2", "64 ex2 (regs)", "ld 16x256b", "ld + ex2 + st P"};
    for (int mode = 0; mode < 5; ++mode)
        for (int nw = 4; nw <= 16; nw += 4) {
            float ms = 0;
            auto run = [&] {
                switch (mode) {
                case 0: k_tmem<0><<<sms, nw * 32>>>(out, iters); break;
                case 1: k_tmem<1><<<sms, nw * 32>>>(out, iters); break;
                case 2: k_tmem<2><<<sms, nw * 32>>>(out, iters); break;
                case 3: k_tmem<3><<<sms, nw * 32>>>(out, iters); break;
                default: k_tmem<4><<<sms, nw * 32>>>(out, iters); break;
                }
            };
            ms = timeit(run);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            const double steps = (double)nw * iters; // warp-steps per SM
            const double cyc = ms * 1e-3 * clk;
            printf("%-16s warps/SM %2d: %7.1f cyc per warp-step (SM), %6.1f B/clk/SM TMEM read, %5.1f ex2/clk/SM\n",
                   names[mode], nw, cyc / steps, (mode == 2 ? 0.0 : steps * 32 * 64 * 4 / cyc),
                   (mode == 1 || mode == 2 || mode == 4 ? steps * 32 * 64 / cyc : 0.0));
        }
    return 0;
}

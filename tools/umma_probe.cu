// umma_probe.cu — standalone check of the tcgen05 building blocks used by longnet_umma.cu:
// S = Q K^T (SS MMA, M=128 N=64 K=64, 128B-swizzled K-major operands), P = bf16(S) written to
// TMEM with tcgen05.st, O = P V (TS MMA, V MN-major).  Bounded mbarrier spins report a
// timeout instead of hanging.  Build: see tools/README or the gpurun command in DESIGN.md.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"
#include "umma.cuh"

using namespace ga;
using namespace ga::tc;
using namespace ga::umma;

__device__ bool wait_bounded(uint32_t mbar, uint32_t phase, int *flag)
{
    for (long long n = 0; n < 20000000; ++n)
        if (mbar_try(mbar, phase)) return true;
    atomicExch(flag, 1);
    return false;
}

__global__ void probe(const __nv_bfloat16 *Q, const __nv_bfloat16 *K, const __nv_bfloat16 *V, float *S_out,
                      float *O_out, int *flag, int mode)
{
    constexpr int D = 64, RB = 128, N = 64;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sQ = (raw + 1023u) & ~1023u;
    const uint32_t sK = sQ + 128 * RB, sV = sK + N * RB;
    __shared__ uint64_t mbar[2];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int idx = tid; idx < 128 * 8; idx += 128) {
        const int r = idx / 8, c = idx % 8;
        cp_async16(sQ + swz<D>(r, c), reinterpret_cast<const char *>(Q) + r * RB + c * 16);
    }
    for (int idx = tid; idx < N * 8; idx += 128) {
        const int r = idx / 8, c = idx % 8;
        cp_async16(sK + swz<D>(r, c), reinterpret_cast<const char *>(K) + r * RB + c * 16);
        cp_async16(sV + swz<D>(r, c), reinterpret_cast<const char *>(V) + r * RB + c * 16);
    }
    cp_async_commit();
    cp_async_wait<0>();
    fence_proxy_async();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tbase))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const uint32_t mS = (uint32_t)__cvta_generic_to_shared(&mbar[0]), mO = (uint32_t)__cvta_generic_to_shared(&mbar[1]);
    if (tid == 0) {
        mbar_init(mS, 1);
        mbar_init(mO, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tbase;
    const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
    if (tid == 0) {
        fence_after();
        const uint32_t id = idesc<__nv_bfloat16>(128, N, false);
        for (int kk = 0; kk < D / 16; ++kk)
            mma_ss(tmem + 0, sdesc_sw128(sQ + kk * 32), sdesc_sw128(sK + kk * 32), id, kk > 0);
        mma_commit(mS);
    }
    bool ok = wait_bounded(mS, 0, flag);
    fence_after();
    float sv[64];
    tmem_ld32(tl + 0, sv);
    tmem_ld32(tl + 32, sv + 32);
    tmem_wait_ld();
    for (int j = 0; j < N; ++j) S_out[tid * N + j] = ok ? sv[j] : -999.f;
    if (mode >= 1) {
        uint32_t pk[32];
        for (int i = 0; i < 32; ++i) pk[i] = tc::pack2<__nv_bfloat16>(sv[2 * i], sv[2 * i + 1]);
        tmem_st32(tl + 64, pk);
        tmem_wait_st();
        fence_before();
        __syncthreads();
        if (tid == 0) {
            fence_after();
            const uint32_t id = idesc<__nv_bfloat16>(128, D, true);
            for (int kk = 0; kk < N / 16; ++kk)
                mma_ts(tmem + 128, tmem + 64 + kk * 8, sdesc_sw128(sV + kk * 16 * RB), id, kk > 0);
            mma_commit(mO);
        }
        ok = wait_bounded(mO, 0, flag);
        fence_after();
        float ov[64];
        tmem_ld32(tl + 128, ov);
        tmem_ld32(tl + 160, ov + 32);
        tmem_wait_ld();
        for (int j = 0; j < D; ++j) O_out[tid * D + j] = ok ? ov[j] : -999.f;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
    }
}

static float bf(float x) { __nv_bfloat16 b = __float2bfloat16(x); return __bfloat162float(b); }

int main(int argc, char **argv)
{
    const int mode = argc > 1 ? atoi(argv[1]) : 1;
    std::vector<__nv_bfloat16> q(128 * 64), k(64 * 64), v(64 * 64);
    std::vector<float> qf(128 * 64), kf(64 * 64), vf(64 * 64);
    for (int i = 0; i < 128; ++i)
        for (int c = 0; c < 64; ++c) { qf[i * 64 + c] = bf(((i * 7 + c * 3) % 9 - 4) * 0.125f); q[i * 64 + c] = __float2bfloat16(qf[i * 64 + c]); }
    for (int j = 0; j < 64; ++j)
        for (int c = 0; c < 64; ++c) {
            kf[j * 64 + c] = bf(((j * 5 + c * 11) % 7 - 3) * 0.25f); k[j * 64 + c] = __float2bfloat16(kf[j * 64 + c]);
            vf[j * 64 + c] = bf(((j * 3 + c * 13) % 11 - 5) * 0.0625f); v[j * 64 + c] = __float2bfloat16(vf[j * 64 + c]);
        }
    __nv_bfloat16 *dq, *dk, *dv;
    float *ds, *dO;
    int *dflag;
    cudaMalloc(&dq, q.size() * 2); cudaMalloc(&dk, k.size() * 2); cudaMalloc(&dv, v.size() * 2);
    cudaMalloc(&ds, 128 * 64 * 4); cudaMalloc(&dO, 128 * 64 * 4); cudaMalloc(&dflag, 4);
    cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, k.data(), k.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), v.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dflag, 0, 4);
    cudaMemset(dO, 0, 128 * 64 * 4);
    const int smem = 1024 + 128 * 128 + 2 * 64 * 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(dq, dk, dv, ds, dO, dflag, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> S(128 * 64), O(128 * 64);
    int flag = 0;
    cudaMemcpy(S.data(), ds, S.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&flag, dflag, 4, cudaMemcpyDeviceToHost);
    double es = 0, eo = 0;
    std::vector<float> Sr(128 * 64);
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 64; ++j) {
            double a = 0;
            for (int c = 0; c < 64; ++c) a += (double)qf[i * 64 + c] * kf[j * 64 + c];
            Sr[i * 64 + j] = (float)a;
            es = std::max(es, std::abs(a - S[i * 64 + j]));
        }
    for (int i = 0; i < 128; ++i)
        for (int c = 0; c < 64; ++c) {
            double a = 0;
            for (int j = 0; j < 64; ++j) a += (double)bf(Sr[i * 64 + j]) * vf[j * 64 + c];
            eo = std::max(eo, std::abs(a - O[i * 64 + c]));
        }
    printf("timeout flag %d\nS max err %.3g (S[0][0..3] = %g %g %g %g, ref %g %g %g %g)\nO max err %.3g (O[5][0..1] = %g %g)\n",
           flag, es, S[0], S[1], S[2], S[3], Sr[0], Sr[1], Sr[2], Sr[3], eo, O[5 * 64], O[5 * 64 + 1]);
    return (flag == 0 && es < 1e-3 && eo < 1e-2) ? 0 : 1;
}

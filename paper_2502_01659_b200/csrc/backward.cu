// backward.cu — backward pass of graph-view masked attention (the training
// use case of PAPER.md:555, "1B tokens on 32 GPUs").
//
// For O_i = sum_{j in N(i)} P_ij V_j with P_ij = softmax_j(S_ij), S_ij = q_i.k_j / sqrt(d)
// (Eq. 1) and upstream gradients dO, per edge (i, j) of the mask:
//
//   P_ij = 2^(S_ij log2(e) - lse_i)           lse_i = log2 sum_j 2^(S_ij log2(e))  (log2 domain)
//   dP_ij = dO_i . V_j,   D_i = dO_i . O_i,   dS_ij = P_ij (dP_ij - D_i)
//   dQ_i = sum_j dS_ij k_j / sqrt(d)          (row pass: gather over N(i))
//   dK_j = sum_i dS_ij q_i / sqrt(d)          (column pass: gather over N^T(j))
//   dV_j = sum_i P_ij dO_i
//
// Two launches, no atomics, deterministic:
//   row pass     warp per (query row, head): lse (one extra pass over the edges unless the
//                caller passes the forward's lse), D_i, then dQ_i — K_j, V_j gathered per edge;
//   column pass  warp per (key row, head): N^T(j) = N(j) for the symmetric families (every
//                paper mask: window, dilated, block-dilated, LongNet — their predicates are
//                symmetric in i, j), else a transposed CSR built on the device (stable radix
//                sort of the column indices, multiplicities kept) — q_i, dO_i, lse_i, D_i
//                gathered per edge.
// Each edge's score and weight are recomputed in both passes (the L x L matrix is never
// formed, as in the forward).  Lane layout as in the forward edge kernel (edge_core.cuh): a
// (row, head) vector is CH 16-byte chunks, a lane owns NC of them, G = CH / NC lanes per edge,
// E = 32 / G edges in flight per warp.
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace ga {
namespace bwd {

template <typename T, int D> struct Lay {
    static constexpr int VEC = DT<T>::VEC;
    static constexpr int CH = D / VEC;
    static constexpr int NCMAX = sizeof(T) == 2 ? 1 : 4;
    static constexpr int NC = CH >= NCMAX ? NCMAX : CH;
    static constexpr int G = CH / NC;
    static constexpr int E = 32 / G;
    static constexpr int PER = NC * VEC; // elements per lane
};

template <typename T, int D>
__device__ __forceinline__ void load_slice(const void *base, int64_t row, int h, int H, int sub, float *f)
{
    using Y = Lay<T, D>;
    const char *p = reinterpret_cast<const char *>(base) + ((size_t)row * H + h) * D * sizeof(T) +
                    (size_t)sub * Y::PER * sizeof(T);
#pragma unroll
    for (int c = 0; c < Y::NC; ++c) unpack<T>(ldg16(p + 16 * c), f + Y::VEC * c);
}

template <int G> __device__ __forceinline__ float group_sum(float x)
{
#pragma unroll
    for (int off = 1; off < G; off <<= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    return x;
}

template <int PER> __device__ __forceinline__ float dot(const float *a, const float *b)
{
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int e = 0; e < PER; e += 2) {
        s0 = fmaf(a[e], b[e], s0);
        s1 = fmaf(a[e + 1], b[e + 1], s1);
    }
    return s0 + s1;
}

// Neighbour source of one row: the implicit pieces of the family, or a CSR (the transposed
// one in the column pass).
struct Nbrs {
    const int64_t *rp; // CSR row_ptr, or nullptr for the implicit pieces of `M`
    const int32_t *ci;
};

__device__ __forceinline__ int npieces(const DevMask &M, const Nbrs &nb, int64_t i, int h)
{
    return nb.rp ? 1 : num_pieces_h(M, i, h);
}

__device__ __forceinline__ Piece piece(const DevMask &M, const Nbrs &nb, int64_t i, int pc, int h)
{
    if (!nb.rp) return get_piece_h(M, i, pc, h);
    Piece P;
    P.mode = P_CSR;
    P.cols = nb.ci;
    P.base = nb.rp[i];
    P.step = 1;
    P.count = nb.rp[i + 1] - P.base;
    P.alpha = P.rexcl = P.pad = 0;
    return P;
}

struct Args {
    const void *O, *dO;
    float *lse, *Dv;     // [L, H] scratch: the row pass writes them, the column pass reads them
    const float *lse_in; // caller's forward lse (log2 domain) or nullptr
    float *dQ, *dK, *dV; // fp32 [L, H, d]
    Nbrs fwd, tr;        // N(i) and N^T(j)
};

// row pass: lse_i, D_i, dQ_i
template <typename T, int D>
__global__ void __launch_bounds__(256) row_kernel(const __grid_constant__ AttnParams p, const Args a)
{
    using Y = Lay<T, D>;
    const int lane = threadIdx.x & 31, g = lane / Y::G, sub = lane % Y::G;
    const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int H = p.H;
    if (gw >= p.mask.L * H) return;
    const int64_t i = gw / H;
    const int h = (int)(gw - i * H);
    const float sl2 = p.scale_log2;
    float q[Y::PER], dO[Y::PER], x[Y::PER], y[Y::PER];
    load_slice<T, D>(p.Q, i, h, H, sub, q);
    load_slice<T, D>(a.dO, i, h, H, sub, dO);
    load_slice<T, D>(a.O, i, h, H, sub, x);
    const float Di = group_sum<Y::G>(dot<Y::PER>(dO, x));
    const int np = npieces(p.mask, a.fwd, i, h);
    float lse;
    if (a.lse_in) {
        lse = a.lse_in[gw];
    } else { // log2-sum-exp2 of the row's scores: online (m, l) per lane group, then merged
        float m = -INFINITY, l = 0.f;
        for (int pc = 0; pc < np; ++pc) {
            const Piece P = piece(p.mask, a.fwd, i, pc, h);
            for (int64_t k0 = 0; k0 < P.count; k0 += Y::E) {
                const int64_t k = k0 + g;
                const bool v = k < P.count;
                if (v) load_slice<T, D>(p.K, piece_at(P, k), h, H, sub, x);
                const float s = group_sum<Y::G>(v ? dot<Y::PER>(q, x) : 0.f) * sl2;
                if (v) {
                    if (s > m) {
                        l *= ex2(m - s);
                        m = s;
                    }
                    l += ex2(s - m);
                }
            }
        }
#pragma unroll
        for (int off = Y::G; off < 32; off <<= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, off), l2 = __shfl_xor_sync(0xffffffffu, l, off);
            const float mn = fmaxf(m, m2);
            l = (m == -INFINITY ? 0.f : l * ex2(m - mn)) + (m2 == -INFINITY ? 0.f : l2 * ex2(m2 - mn));
            m = mn;
        }
        lse = l > 0.f ? m + __log2f(l) : -INFINITY;
    }
    float dq[Y::PER];
#pragma unroll
    for (int e = 0; e < Y::PER; ++e) dq[e] = 0.f;
    for (int pc = 0; pc < np; ++pc) {
        const Piece P = piece(p.mask, a.fwd, i, pc, h);
        for (int64_t k0 = 0; k0 < P.count; k0 += Y::E) {
            const int64_t k = k0 + g;
            const bool v = k < P.count;
            if (v) {
                const int64_t j = piece_at(P, k);
                load_slice<T, D>(p.K, j, h, H, sub, x);
                load_slice<T, D>(p.V, j, h, H, sub, y);
            }
            const float s = group_sum<Y::G>(v ? dot<Y::PER>(q, x) : 0.f) * sl2;
            const float dp = group_sum<Y::G>(v ? dot<Y::PER>(dO, y) : 0.f);
            if (v) {
                const float ds = ex2(s - lse) * (dp - Di);
#pragma unroll
                for (int e = 0; e < Y::PER; ++e) dq[e] = fmaf(ds, x[e], dq[e]);
            }
        }
    }
#pragma unroll
    for (int off = Y::G; off < 32; off <<= 1)
#pragma unroll
        for (int e = 0; e < Y::PER; ++e) dq[e] += __shfl_xor_sync(0xffffffffu, dq[e], off);
    if (g == 0) {
        const float isd = sl2 * 0.69314718055994531f; // 1 / sqrt(d)
        float4 *dst = reinterpret_cast<float4 *>(a.dQ + gw * D + sub * Y::PER);
#pragma unroll
        for (int e = 0; e < Y::PER; e += 4)
            dst[e / 4] = make_float4(dq[e] * isd, dq[e + 1] * isd, dq[e + 2] * isd, dq[e + 3] * isd);
        if (sub == 0) {
            a.lse[gw] = lse;
            a.Dv[gw] = Di;
        }
    }
}

// column pass: dK_j, dV_j over N^T(j)
template <typename T, int D>
__global__ void __launch_bounds__(256) col_kernel(const __grid_constant__ AttnParams p, const Args a)
{
    using Y = Lay<T, D>;
    const int lane = threadIdx.x & 31, g = lane / Y::G, sub = lane % Y::G;
    const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int H = p.H;
    if (gw >= p.mask.L * H) return;
    const int64_t j = gw / H;
    const int h = (int)(gw - j * H);
    const float sl2 = p.scale_log2;
    float kj[Y::PER], vj[Y::PER], qi[Y::PER], gi[Y::PER], dk[Y::PER], dv[Y::PER];
    load_slice<T, D>(p.K, j, h, H, sub, kj);
    load_slice<T, D>(p.V, j, h, H, sub, vj);
#pragma unroll
    for (int e = 0; e < Y::PER; ++e) dk[e] = dv[e] = 0.f;
    const int np = npieces(p.mask, a.tr, j, h);
    for (int pc = 0; pc < np; ++pc) {
        const Piece P = piece(p.mask, a.tr, j, pc, h);
        for (int64_t k0 = 0; k0 < P.count; k0 += Y::E) {
            const int64_t k = k0 + g;
            const bool v = k < P.count;
            float lse = 0.f, Di = 0.f;
            if (v) {
                const int64_t i = piece_at(P, k);
                load_slice<T, D>(p.Q, i, h, H, sub, qi);
                load_slice<T, D>(a.dO, i, h, H, sub, gi);
                lse = a.lse[i * H + h];
                Di = a.Dv[i * H + h];
            }
            const float s = group_sum<Y::G>(v ? dot<Y::PER>(qi, kj) : 0.f) * sl2;
            const float dp = group_sum<Y::G>(v ? dot<Y::PER>(gi, vj) : 0.f);
            if (v) {
                const float pw = ex2(s - lse), ds = pw * (dp - Di);
#pragma unroll
                for (int e = 0; e < Y::PER; ++e) {
                    dv[e] = fmaf(pw, gi[e], dv[e]);
                    dk[e] = fmaf(ds, qi[e], dk[e]);
                }
            }
        }
    }
#pragma unroll
    for (int off = Y::G; off < 32; off <<= 1)
#pragma unroll
        for (int e = 0; e < Y::PER; ++e) {
            dk[e] += __shfl_xor_sync(0xffffffffu, dk[e], off);
            dv[e] += __shfl_xor_sync(0xffffffffu, dv[e], off);
        }
    if (g == 0) {
        const float isd = sl2 * 0.69314718055994531f;
        float4 *dK = reinterpret_cast<float4 *>(a.dK + gw * D + sub * Y::PER);
        float4 *dV = reinterpret_cast<float4 *>(a.dV + gw * D + sub * Y::PER);
#pragma unroll
        for (int e = 0; e < Y::PER; e += 4) {
            dK[e / 4] = make_float4(dk[e] * isd, dk[e + 1] * isd, dk[e + 2] * isd, dk[e + 3] * isd);
            dV[e / 4] = make_float4(dv[e], dv[e + 1], dv[e + 2], dv[e + 3]);
        }
    }
}

// transposed CSR: row ids of every edge, stable radix sort by column (multiplicities kept),
// row_ptr^T[c] = lower_bound(sorted columns, c)
__global__ void edge_rows_kernel(const int64_t *rp, int64_t L, int32_t *rows)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) rows[e] = (int32_t)i;
}

__global__ void tr_rowptr_kernel(const int32_t *cols_sorted, int64_t nnz, int64_t L, int64_t *rpt)
{
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= L; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)cols_sorted[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        rpt[c] = lo;
    }
}

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <typename T> static ga_status launch_d(const AttnParams &p, const Args &a, cudaStream_t s)
{
    const unsigned blocks = (unsigned)((p.mask.L * p.H + 7) / 8);
    switch (p.d) {
    case 32:
        row_kernel<T, 32><<<blocks, 256, 0, s>>>(p, a);
        col_kernel<T, 32><<<blocks, 256, 0, s>>>(p, a);
        break;
    case 64:
        row_kernel<T, 64><<<blocks, 256, 0, s>>>(p, a);
        col_kernel<T, 64><<<blocks, 256, 0, s>>>(p, a);
        break;
    case 128:
        row_kernel<T, 128><<<blocks, 256, 0, s>>>(p, a);
        col_kernel<T, 128><<<blocks, 256, 0, s>>>(p, a);
        break;
    default: set_error("d=%d unsupported", p.d); return GA_ERR_UNSUPPORTED;
    }
    note_launches(1);
    GA_CHECK_LAUNCH("bwd::row/col_kernel");
    return GA_OK;
}

} // namespace bwd

// GA_BWD_CUDACORE=1 forces the CUDA-core gather kernels (A/B against the tensor-core band path)
static bool getenv_off(const char *name)
{
    const char *v = getenv(name);
    return v != nullptr && v[0] != 0 && v[0] != '0';
}

ga_status attention_backward(const AttnParams &p, ga_dtype dt, const void *O, const void *dO, const float *lse_in,
                             float *dQ, float *dK, float *dV, cudaStream_t s)
{
    const DevMask &M = p.mask;
    const int64_t L = M.L, H = p.H;
    const bool csr = M.kind == K_CSR;
    const int64_t nnz = csr ? M.nnz : 0;
    // scratch: lse, D [L, H] fp32 | CSR only: edge rows int32 [nnz], sorted rows / cols [nnz],
    // row_ptr^T int64 [L + 1], CUB temp
    size_t sort_bytes = 0;
    if (csr && nnz > 0)
        cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int32_t *)nullptr, (int32_t *)nullptr,
                                        (const int32_t *)nullptr, (int32_t *)nullptr, nnz, 0, 32, s);
    const size_t sLH = bwd::align256(sizeof(float) * (size_t)(L * H));
    const size_t sE = bwd::align256(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    const size_t total = 2 * sLH + (csr ? 3 * sE + bwd::align256(sizeof(int64_t) * (size_t)(L + 1)) + sort_bytes : 0);
    char *w = nullptr;
    cudaError_t e = scratch_alloc(reinterpret_cast<void **>(&w), total, s);
    if (e != cudaSuccess) return cuda_fail(e, "backward scratch");
    bwd::Args a{};
    a.O = O;
    a.dO = dO;
    a.lse = reinterpret_cast<float *>(w);
    a.Dv = reinterpret_cast<float *>(w + sLH);
    a.lse_in = lse_in;
    a.dQ = dQ;
    a.dK = dK;
    a.dV = dV;
    ga_status st = GA_OK;
    if (backward_tc_supported(p, dt) && !getenv_off("GA_BWD_CUDACORE")) { // window bands on mma.sync
        st = launch_backward_tc(p, dt, O, dO, lse_in, a.lse, a.Dv, dQ, dK, dV, s);
        scratch_free(w, s);
        return st;
    }
    if (csr) {
        char *c = w + 2 * sLH;
        int32_t *rows = reinterpret_cast<int32_t *>(c), *rows_s = reinterpret_cast<int32_t *>(c + sE),
                *cols_s = reinterpret_cast<int32_t *>(c + 2 * sE);
        int64_t *rpt = reinterpret_cast<int64_t *>(c + 3 * sE);
        void *tmp = c + 3 * sE + bwd::align256(sizeof(int64_t) * (size_t)(L + 1));
        a.fwd = bwd::Nbrs{M.row_ptr, M.col_idx};
        a.tr = bwd::Nbrs{rpt, rows_s};
        const unsigned blocks = (unsigned)imin((L + 255) / 256, 148 * 16);
        if (nnz > 0) {
            bwd::edge_rows_kernel<<<blocks, 256, 0, s>>>(M.row_ptr, L, rows);
            note_launches(1);
            size_t tb = sort_bytes;
            if ((e = cub::DeviceRadixSort::SortPairs(tmp, tb, M.col_idx, cols_s, rows, rows_s, nnz, 0, 32, s)) !=
                cudaSuccess)
                st = cuda_fail(e, "backward: transpose sort");
        }
        if (st == GA_OK) {
            bwd::tr_rowptr_kernel<<<(unsigned)imin((L + 256) / 256, 148 * 16), 256, 0, s>>>(cols_s, nnz, L, rpt);
            GA_CHECK_LAUNCH("bwd::tr_rowptr_kernel");
        }
    }
    if (st == GA_OK) {
        switch (dt) {
        case GA_F32: st = bwd::launch_d<float>(p, a, s); break;
        case GA_BF16: st = bwd::launch_d<__nv_bfloat16>(p, a, s); break;
        case GA_F16: st = bwd::launch_d<__half>(p, a, s); break;
        }
    }
    scratch_free(w, s);
    return st;
}

} // namespace ga

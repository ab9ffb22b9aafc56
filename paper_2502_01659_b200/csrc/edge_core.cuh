// edge_core.cuh — the per-(row, head) edge loop shared by the generic edge kernel and the
// CSR heavy-row chunk kernel.  See edge_kernel.cu for the mapping onto lanes.
#pragma once
#include "common.cuh"

namespace ga {

template <typename T, int D, bool PROBE> struct EdgeAcc {
    static constexpr int VEC = DT<T>::VEC;
    static constexpr int G = D / VEC; // lanes per (edge, head) vector
    static constexpr int E = 32 / G;  // edges in flight per warp
    static constexpr bool H16 = sizeof(T) == 2; // bf16/fp16: FHFMA on packed pairs
    float q[VEC], o[VEC];
    uint32_t qp[4]; // packed 16-bit q (H16)
    float sl2;      // log2(e)/sqrt(d), applied after the reduction on the H16 path
    float m, l;
    unsigned long long n_edges, sum_j, sum_h;
    int g, sub;
    const AttnParams *prm;
    size_t row_bytes, hoff; // token row stride; this lane's (head, sub-vector) byte offset

    __device__ __forceinline__ void init(const AttnParams &p, int64_t t, int h, int lane)
    {
        g = lane / G;
        sub = lane % G;
        const T *Qp = reinterpret_cast<const T *>(p.Q) + ((size_t)t * p.H + h) * D + sub * VEC;
        prm = &p;
        hoff = ((size_t)h * D + sub * VEC) * sizeof(T);
        row_bytes = (size_t)p.H * D * sizeof(T);
        uint4 raw = ldg16(Qp);
        qp[0] = raw.x; qp[1] = raw.y; qp[2] = raw.z; qp[3] = raw.w;
        sl2 = p.scale_log2;
        unpack<T>(raw, q);
#pragma unroll
        for (int c = 0; c < VEC; ++c) { q[c] *= p.scale_log2; o[c] = 0.f; }
        m = -INFINITY;
        l = 0.f;
        n_edges = sum_j = sum_h = 0;
    }

    // neighbours k in [kb, ke) of piece P (warp-uniform bounds)
    __device__ __forceinline__ void run(const Piece &P, int64_t kb, int64_t ke)
    {
        for (int64_t k0 = kb; k0 < ke; k0 += 2 * E) {
            const int64_t ka = k0 + g, kk = k0 + E + g;
            const bool va = ka < ke, vb = kk < ke;
            uint4 kra = make_uint4(0, 0, 0, 0), vra = kra, krb = kra, vrb = kra;
            int64_t ja = 0, jb = 0;
            if (va) {
                ja = piece_at(P, ka);
                load(ja, kra, vra);
            }
            if (vb) {
                jb = piece_at(P, kk);
                load(jb, krb, vrb);
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (u == 1 && k0 + E >= ke) break; // warp-uniform: no group has work
                const float sc = score(u == 0 ? kra : krb);
                update(sc, u == 0 ? vra : vrb, u == 0 ? va : vb, u == 0 ? ja : jb);
            }
        }
    }

    // this lane's 16-byte slices of K_j and V_j (local buffer or the owning peer's)
    __device__ __forceinline__ void load(int64_t j, uint4 &kraw, uint4 &vraw) const
    {
        const char *kr, *vr;
        kv_row(*prm, j, row_bytes, kr, vr);
        kraw = ldg16(kr + hoff);
        vraw = ldg16(vr + hoff);
    }

    // one (key, value) edge into the group state (score already reduced over the group)
    __device__ __forceinline__ void update(float s, const uint4 &vraw, bool valid, int64_t j)
    {
        if (!valid) return;
        if (s > m) { // lazy rescale: only when the running max grows
            const float a = ex2(m - s);
            l *= a;
#pragma unroll
            for (int c = 0; c < VEC; ++c) o[c] *= a;
            m = s;
        }
        const float pr = ex2(s - m);
        l += pr;
        if constexpr (H16) { // o += p v with p rounded to the input type (as on the MMA paths)
            const uint32_t p2 = pack2<T>(pr, pr);
            axpy2h<T>(p2, vraw.x, o[0], o[1]);
            axpy2h<T>(p2, vraw.y, o[2], o[3]);
            axpy2h<T>(p2, vraw.z, o[4], o[5]);
            axpy2h<T>(p2, vraw.w, o[6], o[7]);
        } else {
            float vf[VEC];
            unpack<T>(vraw, vf);
#pragma unroll
            for (int c = 0; c < VEC; ++c) o[c] = fmaf(pr, vf[c], o[c]);
        }
        if (PROBE) {
            n_edges += 1;
            sum_j += (unsigned long long)j;
            sum_h += splitmix64((uint64_t)j);
        }
    }

    // q.k over the group (exp2 domain: scaled by log2(e)/sqrt(d))
    __device__ __forceinline__ float score(const uint4 &kraw) const
    {
        float s;
        if constexpr (H16) { // bf16 x bf16 + f32 without unpacking (FHFMA)
            const float s0 = fma2h<T>(qp[2], kraw.z, fma2h<T>(qp[0], kraw.x, 0.f));
            const float s1 = fma2h<T>(qp[3], kraw.w, fma2h<T>(qp[1], kraw.y, 0.f));
            s = s0 + s1;
        } else {
            float kf[VEC];
            unpack<T>(kraw, kf);
            s = 0.f;
#pragma unroll
            for (int c = 0; c < VEC; ++c) s = fmaf(q[c], kf[c], s);
        }
#pragma unroll
        for (int off = 1; off < G; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        return H16 ? s * sl2 : s;
    }

    // Explicit CSR piece, gather-bound: a warp loads 32 column indices with one coalesced
    // load and broadcasts them to the lane groups by shuffle, then issues the K/V loads of
    // DEPTH edge steps before consuming any (DEPTH * E edges in flight per warp), so the
    // random row gathers overlap instead of waiting on dependent index loads.
    template <int DEPTH>
    __device__ __forceinline__ void run_csr(const int32_t *cols, int64_t kb, int64_t ke)
    {
        static_assert(32 % (E * DEPTH) == 0 || E * DEPTH >= 32, "batch shape");
        constexpr int STEP = E * DEPTH; // edges per pass
        const int lane = (int)(threadIdx.x & 31);
        for (int64_t b0 = kb; b0 < ke; b0 += 32) {
            const int64_t kl = b0 + lane;
            const int my_j = kl < ke ? cols[kl] : -1;
#pragma unroll 1
            for (int e0 = 0; e0 < 32 && b0 + e0 < ke; e0 += STEP) {
                uint4 kr[DEPTH], vr[DEPTH];
                int jj[DEPTH];
#pragma unroll
                for (int u = 0; u < DEPTH; ++u) {
                    const int src = e0 + u * E + g;
                    jj[u] = __shfl_sync(0xffffffffu, my_j, src & 31);
                    if (src >= 32) jj[u] = -1;
                    if (jj[u] >= 0) {
                        load(jj[u], kr[u], vr[u]);
                    } else {
                        kr[u] = vr[u] = make_uint4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int u = 0; u < DEPTH; ++u) {
                    if (e0 + u * E >= 32 || b0 + e0 + u * E >= ke) break; // warp-uniform
                    const float s = score(kr[u]);
                    update(s, vr[u], jj[u] >= 0, jj[u]);
                }
            }
        }
    }

    // merge the E lane-group states: (m,l,o) (+) (m',l',o'), m* = max, rescaled sums
    __device__ __forceinline__ void merge_groups()
    {
#pragma unroll
        for (int off = G; off < 32; off <<= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
            const float l2 = __shfl_xor_sync(0xffffffffu, l, off);
            const float mn = fmaxf(m, m2);
            const float a = (m == -INFINITY) ? 0.f : ex2(m - mn);
            const float b = (m2 == -INFINITY) ? 0.f : ex2(m2 - mn);
            l = l * a + l2 * b;
#pragma unroll
            for (int c = 0; c < VEC; ++c) {
                const float o2 = __shfl_xor_sync(0xffffffffu, o[c], off);
                o[c] = o[c] * a + o2 * b;
            }
            m = mn;
        }
    }

    // normalise and store the row (lane group 0 holds the merged state)
    __device__ __forceinline__ void store(const AttnParams &p, int64_t t, int h) const
    {
        if (g != 0) return;
        float r[VEC];
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
        for (int c = 0; c < VEC; ++c) r[c] = o[c] * inv;
        T *Op = reinterpret_cast<T *>(p.out) + ((size_t)t * p.H + h) * D + sub * VEC;
        stg16(Op, pack<T>(r));
    }

    // warp totals of the probe counters (one lane per group counts)
    __device__ __forceinline__ void probe_totals(unsigned long long &ne, unsigned long long &sj,
                                                 unsigned long long &sh) const
    {
        ne = sub == 0 ? n_edges : 0;
        sj = sub == 0 ? sum_j : 0;
        sh = sub == 0 ? sum_h : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            ne += __shfl_xor_sync(0xffffffffu, ne, off);
            sj += __shfl_xor_sync(0xffffffffu, sj, off);
            sh += __shfl_xor_sync(0xffffffffu, sh, off);
        }
    }
};

// One (row, head) of Algorithm 1 by one warp: all pieces of N(i), merge, store.
// t = local query row (global row q_begin + t).
template <typename T, int D>
__device__ __forceinline__ void edge_row(const AttnParams &p, int64_t t, int h, int lane)
{
    EdgeAcc<T, D, false> acc;
    acc.init(p, t, h, lane);
    const int64_t i = p.q_begin + t;
    const int np = num_pieces(p.mask, i);
    for (int pc = 0; pc < np; ++pc) {
        const Piece P = get_piece(p.mask, i, pc);
        acc.run(P, 0, P.count);
    }
    acc.merge_groups();
    acc.store(p, t, h);
}

} // namespace ga

// edge_core.cuh — the per-(row, head) edge loop shared by the generic edge kernel and the
// CSR heavy-row chunk kernel.  See edge_kernel.cu for the mapping onto lanes.
#pragma once
#include "common.cuh"

namespace ga {

// Lane layout: a (row, head) vector of D elements is CH = D*sizeof(T)/16 chunks of 16 bytes;
// a lane owns NC = min(4, CH) consecutive chunks (64 bytes of K_j and of V_j per edge), so
// G = CH / NC lanes cover one edge (G = 2 for bf16 d=64, 1 for bf16 d=32, 4 for fp32 d=64)
// and a warp keeps E = 32 / G edges in flight per step.  The per-edge score needs only
// log2(G) shuffles, and each lane's softmax state (m, l) is shared by fewer lanes than with
// 16-byte lane slices.
template <typename T, int D, bool PROBE> struct EdgeAcc {
    static constexpr int VEC = DT<T>::VEC;      // elements per 16-byte chunk
    static constexpr int CH = D / VEC;          // chunks per (row, head) vector
    static constexpr int NCMAX = sizeof(T) == 2 ? 1 : 4; // 16-bit: 16 B per lane (random CSR gathers)
    static constexpr int NC = CH >= NCMAX ? NCMAX : CH; // chunks per lane
    static constexpr int G = CH / NC;           // lanes per edge
    static constexpr int E = 32 / G;            // edges in flight per warp and step
    static constexpr int PER = NC * VEC;        // elements of o per lane
    static constexpr bool H16 = sizeof(T) == 2; // bf16/fp16: FHFMA on packed pairs
    uint4 qraw[NC]; // this lane's slice of q (stored type)
    float o[PER];
    float sl2;      // log2(e)/sqrt(d): scores are kept in the exp2 domain
    float m, l;
    unsigned long long n_edges, sum_j, sum_h;
    int g, sub;
    const AttnParams *prm;
    size_t row_bytes, hoff; // token row stride; this lane's (head, slice) byte offset

    __device__ __forceinline__ void init(const AttnParams &p, int64_t t, int h, int lane)
    {
        g = lane / G;
        sub = lane % G;
        prm = &p;
        hoff = ((size_t)h * D + sub * PER) * sizeof(T);
        row_bytes = (size_t)p.H * D * sizeof(T);
        const char *Qp = reinterpret_cast<const char *>(p.Q) + (size_t)t * row_bytes + hoff;
#pragma unroll
        for (int c = 0; c < NC; ++c) qraw[c] = ldg16(Qp + 16 * c);
        sl2 = p.scale_log2;
#pragma unroll
        for (int e = 0; e < PER; ++e) o[e] = 0.f;
        m = -INFINITY;
        l = 0.f;
        n_edges = sum_j = sum_h = 0;
    }

    // this lane's slices of K_j and V_j (local buffer or the owning peer's)
    __device__ __forceinline__ void load(int64_t j, uint4 *kraw, uint4 *vraw) const
    {
        const char *kr, *vr;
        kv_row(*prm, j, row_bytes, kr, vr);
        kr += hoff;
        vr += hoff;
#pragma unroll
        for (int c = 0; c < NC; ++c) kraw[c] = ldg16(kr + 16 * c);
#pragma unroll
        for (int c = 0; c < NC; ++c) vraw[c] = ldg16(vr + 16 * c);
    }

    // q.k over the edge's G lanes, in the exp2 domain (scaled by log2(e)/sqrt(d))
    __device__ __forceinline__ float score(const uint4 *kraw) const
    {
        float s;
        if constexpr (H16) { // bf16 x bf16 + f32 without unpacking (FHFMA), 2 chains
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                a0 = fma2h<T>(qraw[c].x, kraw[c].x, a0);
                a1 = fma2h<T>(qraw[c].y, kraw[c].y, a1);
                a0 = fma2h<T>(qraw[c].z, kraw[c].z, a0);
                a1 = fma2h<T>(qraw[c].w, kraw[c].w, a1);
            }
            s = a0 + a1;
        } else {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                float qf[4], kf[4];
                unpack<T>(qraw[c], qf);
                unpack<T>(kraw[c], kf);
                a0 = fmaf(qf[0], kf[0], a0);
                a1 = fmaf(qf[1], kf[1], a1);
                a0 = fmaf(qf[2], kf[2], a0);
                a1 = fmaf(qf[3], kf[3], a1);
            }
            s = a0 + a1;
        }
#pragma unroll
        for (int off = 1; off < G; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        return s * sl2;
    }

    // one (key, value) edge into the lane group's state
    __device__ __forceinline__ void update(float s, const uint4 *vraw, bool valid, int64_t j)
    {
        if (!valid) return;
        if (s > m) { // lazy rescale: only when the running max grows
            const float a = ex2(m - s);
            l *= a;
#pragma unroll
            for (int e = 0; e < PER; ++e) o[e] *= a;
            m = s;
        }
        const float pr = ex2(s - m);
        l += pr;
        if constexpr (H16) { // o += p v with p rounded to the input type (as on the MMA paths)
            const uint32_t p2 = pack2<T>(pr, pr);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                axpy2h<T>(p2, vraw[c].x, o[8 * c + 0], o[8 * c + 1]);
                axpy2h<T>(p2, vraw[c].y, o[8 * c + 2], o[8 * c + 3]);
                axpy2h<T>(p2, vraw[c].z, o[8 * c + 4], o[8 * c + 5]);
                axpy2h<T>(p2, vraw[c].w, o[8 * c + 6], o[8 * c + 7]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                float vf[VEC];
                unpack<T>(vraw[c], vf);
#pragma unroll
                for (int e = 0; e < VEC; ++e) o[VEC * c + e] = fmaf(pr, vf[e], o[VEC * c + e]);
            }
        }
        if (PROBE) {
            n_edges += 1;
            sum_j += (unsigned long long)j;
            sum_h += splitmix64((uint64_t)j);
        }
    }

    // neighbours k in [kb, ke) of piece P (warp-uniform bounds): two edges per lane group
    // per step, both loads issued before either is consumed
    __device__ __forceinline__ void run(const Piece &P, int64_t kb, int64_t ke)
    {
        for (int64_t k0 = kb; k0 < ke; k0 += 2 * E) {
            const int64_t ka = k0 + g, kk = k0 + E + g;
            const bool va = ka < ke, vb = kk < ke;
            uint4 kra[NC], vra[NC], krb[NC], vrb[NC];
            int64_t ja = 0, jb = 0;
            if (va) {
                ja = piece_at(P, ka);
                load(ja, kra, vra);
            } else {
#pragma unroll
                for (int c = 0; c < NC; ++c) kra[c] = vra[c] = make_uint4(0, 0, 0, 0);
            }
            if (vb) {
                jb = piece_at(P, kk);
                load(jb, krb, vrb);
            } else {
#pragma unroll
                for (int c = 0; c < NC; ++c) krb[c] = vrb[c] = make_uint4(0, 0, 0, 0);
            }
            const float sa = score(kra);
            update(sa, vra, va, ja);
            if (k0 + E < ke) { // warp-uniform: some group has a second edge
                const float sb = score(krb);
                update(sb, vrb, vb, jb);
            }
        }
    }

    // Explicit CSR piece, gather-bound: a warp loads 32 column indices with one coalesced
    // load and broadcasts them to the lane groups by shuffle, then issues the K/V loads of
    // DEPTH edge steps before consuming any (DEPTH * E edges in flight per warp), so the
    // random row gathers overlap instead of waiting on dependent index loads.
    template <int DEPTH>
    __device__ __forceinline__ void run_csr(const int32_t *cols, int64_t kb, int64_t ke)
    {
        constexpr int STEP = E * DEPTH; // edges per pass
        const int lane = (int)(threadIdx.x & 31);
        for (int64_t b0 = kb; b0 < ke; b0 += 32) {
            const int64_t kl = b0 + lane;
            const int my_j = kl < ke ? cols[kl] : -1;
#pragma unroll 1
            for (int e0 = 0; e0 < 32 && b0 + e0 < ke; e0 += STEP) {
                uint4 kr[DEPTH][NC], vr[DEPTH][NC];
                int jj[DEPTH];
#pragma unroll
                for (int u = 0; u < DEPTH; ++u) {
                    const int src = e0 + u * E + g;
                    jj[u] = __shfl_sync(0xffffffffu, my_j, src & 31);
                    if (src >= 32) jj[u] = -1;
                    if (jj[u] >= 0) {
                        load(jj[u], kr[u], vr[u]);
                    } else {
#pragma unroll
                        for (int c = 0; c < NC; ++c) kr[u][c] = vr[u][c] = make_uint4(0, 0, 0, 0);
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
            for (int e = 0; e < PER; ++e) {
                const float o2 = __shfl_xor_sync(0xffffffffu, o[e], off);
                o[e] = o[e] * a + o2 * b;
            }
            m = mn;
        }
    }

    // normalise and store the row (lane group 0 holds the merged state)
    __device__ __forceinline__ void store(const AttnParams &p, int64_t t, int h) const
    {
        if (g != 0) return;
        const float inv = l > 0.f ? 1.f / l : 0.f;
        char *Op = reinterpret_cast<char *>(p.out) + (size_t)t * row_bytes + hoff;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            float r[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) r[e] = o[VEC * c + e] * inv;
            stg16(Op + 16 * c, pack<T>(r));
        }
    }

    // carried state (ga_state): write or (+)-combine the merged (m, l, o) of this call's
    // edges into the caller's buffers; with p.out also store the normalised row
    __device__ __forceinline__ void store_state(const AttnParams &p, int64_t t, int h)
    {
        const size_t rh = (size_t)t * p.H + h;
        float *so = p.state.o + rh * D + sub * PER;
        float mm = m, ll = l;
        if (g == 0 && p.state_mode == GA_STATE_ACCUMULATE) {
            const float l2 = p.state.l[rh];
            if (l2 > 0.f) { // l == 0 marks an empty state (its m is ignored)
                const float m2 = p.state.m[rh];
                const float mn = ll > 0.f ? fmaxf(mm, m2) : m2;
                const float a = ll > 0.f ? ex2(mm - mn) : 0.f, b = ex2(m2 - mn);
                ll = ll * a + l2 * b;
#pragma unroll
                for (int e = 0; e < PER; ++e) o[e] = o[e] * a + so[e] * b;
                mm = mn;
            }
        }
        __syncwarp(); // every lane has read the old state before any lane overwrites it
        if (g != 0) return;
        if (sub == 0) {
            p.state.m[rh] = mm;
            p.state.l[rh] = ll;
        }
#pragma unroll
        for (int e = 0; e < PER; ++e) so[e] = o[e];
        if (p.out) {
            l = ll;
            store(p, t, h);
        }
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

// edge steps a CSR batch issues before consuming (DEPTH * E edges in flight per warp)
template <typename T, int D> constexpr int csr_depth()
{
    return EdgeAcc<T, D, false>::E >= 16 ? 1 : 32 / EdgeAcc<T, D, false>::E > 4 ? 4 : 32 / EdgeAcc<T, D, false>::E;
}

// One (row, head) of Algorithm 1 by one warp: all pieces of N(i), merge, store.
// t = local query row (global row q_begin + t).
template <typename T, int D>
__device__ __forceinline__ void edge_row(const AttnParams &p, int64_t t, int h, int lane)
{
    EdgeAcc<T, D, false> acc;
    acc.init(p, t, h, lane);
    const int64_t i = p.q_begin + t;
    const int np = num_pieces_h(p.mask, i, h);
    for (int pc = 0; pc < np; ++pc) {
        const Piece P = get_piece_h(p.mask, i, pc, h);
        acc.run(P, 0, P.count);
    }
    acc.merge_groups();
    acc.store(p, t, h);
}

} // namespace ga

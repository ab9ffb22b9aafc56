/*
 * oracle.c — plain, slow, obviously-correct fp64 CPU oracle for graph-view masked
 * attention (arXiv 2502.01659, "Longer Attention Span").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2502_01659_b200/, libga.so) never links, imports or calls it, and this file
 * shares no header, helper, table or constant generator with the CUDA path.
 *
 * What it computes (the plain definition, DESIGN.md "Readings" R1-R22):
 *
 *   O[i,h,:] = sum_{j in N(i)} softmax_j(s_ij) * V[j,h,:],  s_ij = Q[i,h,:].K[j,h,:] / sqrt(d)
 *   O[i,h,:] = 0 when N(i) is empty.
 *
 *   Eq. (1) PAPER.md:71 gives softmax(QK^T/sqrt(d_k))V; the graph model
 *   says edge (i,j) exists iff A_ij = 1; Algorithm 1 restricts the
 *   sum to Get_Neighbors(G,i,P_a).  Because the method reaches exactly (up to rounding)
 *   the masked-softmax result (work-optimality paragraph), the oracle
 *   is that definition evaluated in two passes in fp64 with libm exp; it is NOT a replay
 *   of the method.  A literal Algorithm 1 replay (per-step division) is
 *   provided separately (orc_attention_alg1) so tests can check the two agree.
 *
 * Neighbour sets N(i) are enumerated from the mask DEFINITIONS (PAPER.md:124-158,
 * 232-235) — predicate/union form, sorted ascending — never from the GPU's closed-form
 * index arithmetic:
 *   WINDOW(w,r)          |i-j| < w  and  |i-j| mod r == 0          (reading R1,R2)
 *   BLOCK_DILATED(seg,r) floor(i/seg)==floor(j/seg) and (i mod seg) mod r == 0 and
 *                        (j mod seg) mod r == 0                      (reading R3)
 *   LONGNET(w0,alpha)    OR over k = 0..K of BLOCK_DILATED(w0*alpha^k, alpha^k),
 *                        K = max{k : w0*alpha^k <= L}                (reading R11);
 *                        parts = 1: the multiset union (a pair in n levels' blocks listed n
 *                        times, so it weighs n times in the softmax; reading R11b)
 *   BIGBIRD(w,G,nr,seed) global rows/cols UNION window(w) UNION random
 *                        columns drawn by the counter hash of reading R10.
 *                        The window may be dilated (r: |i-j| < w and |i-j| mod r == 0, as
 *                        WINDOW).  `parts` selects disjoint components (bit 0 window, bit 1
 *                        global rows/cols minus the window — the paper's "global minus local"
 *                        kernel, PAPER.md:235 —, bit 2 random; 0 = all): the composition
 *                        API of SURVEY §8(f) f1 runs them as separate calls.
 *   CSR                  the given row_ptr/col_idx
 *
 * Seeded inputs (reading R22) are regenerated on demand from the counter hash so the
 * oracle never needs the full Q/K/V of a 160M-token configuration.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------------ */
/* Mask description (oracle-private; deliberately NOT include/ga.h)                 */
/* ------------------------------------------------------------------------------ */
enum { ORC_CSR = 0, ORC_WINDOW = 1, ORC_LONGNET = 2, ORC_BIGBIRD = 3, ORC_BLOCK_DILATED = 4 };

typedef struct {
    int64_t kind;
    int64_t L;
    const int64_t *row_ptr; /* CSR, host */
    const int32_t *col_idx; /* CSR, host */
    int64_t w, r;           /* window / dilation                               */
    int64_t w0, alpha;      /* LongNet                                          */
    int64_t seg;            /* block-dilated segment length                     */
    const int64_t *global_idx; /* BigBird global tokens, sorted; NULL = evenly spaced */
    int64_t n_global;
    int64_t n_random;
    uint64_t seed;
    int64_t parts;          /* BigBird components (0 = all); LongNet: bit 0 multiset,
                               bit 1 per-head offsets (reading R11c)              */
    int64_t head;           /* LongNet per-head offsets: the head whose set N(i) is enumerated */
} orc_mask;

enum { ORC_F32 = 0, ORC_BF16 = 1, ORC_F16 = 2, ORC_F64 = 3 };

/* ------------------------------------------------------------------------------ */
/* Counter-based generator (reading R22; golden values in tests/golden/rng.txt)     */
/* ------------------------------------------------------------------------------ */
uint64_t orc_splitmix64(uint64_t x)
{
    /* SplitMix64 output function applied to state x + golden gamma (Steele et al. 2014;
       splitmix64(0) is the generator's well-known first output 0xe220a8397b1dcdaf). */
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static float orc_u01(uint64_t seed, int tensor, uint64_t e)
{
    uint64_t u = orc_splitmix64(orc_splitmix64(seed + (uint64_t)tensor) ^ e);
    return (float)(u >> 40) * (1.0f / 16777216.0f); /* exact: 24-bit integer * 2^-24 */
}

static double orc_round_to(float x, int dtype)
{
    if (dtype == ORC_BF16) {
        uint32_t b;
        memcpy(&b, &x, 4);
        b += 0x7fffu + ((b >> 16) & 1u); /* round to nearest even on the dropped 16 bits */
        b &= 0xffff0000u;
        float y;
        memcpy(&y, &b, 4);
        return (double)y;
    }
    if (dtype == ORC_F16) {
        _Float16 h = (_Float16)x; /* C conversion: round-to-nearest-even incl. subnormals */
        return (double)h;
    }
    return (double)x;
}

/* Stored value of element e of tensor tau (0=Q, 1=K, 2=V), upcast exactly to fp64. */
double orc_input_value(uint64_t seed, int tensor, uint64_t e, int dtype)
{
    return orc_round_to(orc_u01(seed, tensor, e), dtype);
}

void orc_fill_inputs(uint64_t seed, int tensor, uint64_t e0, int64_t n, int dtype, double *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n; ++t) out[t] = orc_input_value(seed, tensor, e0 + (uint64_t)t, dtype);
}

/* ------------------------------------------------------------------------------ */
/* Neighbour enumeration from the definitions                                      */
/* ------------------------------------------------------------------------------ */
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static int64_t sort_unique(int64_t *v, int64_t n)
{
    if (n <= 1) return n;
    qsort(v, (size_t)n, sizeof(int64_t), cmp_i64);
    int64_t k = 1;
    for (int64_t t = 1; t < n; ++t)
        if (v[t] != v[k - 1]) v[k++] = v[t];
    return k;
}

static int64_t i64abs(int64_t x) { return x < 0 ? -x : x; }

/* Global token set G: given list, or the evenly spaced reading R9: G = {floor(k*L/g)}. */
static int64_t global_at(const orc_mask *m, int64_t k)
{
    if (m->global_idx) return m->global_idx[k];
    return (int64_t)(((__int128)k * m->L) / m->n_global);
}

static int is_global(const orc_mask *m, int64_t j)
{
    for (int64_t k = 0; k < m->n_global; ++k)
        if (global_at(m, k) == j) return 1;
    return 0;
}

static int in_window(int64_t i, int64_t j, int64_t w) { return i64abs(i - j) < w; }

/* BigBird's window: WINDOW(w, r) (r = 1 unless dilated) */
static int bb_in_window(const orc_mask *m, int64_t i, int64_t j)
{
    int64_t r = m->r > 0 ? m->r : 1;
    return i64abs(i - j) < m->w && i64abs(i - j) % r == 0;
}

/* LongNet level count K = max{k : w0 * alpha^k <= L} (reading R11). */
int64_t orc_longnet_levels(int64_t w0, int64_t alpha, int64_t L)
{
    int64_t K = 0;
    __int128 seg = w0;
    if (seg > L) return 0; /* level 0 always exists (a single partial segment) */
    while (seg * alpha <= L) { seg *= alpha; ++K; }
    return K;
}

/* Upper bound on the degree of any row (for buffer sizing). */
int64_t orc_max_degree(const orc_mask *m)
{
    int64_t L = m->L;
    switch (m->kind) {
    case ORC_CSR: {
        int64_t mx = 0;
        for (int64_t i = 0; i < L; ++i) {
            int64_t d = m->row_ptr[i + 1] - m->row_ptr[i];
            if (d > mx) mx = d;
        }
        return mx;
    }
    case ORC_WINDOW: return 2 * m->w + 1;
    case ORC_BLOCK_DILATED: return m->seg + 1;
    case ORC_LONGNET: return (orc_longnet_levels(m->w0, m->alpha, L) + 1) * (m->w0 + 1);
    case ORC_BIGBIRD: return L + m->n_global + 2 * m->w + 1; /* pre-dedup union size */
    }
    return L;
}

/* BigBird random columns of non-global row i (reading R10): candidates
 *   c_t = floor((splitmix64(splitmix64(seed) ^ (i*2^20 + t)) >> 32) * L / 2^32),  t = 0,1,...
 * accepted in order when not yet accepted and outside window(i) UNION G, until n_random are
 * accepted or the complement of window UNION G is exhausted (then all of it is taken). */
static int64_t bigbird_random(const orc_mask *m, int64_t i, int64_t *out)
{
    int64_t L = m->L;
    /* size of W_i UNION G: the window predicate over the only j that can pass, plus the
       globals outside it */
    int64_t lo = i - m->w + 1 < 0 ? 0 : i - m->w + 1;
    int64_t hi = i + m->w - 1 > L - 1 ? L - 1 : i + m->w - 1;
    int64_t wg = 0;
    for (int64_t j = lo; j <= hi; ++j)
        if (bb_in_window(m, i, j)) ++wg;
    for (int64_t k = 0; k < m->n_global; ++k)
        if (!bb_in_window(m, i, global_at(m, k))) ++wg;
    int64_t complement = L - wg;
    if (complement <= m->n_random) {
        int64_t n = 0;
        for (int64_t j = 0; j < L; ++j)
            if (!bb_in_window(m, i, j) && !is_global(m, j)) out[n++] = j;
        return n;
    }
    uint64_t base = orc_splitmix64(m->seed);
    int64_t n = 0;
    for (uint64_t t = 0; n < m->n_random; ++t) {
        uint64_t h = orc_splitmix64(base ^ ((uint64_t)i * (1ULL << 20) + t));
        int64_t c = (int64_t)(((__int128)(h >> 32) * L) >> 32);
        if (bb_in_window(m, i, c) || is_global(m, c)) continue;
        int dup = 0;
        for (int64_t q = 0; q < n; ++q)
            if (out[q] == c) { dup = 1; break; }
        if (!dup) out[n++] = c;
    }
    return n;
}

/* N(i), ascending, into out (capacity >= orc_max_degree). Returns |N(i)|. */
int64_t orc_row_neighbors(const orc_mask *m, int64_t i, int64_t *out)
{
    int64_t L = m->L, n = 0;
    switch (m->kind) {
    case ORC_CSR:
        for (int64_t e = m->row_ptr[i]; e < m->row_ptr[i + 1]; ++e) out[n++] = m->col_idx[e];
        return n;
    case ORC_WINDOW: {
        /* predicate |i-j| < w && |i-j| mod r == 0, scanned over the only j that can pass */
        int64_t lo = i - m->w + 1 < 0 ? 0 : i - m->w + 1;
        int64_t hi = i + m->w - 1 > L - 1 ? L - 1 : i + m->w - 1;
        for (int64_t j = lo; j <= hi; ++j)
            if (i64abs(i - j) < m->w && i64abs(i - j) % m->r == 0) out[n++] = j;
        return n;
    }
    case ORC_BLOCK_DILATED: {
        int64_t s = m->seg, b = i / s;
        if ((i % s) % m->r != 0) return 0;
        for (int64_t j = b * s; j < (b + 1) * s && j < L; ++j)
            if (j / s == b && (j % s) % m->r == 0) out[n++] = j;
        return n;
    }
    case ORC_LONGNET: {
        /* union over levels k of BlockDilated(seg_k = w0*alpha^k, r_k = alpha^k); with per-head
           offsets (parts bit 1, reading R11c: LongNet's s_j = j mod r) head h keeps the
           in-segment offsets congruent to h mod r_k instead of 0 */
        int64_t K = orc_longnet_levels(m->w0, m->alpha, L);
        int64_t seg = m->w0, r = 1;
        for (int64_t k = 0; k <= K; ++k) {
            int64_t b = i / seg, off = (m->parts & 2) ? m->head % r : 0;
            if ((i % seg) % r == off)
                for (int64_t j = b * seg + off; j < (b + 1) * seg && j < L; j += r)
                    if ((j % seg) % r == off) out[n++] = j;
            seg *= m->alpha;
            r *= m->alpha;
        }
        if (m->parts & 1) { /* multiset union (LongNet's mixture, reading R11b): keep repeats */
            if (n > 1) qsort(out, (size_t)n, sizeof(int64_t), cmp_i64);
            return n;
        }
        return sort_unique(out, n);
    }
    case ORC_BIGBIRD: {
        int64_t parts = m->parts ? m->parts : 7;
        if (is_global(m, i)) { /* a global token attends to every token */
            for (int64_t j = 0; j < L; ++j) {
                int w = bb_in_window(m, i, j);
                if ((w && (parts & 1)) || (!w && (parts & 2))) out[n++] = j;
            }
            return n;
        }
        if (parts & 1) {                                                       /* window  */
            int64_t lo = i - m->w + 1 < 0 ? 0 : i - m->w + 1;
            int64_t hi = i + m->w - 1 > L - 1 ? L - 1 : i + m->w - 1;
            for (int64_t j = lo; j <= hi; ++j)
                if (bb_in_window(m, i, j)) out[n++] = j;
        }
        if (parts & 2)                                              /* global columns \ W */
            for (int64_t k = 0; k < m->n_global; ++k)
                if (!bb_in_window(m, i, global_at(m, k))) out[n++] = global_at(m, k);
        if (parts & 4) n += bigbird_random(m, i, out + n);                     /* random  */
        return sort_unique(out, n);
    }
    }
    return 0;
}

/* Masks whose neighbour sets depend on the head (LongNet per-head offsets). */
static int per_head(const orc_mask *m) { return m->kind == ORC_LONGNET && (m->parts & 2); }

/* N(i) of head h. */
int64_t orc_row_neighbors_head(const orc_mask *m, int64_t i, int64_t h, int64_t *out)
{
    orc_mask mh = *m;
    mh.head = h;
    return orc_row_neighbors(&mh, i, out);
}

/* Exact nnz and row_ptr (exclusive scan of degrees) / col_idx.  col_idx may be NULL. */
int64_t orc_mask_to_csr(const orc_mask *m, int64_t *row_ptr, int32_t *col_idx)
{
    int64_t L = m->L;
    int64_t cap = orc_max_degree(m);
    int64_t *deg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(L > 0 ? L : 1));
#pragma omp parallel
    {
        int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + 1));
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < L; ++i) deg[i] = orc_row_neighbors(m, i, buf);
        free(buf);
    }
    int64_t acc = 0;
    for (int64_t i = 0; i < L; ++i) {
        if (row_ptr) row_ptr[i] = acc;
        acc += deg[i];
    }
    if (row_ptr) row_ptr[L] = acc;
    if (col_idx && row_ptr) {
#pragma omp parallel
        {
            int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + 1));
#pragma omp for schedule(dynamic, 64)
            for (int64_t i = 0; i < L; ++i) {
                int64_t n = orc_row_neighbors(m, i, buf);
                for (int64_t t = 0; t < n; ++t) col_idx[row_ptr[i] + t] = (int32_t)buf[t];
            }
            free(buf);
        }
    }
    free(deg);
    return acc;
}

/* ------------------------------------------------------------------------------ */
/* Attention                                                                        */
/* ------------------------------------------------------------------------------ */
/* Input source: explicit fp64 arrays [L,H,d] (q/k/v non-NULL) or the seeded generator
 * (seed, dtype) when the arrays are NULL. */
typedef struct {
    const double *q, *k, *v;
    uint64_t seed;
    int64_t dtype;
    int64_t kv_rows; /* reserved */
} orc_inputs;

static void load_row(const orc_inputs *in, int tensor, int64_t tok, int64_t h, int64_t H, int64_t d,
                     double *dst)
{
    const double *src = tensor == 0 ? in->q : tensor == 1 ? in->k : in->v;
    uint64_t e0 = ((uint64_t)tok * (uint64_t)H + (uint64_t)h) * (uint64_t)d;
    if (src) {
        memcpy(dst, src + e0, sizeof(double) * (size_t)d);
    } else {
        for (int64_t c = 0; c < d; ++c) dst[c] = orc_input_value(in->seed, tensor, e0 + (uint64_t)c, (int)in->dtype);
    }
}

/* Two-pass masked softmax attention for the listed rows (rows == NULL: all L rows).
 * out: [nrows, H, d] fp64.  Returns the number of edges (sum of |N(i)| over rows, x H). */
int64_t orc_attention(const orc_inputs *in, const orc_mask *m, int64_t H, int64_t d, const int64_t *rows,
                      int64_t nrows, double *out)
{
    int64_t cap = orc_max_degree(m);
    int64_t edges = 0;
    double inv_sqrt_d = 1.0 / sqrt((double)d); /* Eq. (1) scale; reading R4 */
#pragma omp parallel reduction(+ : edges)
    {
        int64_t *nb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + 1));
        double *s = (double *)malloc(sizeof(double) * (size_t)(cap + 1));
        double *q = (double *)malloc(sizeof(double) * (size_t)d);
        double *kv = (double *)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < nrows; ++t) {
            int64_t i = rows ? rows[t] : t;
            int64_t n = orc_row_neighbors(m, i, nb);
            for (int64_t h = 0; h < H; ++h) {
                double *o = out + ((size_t)t * (size_t)H + (size_t)h) * (size_t)d;
                for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
                if (per_head(m)) n = orc_row_neighbors_head(m, i, h, nb);
                if (n == 0) continue; /* empty row -> 0 (reading R6) */
                load_row(in, 0, i, h, H, d, q);
                double mx = -INFINITY;
                for (int64_t e = 0; e < n; ++e) { /* pass 1: scores and their max */
                    load_row(in, 1, nb[e], h, H, d, kv);
                    double acc = 0.0;
                    for (int64_t c = 0; c < d; ++c) acc += q[c] * kv[c];
                    s[e] = acc * inv_sqrt_d;
                    if (s[e] > mx) mx = s[e];
                }
                double z = 0.0;
                for (int64_t e = 0; e < n; ++e) { /* pass 2: weights and weighted sum of V */
                    double p = exp(s[e] - mx);
                    z += p;
                    load_row(in, 2, nb[e], h, H, d, kv);
                    for (int64_t c = 0; c < d; ++c) o[c] += p * kv[c];
                }
                for (int64_t c = 0; c < d; ++c) o[c] /= z;
                edges += n;
            }
        }
        free(nb); free(s); free(q); free(kv);
    }
    return edges;
}

/* Literal Algorithm 1 in fp64, with the 1/sqrt(d) of Eq. (1):
 * per neighbour j (ascending): W = Q_i.K_j / sqrt(d); m_new = max(m, W);
 * l_new = l*exp(m - m_new) + exp(W - m_new);
 * O_i = (1/l_new) * [ l*exp(m - m_new)*O_i + exp(W - m_new)*V_j ];  l = l_new; m = m_new.
 * The first neighbour uses exp(-inf) = 0. */
int64_t orc_attention_alg1(const orc_inputs *in, const orc_mask *m, int64_t H, int64_t d, const int64_t *rows,
                           int64_t nrows, double *out)
{
    int64_t cap = orc_max_degree(m);
    int64_t edges = 0;
    double inv_sqrt_d = 1.0 / sqrt((double)d);
#pragma omp parallel reduction(+ : edges)
    {
        int64_t *nb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + 1));
        double *q = (double *)malloc(sizeof(double) * (size_t)d);
        double *kv = (double *)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < nrows; ++t) {
            int64_t i = rows ? rows[t] : t;
            int64_t n = orc_row_neighbors(m, i, nb);
            for (int64_t h = 0; h < H; ++h) {
                double *o = out + ((size_t)t * (size_t)H + (size_t)h) * (size_t)d;
                for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
                if (per_head(m)) n = orc_row_neighbors_head(m, i, h, nb);
                load_row(in, 0, i, h, H, d, q);
                double mi = -INFINITY, li = 0.0;
                for (int64_t e = 0; e < n; ++e) {
                    load_row(in, 1, nb[e], h, H, d, kv);               /* Pull(K_j) */
                    double W = 0.0;
                    for (int64_t c = 0; c < d; ++c) W += q[c] * kv[c];
                    W *= inv_sqrt_d;
                    double mnew = mi > W ? mi : W;
                    double a = (mi == -INFINITY) ? 0.0 : exp(mi - mnew);
                    double b = exp(W - mnew);
                    double lnew = li * a + b;
                    load_row(in, 2, nb[e], h, H, d, kv);               /* Pull(V_j) */
                    for (int64_t c = 0; c < d; ++c) o[c] = (li * a * o[c] + b * kv[c]) / lnew;
                    li = lnew;
                    mi = mnew;
                }
                edges += n;
            }
        }
        free(nb); free(q); free(kv);
    }
    return edges;
}

/* Backward pass (the training use case of PAPER.md:555) — the chain rule of
 * O_i = sum_{e in N(i)} P_e V_{j_e}, P_e = softmax_e(S_e), S_e = Q_i.K_{j_e} / sqrt(d), written
 * out per edge e = (i, j) of the (multi)set N(i) in fp64, for upstream gradients dO [L,H,d]:
 *     dV_j += P_e dO_i                       dP_e = dO_i . V_j
 *     D_i   = sum_e P_e dP_e                 dS_e = P_e (dP_e - D_i)      (softmax Jacobian)
 *     dQ_i += dS_e K_j / sqrt(d)             dK_j += dS_e Q_i / sqrt(d)
 * Serial over rows (dK, dV are scattered): small cases only.  dq, dk, dv: [L,H,d], zeroed
 * here.  Empty rows contribute nothing (their O is the constant 0, reading R6).  Returns the
 * number of edges x H.  PARITY PINS: central finite differences of orc_attention and torch
 * autograd of the dense masked softmax (tests/test_oracle_pins.py). */
int64_t orc_attention_backward(const orc_inputs *in, const orc_mask *m, int64_t H, int64_t d, const double *dout,
                               double *dq, double *dk, double *dv)
{
    const int64_t L = m->L, cap = orc_max_degree(m);
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    int64_t edges = 0;
    int64_t *nb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap + 1));
    double *P = (double *)malloc(sizeof(double) * (size_t)(cap + 1));
    double *dP = (double *)malloc(sizeof(double) * (size_t)(cap + 1));
    double *q = (double *)malloc(sizeof(double) * (size_t)d);
    double *kv = (double *)malloc(sizeof(double) * (size_t)d);
    memset(dq, 0, sizeof(double) * (size_t)(L * H * d));
    memset(dk, 0, sizeof(double) * (size_t)(L * H * d));
    memset(dv, 0, sizeof(double) * (size_t)(L * H * d));
    for (int64_t i = 0; i < L; ++i) {
        int64_t n = orc_row_neighbors(m, i, nb);
        for (int64_t h = 0; h < H; ++h) {
            if (per_head(m)) n = orc_row_neighbors_head(m, i, h, nb);
            if (n == 0) continue;
            const size_t ri = ((size_t)i * (size_t)H + (size_t)h) * (size_t)d;
            const double *g = dout + ri;
            load_row(in, 0, i, h, H, d, q);
            double mx = -INFINITY;
            for (int64_t e = 0; e < n; ++e) { /* scores S_e, kept in P */
                load_row(in, 1, nb[e], h, H, d, kv);
                double acc = 0.0;
                for (int64_t c = 0; c < d; ++c) acc += q[c] * kv[c];
                P[e] = acc * inv_sqrt_d;
                if (P[e] > mx) mx = P[e];
            }
            double z = 0.0;
            for (int64_t e = 0; e < n; ++e) { P[e] = exp(P[e] - mx); z += P[e]; }
            double D = 0.0;
            for (int64_t e = 0; e < n; ++e) {
                P[e] /= z;
                load_row(in, 2, nb[e], h, H, d, kv);
                double acc = 0.0;
                for (int64_t c = 0; c < d; ++c) acc += g[c] * kv[c];
                dP[e] = acc;
                D += P[e] * dP[e];
                double *dvj = dv + ((size_t)nb[e] * (size_t)H + (size_t)h) * (size_t)d;
                for (int64_t c = 0; c < d; ++c) dvj[c] += P[e] * g[c];
            }
            for (int64_t e = 0; e < n; ++e) {
                const double dS = P[e] * (dP[e] - D);
                load_row(in, 1, nb[e], h, H, d, kv);
                double *dkj = dk + ((size_t)nb[e] * (size_t)H + (size_t)h) * (size_t)d;
                for (int64_t c = 0; c < d; ++c) {
                    dq[ri + (size_t)c] += dS * kv[c] * inv_sqrt_d;
                    dkj[c] += dS * q[c] * inv_sqrt_d;
                }
            }
            edges += n;
        }
    }
    free(nb); free(P); free(dP); free(q); free(kv);
    return edges;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

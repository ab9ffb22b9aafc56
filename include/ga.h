/*
 * ga.h — C ABI of libga.so: B200-native graph-view masked attention
 * (Tomczak & Kuppannagari, "Longer Attention Span", arXiv 2502.01659).
 *
 * Tokens are graph nodes and attention-mask nonzeros are directed edges
 * (§4.1 "Modeling").  For every query node i and every edge (i,j) the
 * library computes, in ONE fused pass per row (Algorithm 1):
 *
 *     s_ij = q_i . k_j / sqrt(d)                       (Eq. 1; reading R4)
 *     m_i, l_i  <- online softmax over j in N(i)        (Alg. 1)
 *     o_i   = sum_j exp(s_ij - m_i) v_j / l_i           (Alg. 1; deferred /l, R5)
 *     o_i   = 0 if N(i) is empty                        (Alg. 1 init; R6)
 *
 * and never forms the L x L matrix: only the nnz(mask) dot products are computed
 * ("work optimal").
 *
 * Conventions for every entry point
 *   Layout      Q, K, V, out are row-major [tokens, heads, d] ("BSHD" with B = 1): element
 *               (t, h, c) lives at ((t*heads + h)*d + c).  Rows must be 16-byte aligned.
 *   Dtypes      fp32 / bf16 / fp16 storage; all arithmetic in fp32 (reading R15); the
 *               output is rounded to the input dtype (RNE).
 *   d           32, 64 or 128.
 *   Ownership   every pointer is caller-owned; the library never frees or retains
 *               anything past the call (device memory comes from torch / cudaMalloc).
 *   Streams     `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *               stream).  All device work is enqueued on it; no entry point synchronises
 *               the device unless its comment says so.
 *   Errors      a ga_status is returned; GA_OK = 0.  Argument errors are detected
 *               synchronously before anything is enqueued.  Launch errors are caught with
 *               cudaPeekAtLastError (GA_ERR_CUDA).  Device faults surface at the
 *               caller's next synchronisation.  ga_last_error() returns a thread-local
 *               message describing the last non-OK status.  No exceptions cross the ABI
 *               and the library never aborts the process.
 */
#ifndef GA_H
#define GA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GA_OK = 0,
    GA_ERR_INVALID_ARG = -1, /* bad pointer / shape / parameter / alignment          */
    GA_ERR_UNSUPPORTED = -2, /* valid but not implemented (e.g. d not in {32,64,128}) */
    GA_ERR_CUDA = -3,        /* a CUDA runtime call or kernel launch failed           */
    GA_ERR_COMM = -4,        /* multi-GPU bootstrap / exchange failed (ga_comm_*)      */
    GA_ERR_OOM = -5,         /* workspace too small / allocation failed               */
    GA_ERR_MASK = -6         /* ga_mask_validate found a malformed CSR                */
} ga_status;

typedef enum { GA_F32 = 0, GA_BF16 = 1, GA_F16 = 2 } ga_dtype;

/* Mask families (§4.2 list, :224-237; SURVEY §8(c) readings). */
typedef enum {
    /* explicit binary CSR: row_ptr int64 [L+1], col_idx int32 [nnz], columns of each row
       strictly increasing (reading R7 — no values vector). */
    GA_MASK_CSR = 0,
    /* |i-j| < w  and  |i-j| mod r == 0: local window (r = 1) and 1D
       dilated window (readings R1, R2). */
    GA_MASK_WINDOW = 1,
    /* LongNet exponentially dilated: OR over k = 0..K of BLOCK_DILATED(w0*alpha^k, alpha^k),
       K = max{k : w0*alpha^k <= L} (reading R11).  With
       parts = GA_LONGNET_MULTISET: the multiset union instead — an edge in n levels' blocks
       counts n times in the softmax (LongNet's own mixture); runs on the
       edge kernel; its CSR (ga_mask_to_csr) repeats such columns (not strictly increasing,
       so ga_mask_validate rejects it, while every attention kernel accepts it). */
    GA_MASK_LONGNET = 2,
    /* BigBird / Longformer: window(w) UNION global rows and columns UNION n_random random
       columns per non-global row (readings R8-R10).  Materialise with
       ga_mask_to_csr; ga_attention rejects it (GA_ERR_UNSUPPORTED) — the paper itself runs
       the composed mask through the CSR kernel. */
    GA_MASK_BIGBIRD = 3,
    /* 2D dilation: floor(i/seg)==floor(j/seg) and (i mod seg) mod r == 0 and
       (j mod seg) mod r == 0 (reading R3). */
    GA_MASK_BLOCK_DILATED = 4
} ga_mask_kind;

/* BIGBIRD components (ga_mask.parts): the window W_i, the global rows and columns minus the
   window (the paper's "global minus local" kernel), the random columns.  They
   are disjoint and their union is the BigBird mask; Longformer = WINDOW + GLOBAL. */
typedef enum { GA_BB_WINDOW = 1, GA_BB_GLOBAL = 2, GA_BB_RANDOM = 4 } ga_bigbird_part;
/* LONGNET variants (ga_mask.parts bits):
   GA_LONGNET_MULTISET     LongNet's multiset mixture (reading R11b);
   GA_LONGNET_HEAD_OFFSETS per-head offsets (reading R11c, LongNet's s_j = j mod r): head h
                           keeps, at level k, the positions whose in-segment offset is
                           congruent to h modulo alpha^k (instead of 0), so each head has its
                           own edge set.  Runs on the edge kernel (forward and backward);
                           ga_mask_count / ga_mask_to_csr return GA_ERR_UNSUPPORTED. */
enum { GA_LONGNET_MULTISET = 1, GA_LONGNET_HEAD_OFFSETS = 2 };

/* Mask descriptor: the paper's "attention-specific parameters P_a" or explicit graph G
   (Algorithm 1 input).  Unused fields are ignored; zero-initialise. */
typedef struct ga_mask {
    int32_t kind;              /* ga_mask_kind                                          */
    int32_t parts;             /* BIGBIRD components to include (ga_bigbird_part bits; 0 =
                                  all): disjoint, so separate calls compose.
                                  LONGNET: 0 = set union, GA_LONGNET_MULTISET = multiset */
    int64_t L;                 /* number of graph nodes (global sequence length)         */
    const int64_t *row_ptr;    /* CSR: DEVICE int64 [L+1], row_ptr[0]=0, nondecreasing     */
    const int32_t *col_idx;    /* CSR: DEVICE int32 [nnz], sorted strictly per row        */
    int64_t nnz;               /* CSR: number of edges (= row_ptr[L])                     */
    int64_t w, r;              /* WINDOW / BIGBIRD window w >= 1; dilation r >= 1 (BIGBIRD:
                                  0 = 1; its window is WINDOW(w, r))                        */
    int64_t w0, alpha;         /* LONGNET: first segment w0 >= 1, ratio alpha >= 2         */
    int64_t seg;               /* BLOCK_DILATED segment length >= 1 (r as above)          */
    const int64_t *global_idx; /* BIGBIRD: DEVICE int64 [n_global] sorted, or NULL for the
                                  evenly spaced set {floor(k*L/n_global)} (reading R9)    */
    int64_t n_global;          /* BIGBIRD global token count                             */
    int64_t n_random;          /* BIGBIRD random columns per non-global row (<= 320)     */
    uint64_t seed;             /* BIGBIRD random-column seed (reading R10)                */
} ga_mask;

/* Kernel selection (ga_opts.kernel). AUTO picks the fastest kernel implemented for the
   (mask, dtype, d) triple; the others force one path (tests compare them). */
typedef enum {
    GA_KERNEL_AUTO = 0,
    GA_KERNEL_EDGE = 1,  /* generic warp-per-(row,head) edge traversal, every family, every dtype */
    GA_KERNEL_TILED = 2, /* bf16/fp16 tensor-core kernel of the family: WINDOW -> band kernel
                            (K/V band in shared memory, mma.sync on fully dense 16x16 blocks,
                            CUDA cores on the partial triangles); LONGNET -> dense-group kernel
                            (rows sharing a neighbour set x their strided key pieces) */
    GA_KERNEL_TC = 3     /* bf16/fp16 tcgen05 (TMEM accumulator) kernel of the family, d = 64:
                            WINDOW with 64 <= m <= 128, r <= 4 -> persistent band kernel (128-row
                            query tiles x 64-key chunks, masked per row; window_tc.cu); LONGNET ->
                            dense groups on tcgen05 + the rest on mma.sync */
} ga_kernel;

/* Carried online-softmax state: for query row i and head h over an edge
   set E (the edges of one call),
       m = max_{j in E} s_ij * log2(e)          (log2 domain; s_ij = q_i.k_j / sqrt(d))
       l = sum_{j in E} 2^(s_ij log2(e) - m)
       o = sum_{j in E} 2^(s_ij log2(e) - m) v_j (fp32, unnormalised)
   Two states of DISJOINT edge sets combine with the associative operator of PAPER.md:374's
   split-and-merge (a7): m = max(m1, m2), l = l1 2^(m1-m) + l2 2^(m2-m), o likewise; the
   attention over the union is o / l (0 when l = 0).  A state with l = 0 is empty (its m is
   ignored), so zero-filled buffers are valid empty states.  Layout: DEVICE fp32, m and l
   [rows, heads], o [rows, heads, d], row-major; rows are the call's query rows. */
typedef struct ga_state {
    float *m;
    float *l;
    float *o;
} ga_state;

typedef enum { GA_STATE_WRITE = 0, GA_STATE_ACCUMULATE = 1 } ga_state_mode;

/* Optional controls for ga_attention_ex.  Zero-initialise, then set what you need. */
typedef struct ga_opts {
    /* Query-range sharding: process global query rows
       [q_begin, q_begin + q_rows).  Q and out hold exactly those rows (row 0 = q_begin).
       q_rows = 0 means L - q_begin. */
    int64_t q_begin, q_rows;
    /* K and V hold global token rows [kv_begin, kv_begin + kv_rows); every neighbour of
       every processed row must lie inside (halo / all-gather responsibility of the caller).
       kv_rows = 0 means L - kv_begin. */
    int64_t kv_begin, kv_rows;
    /* Device workspace, size from ga_workspace_size: needed by CSR inputs with rows above
       the heavy-row threshold; optional for LONGNET bf16/fp16 d=64 (partial states of the
       tcgen05 block path — without it the library takes stream-ordered scratch from its
       private per-device memory pool (cudaMallocFromPoolAsync; freed blocks stay cached in
       that pool, the device's default pool is not modified)). */
    void *workspace;
    size_t workspace_bytes;
    /* Debug / work-optimality probes ("probe build").  When non-NULL a slower
       instrumented kernel runs (the edge kernel; for bf16/fp16 d = 64 windows with only
       edge_counter set, the production tcgen05 window kernel — see tensor_counter):
         edge_counter      DEVICE u64, atomically += number of q.k dot products computed
         row_fingerprint   DEVICE u64 [q_rows*3]: per processed row (head 0): degree,
                           sum of j, sum of splitmix64(j), all mod 2^64. */
    unsigned long long *edge_counter;
    unsigned long long *row_fingerprint;
    int32_t kernel;          /* ga_kernel */
    int32_t heavy_threshold; /* CSR rows with more edges are split into chunks of this size
                                and merged (0 = default 4096) */
    /* Carried state (state.m != NULL): the call also produces the (m, l, o) state of its
       edges, overwriting (GA_STATE_WRITE) or (+)-combining into (GA_STATE_ACCUMULATE) the
       buffers; `out` may then be NULL, otherwise it receives the normalised attention of the
       resulting state.  Runs on the edge kernel (every family); not with the CSR heavy-row
       split (no workspace). */
    ga_state state;
    int32_t state_mode;      /* ga_state_mode */
    /* ga_attention_sharded with an explicit CSR mask: how K/V reach the ranks (SURVEY §8(e),
       §8(f) f2).  GA_EXCHANGE_ALLGATHER (0): every rank gathers the full [L, heads, d] K and V
       (memory 2 L per rank: the context cap does not grow with the rank count).
       GA_EXCHANGE_RING (1): the key dimension is cut into the ranks' shards; rank r streams
       shard (r + s) mod world for s = 0..world-1 through two staging buffers (peer -> local
       copy of the next shard overlapped with the current one's compute), each step computing
       its rows' edges into that shard's key range only and (+)-merging the carried state
       (memory ~6 L / world per rank).  Ignored elsewhere. */
    int32_t exchange;
    /* Probe of the tcgen05 window kernel (with edge_counter and without row_fingerprint the
       window kernel itself is probed instead of the instrumented edge kernel):
         tensor_counter    DEVICE u64, += q.k products the tensor cores computed (whole
                           128 x 64 MMA tiles, masked pairs included: reading R23)
       edge_counter then counts the (row, key) pairs that received a softmax weight (the
       band's edges: nnz x heads when the kernel is work-exact in its weights). */
    unsigned long long *tensor_counter;
} ga_opts;

enum { GA_EXCHANGE_ALLGATHER = 0, GA_EXCHANGE_RING = 1 };

/* The north-star entry point: O = masked-softmax attention of (Q,K,V) over mask.
   Q,K,V,out: DEVICE [L, heads, d] in `dtype`.  `out` must not alias K or V; it may alias
   Q only for implicit masks (one launch owns each row).  Returns GA_ERR_UNSUPPORTED for
   GA_MASK_BIGBIRD (use ga_mask_to_csr) and for CSR masks whose rows exceed the heavy-row
   threshold (those need ga_attention_ex with a workspace). */
ga_status ga_attention(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out,
                       int64_t L, int32_t d, int32_t heads, ga_dtype dtype, void *stream);

/* ga_attention with sharding offsets, workspace, probes and kernel choice (opts may be NULL). */
ga_status ga_attention_ex(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out,
                          int64_t L, int32_t d, int32_t heads, ga_dtype dtype, const ga_opts *opts,
                          void *stream);

/* End-to-end variant on HOST buffers: copies Q,K,V (host, [L,heads,d]) to the device,
   runs the attention, copies out back to host `out`, all enqueued on `stream` using the
   stream-ordered allocator (libga's private pool, cudaMallocFromPoolAsync).  Host buffers should be pinned for
   asynchronous copies; `out` is valid after the caller synchronises `stream`.  CSR arrays
   in `mask` must already be DEVICE pointers.  For WINDOW and CSR masks with L >= 8192 the
   query range runs as 8 aligned chunks whose H2D, launch and D2H overlap on two internal
   copy streams forked from and joined back to `stream` (results identical to one call). */
ga_status ga_attention_host(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out,
                            int64_t L, int32_t d, int32_t heads, ga_dtype dtype, void *stream);

/* Backward pass (training): gradients of O = attention(Q, K,
   V, mask) for the upstream gradient dO, by the chain rule per edge (i, j) of the mask:
       P_ij = softmax_j(q_i.k_j / sqrt(d)),  dP_ij = dO_i.v_j,  D_i = dO_i.O_i,
       dS_ij = P_ij (dP_ij - D_i),  dQ_i = sum_j dS_ij k_j / sqrt(d),
       dK_j = sum_i dS_ij q_i / sqrt(d),  dV_j = sum_i P_ij dO_i.
   Q, K, V, O (the forward output), dO: DEVICE [L, heads, d] in `dtype`; dQ, dK, dV: DEVICE fp32
   [L, heads, d], overwritten (they must not overlap any input).  lse: optional DEVICE fp32
   [L, heads], the forward's log2-sum-exp2 of the row scores, lse_i = log2 sum_j 2^(s_ij log2 e)
   (= m + log2 l of a carried state, ga_state); NULL recomputes it (one extra pass over the
   edges).  Masks: CSR (a transposed CSR is built on the device; repeated columns keep their
   multiplicity), WINDOW, LONGNET, BLOCK_DILATED (symmetric: N^T(j) = N(j)).  BIGBIRD (implicit)
   returns GA_ERR_UNSUPPORTED: pass its ga_mask_to_csr.  Two launches (row pass: lse, D, dQ;
   column pass: dK, dV), no atomics: deterministic.  Scratch is stream-ordered (libga's pool). */
ga_status ga_attention_backward(const void *Q, const void *K, const void *V, const void *O, const void *dO,
                                const ga_mask *mask, const float *lse, float *dQ, float *dK, float *dV, int64_t L,
                                int32_t d, int32_t heads, ga_dtype dtype, void *stream);

/* out = o / l of a carried state (0 where l = 0), rounded to `dtype`: rows x heads x d.
   Composition: run the disjoint component masks of a pattern (e.g. WINDOW + BIGBIRD with
   parts = GA_BB_GLOBAL for Longformer) into one state with
   GA_STATE_ACCUMULATE, then finalise — equal to one call over the union. */
ga_status ga_state_finalize(const ga_state *state, int64_t rows, int32_t heads, int32_t d, ga_dtype dtype,
                            void *out, void *stream);

/* Workspace bytes ga_attention_ex uses for (mask, shape, opts): CSR heavy-row split, or the
   LongNet tcgen05 block partials ([slots][heads][d+4] fp32).  0 when none.  Host only. */
ga_status ga_workspace_size(const ga_mask *mask, int64_t L, int32_t d, int32_t heads, ga_dtype dtype,
                            const ga_opts *opts, size_t *bytes);

/* Query-range alignment in tokens (host): launches whose [q_begin, q_begin + q_rows)
   boundaries are multiples of *tokens compute every row exactly as one launch over the whole
   range does (same tiles, same reduction order), so sharded outputs are bit-identical to the
   single-GPU output.  Band kernel (WINDOW, bf16/fp16): 112 * r; LongNet tensor-core
   kernels: w0 (one level-0 segment); edge kernel: 1. */
ga_status ga_query_alignment(const ga_mask *mask, int32_t d, ga_dtype dtype, int64_t *tokens);

/* Exact number of edges of an implicit pattern (host; closed forms per family, SURVEY
   §8(c)).  For GA_MASK_CSR returns mask->nnz.  For BIGBIRD with a device global_idx the
   list is copied to the host (synchronous). */
ga_status ga_mask_count(const ga_mask *pattern, int64_t *nnz_out);

/* Materialise an implicit pattern as binary CSR on the device:
   degrees -> exclusive scan -> fill, columns ascending.  row_ptr: DEVICE int64 [L+1];
   col_idx: DEVICE int32 [nnz] with nnz from ga_mask_count.  The result equals the CPU
   enumeration bit for bit.  Temporary scan storage is stream-ordered (libga's private pool). */
ga_status ga_mask_to_csr(const ga_mask *pattern, int64_t *row_ptr, int32_t *col_idx, void *stream);

/* COO input ("COO" mask storage): convert an edge list
   (rows[e], cols[e]), e < n, in any order, to binary CSR on the device.  Duplicates are
   counted once (a 0-1 mask, reading R7).  Method: keys row*L + col -> radix sort (CUB) ->
   unique -> col_idx = key mod L, row_ptr[r] = lower_bound(keys, r*L).  The paper's COO
   kernel searches the list per row; here COO is converted once, never searched.
   rows, cols: DEVICE int32 [n]; row_ptr: DEVICE int64 [L+1] (written); col_idx: DEVICE
   int32, capacity n (the first *nnz_out entries written, ascending per row); nnz_out: HOST,
   the number of distinct edges (the call synchronises `stream` to read it).  Scratch is
   stream-ordered (libga's private pool).  Errors: GA_ERR_INVALID_ARG (L <= 0 or L > 2^31-1,
   n < 0, NULL buffers), GA_ERR_MASK (an index outside [0, L); outputs then undefined),
   GA_ERR_CUDA. */
ga_status ga_coo_to_csr(int64_t L, const int32_t *rows, const int32_t *cols, int64_t n, int64_t *row_ptr,
                        int32_t *col_idx, int64_t *nnz_out, void *stream);

/* O(L + nnz) validity check of an explicit CSR (S:97-98 invariants).  Synchronises the
   stream.  *ok = 1 when valid; returns GA_ERR_MASK (and *ok = 0) otherwise. */
ga_status ga_mask_validate(const ga_mask *csr, void *stream, int *ok);

/* Synthetic inputs (reading R22): dst[t] = round_dtype(x(e0 + t)) for
   t in [0, n), x(e) = (splitmix64(splitmix64(seed + tensor) ^ e) >> 40) * 2^-24,
   plus `shift` (added in fp32 before rounding; 0 for the paper's U[0,1)).  DEVICE dst. */
ga_status ga_fill_inputs(void *dst, ga_dtype dtype, int64_t n, uint64_t seed, int32_t tensor, int64_t e0,
                         float shift, void *stream);

/* ------------------------------------------------------------------------------------
 * Multi-GPU (SURVEY §8(b) comm entry points, §8(e) partitioning).  One process per GPU;
 * the sequence is cut into equal contiguous query shards, rank q owning token rows
 * [q*S, min(L, (q+1)*S)), S = ceil(L / world) (rows are independent).
 * K and V shards live in SYMMETRIC buffers (ga_comm_alloc) that every rank maps with CUDA
 * IPC, so the attention kernels read the rows they need from other ranks directly over
 * NVLink while they compute — the window halo (PAPER.md:124-136 masks reach w-1 rows past a
 * shard edge) and LongNet's strided long-range rows — with no separate exchange launch.
 * Explicit CSR masks (unstructured columns) all-gather K/V with copy engines first.
 * One node: the bootstrap rendezvous is a TCP socket on 127.0.0.1.
 * ------------------------------------------------------------------------------------ */
typedef struct ga_comm ga_comm; /* opaque */
#define GA_COMM_ID_BYTES 128

/* Rank 0 only: create the 128-byte bootstrap id (opens a listening socket on 127.0.0.1 in
   this process) and hand it to the other ranks (e.g. torch.distributed broadcast). */
ga_status ga_comm_get_unique_id(void *id128);

/* Collective over `world` processes: connect to rank 0 through the id, then (device >= 0)
   allocate the device barrier flags on CUDA device `device`.  device = -1 creates a
   host-only comm (bootstrap and ga_comm_host_allgather only).  Blocks until every rank has
   joined (timeout 120 s -> GA_ERR_COMM).  Every pair of distinct devices must have peer
   access (cudaDeviceCanAccessPeer; the kernels load peer rows over NVLink): otherwise every
   rank returns GA_ERR_COMM.  *comm is owned by the caller until ga_comm_destroy. */
ga_status ga_comm_create(int32_t world, int32_t rank, const void *id128, int32_t device, ga_comm **comm);

/* Collective: allocate `bytes` (same on every rank) of DEVICE memory whose copies on all
   ranks are mapped into each other's address space.  *local is this rank's copy (owned by
   the comm; released by ga_comm_free / ga_comm_destroy).  Put the K and V shards
   ([S, heads, d]) of ga_attention_sharded here. */
ga_status ga_comm_alloc(ga_comm *comm, size_t bytes, void **local);

/* Collective: release a ga_comm_alloc buffer (synchronises the device). */
ga_status ga_comm_free(ga_comm *comm, void *local);

/* Device-side barrier enqueued on `stream`: returns once every rank's stream has reached
   its matching barrier (all ranks call barriers in the same order).  A rank that does not
   arrive within 60 s releases the others and sets the flag read by ga_comm_status. */
ga_status ga_comm_barrier(ga_comm *comm, void *stream);

/* Host all-gather of `bytes` per rank into all[world * bytes] over the bootstrap sockets
   (small control data; also the CPU test hook of the bootstrap). */
ga_status ga_comm_host_allgather(ga_comm *comm, const void *mine, size_t bytes, void *all);

/* *timed_out = 1 if a device barrier of this comm gave up waiting for a peer.  The flag lives
   in device-mapped pinned host memory: no synchronisation, but it reflects only barriers that
   have already executed (synchronise the stream first for a definite answer). */
ga_status ga_comm_status(ga_comm *comm, int *timed_out);

/* Sharded attention: this rank's query rows [row_begin, row_end) of a length-L sequence.
   Q, out: DEVICE [row_end - row_begin, heads, d] (local rows).  K, V: this rank's shard of
   the keys/values, [row_end - row_begin, heads, d], inside ga_comm_alloc buffers at the
   same offset on every rank.  row_begin/row_end must be this rank's shard as defined above.
   WINDOW / LONGNET / BLOCK_DILATED read remote rows in-kernel over peer memory; CSR (row_ptr
   and col_idx are the full GLOBAL arrays, on every rank) all-gathers K and V into a
   comm-owned [L, heads, d] buffer first.  Enqueued on `stream` between two device barriers:
   the entry barrier makes every rank's K/V visible, the exit barrier keeps them unchanged
   until every rank has finished reading.  opts: kernel choice, CSR workspace, probes (its
   q_/kv_ ranges are ignored).  Shards that are multiples of ga_query_alignment produce
   rows bit-identical to ga_attention on one GPU.  Failure of a peer: if either barrier
   times out, this rank's `out` is overwritten with NaN (0xff bytes) on the stream, and every
   later call on the comm returns GA_ERR_COMM without enqueuing anything. */
ga_status ga_attention_sharded(const void *Q, const void *K, const void *V, const ga_mask *mask, void *out,
                               int64_t L, int64_t row_begin, int64_t row_end, int32_t d, int32_t heads,
                               ga_dtype dtype, const ga_opts *opts, ga_comm *comm, void *stream);

/* Collective: free every symmetric buffer and close the bootstrap sockets. */
ga_status ga_comm_destroy(ga_comm *comm);

/* Thread-local description of the last non-OK status ("" if none). */
const char *ga_last_error(void);

/* Telemetry: number of CUDA kernels this library has launched since it was loaded
   (host counter; bench.py reports it as gpu_launches). */
unsigned long long ga_launch_count(void);

/* Library version string. */
const char *ga_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GA_H */

/*
 * dr.h — C ABI of the B200-native DR-CircuitGNN hot path (arXiv 2508.16769).
 *
 * Library: paper_2508_16769_b200/libdr.so (sm_100a). Plain C types only.
 * Citations: P:<n> = /root/reference/PAPER.md line n (section / equation /
 * algorithm named beside it); Q<n> = a reading listed in DESIGN.md.
 *
 * Conventions (all entry points)
 *   - Tensors are DEVICE pointers owned by the caller, fp32, row-major,
 *     contiguous, unless documented otherwise. The library never frees caller
 *     memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream). Compute calls are asynchronous and stream-ordered; internal
 *     streams fork from and join back to `stream` with events.
 *   - Validation of sizes, pointers and k is synchronous and precedes any
 *     launch; on failure nothing is launched and a non-zero dr_status is
 *     returned, with detail in dr_last_error(). Asynchronous kernel faults
 *     surface as DR_ERR_CUDA at a later call or at the caller's synchronise.
 *   - On failure outputs are unspecified; no handle is created; nothing leaks.
 *   - GPU restrictions of this build: 1 <= k <= 128 and k a power of two
 *     (§4.3: "the number of non-zero elements remaining ... is a power
 *     of two to maximize GPU parallel resource utilization"); k <= dim <= 256
 *     (CBSR indices are one byte); dim % 4 == 0; every relation nnz < 2^31.
 */
#ifndef DR_H_
#define DR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
typedef enum {
    DR_OK = 0,
    DR_ERR_INVALID_ARGUMENT = 1,   /* null pointer, negative size, bad enum       */
    DR_ERR_BAD_K = 2,              /* k outside the restrictions above            */
    DR_ERR_SHAPE_MISMATCH = 3,     /* tensor / graph / layer dims disagree        */
    DR_ERR_OUT_OF_RANGE = 4,       /* CSR column or row pointer out of range      */
    DR_ERR_DUPLICATE_EDGE = 5,     /* CSR row not strictly increasing             */
    DR_ERR_TRANSPOSE_MISMATCH = 6, /* pinned != pins^T, or CSC != CSR^T           */
    DR_ERR_NONFINITE = 7,          /* non-finite edge weight                      */
    DR_ERR_TAPE_MISMATCH = 8,      /* tape/workspace too small or from other call */
    DR_ERR_OUT_OF_MEMORY = 9,
    DR_ERR_CUDA = 10,
    DR_ERR_NCCL = 11,
    DR_ERR_UNSUPPORTED = 12
} dr_status;

const char *dr_status_str(dr_status s);
/* Thread-local detail of this thread's last failure ("" if none). */
const char *dr_last_error(void);
/* Library build string (arch, version). */
const char *dr_version(void);

/* ------------------------------------------------------------------ graph
 * A circuit heterograph (§2.2): node types cell (n_cell) and net
 * (n_net); relations near (cell<-cell, geometric), pins (net<-cell) and
 * pinned (cell<-net), pins and pinned mutually transposed. Each
 * relation is an n_dst x n_src adjacency A^psi, rows = destinations (Eq. 4,
 * P:236-238), given as HOST CSR read only during dr_graph_create.
 */
typedef struct dr_graph dr_graph;        /* opaque, immutable, safe for concurrent readers */
typedef enum { DR_NEAR = 0, DR_PINS = 1, DR_PINNED = 2 } dr_rel;
/* Module of a relation: its degree normaliser and root-weight semantics
 * ("two SageConv modules and one GraphConv module"; reading Q1/Q12):
 *   DR_SAGE_MEAN     : c_i = 1/max(deg_in(i),1),        s_j = 1
 *   DR_GRAPHCONV_SYM : c_i = max(deg_in(i),1)^-1/2,     s_j = max(deg_out(j),1)^-1/2
 * Degrees are unweighted edge counts. */
typedef enum { DR_SAGE_MEAN = 0, DR_GRAPHCONV_SYM = 1 } dr_module;
typedef enum { DR_MERGE_MAX = 0, DR_MERGE_SUM = 1 } dr_merge;   /* Eq. 8 / Eq. 6 variant */

typedef struct {
    int32_t n_dst, n_src;
    int64_t nnz;
    const int64_t *row_ptr;   /* HOST [n_dst+1], row_ptr[0]=0, row_ptr[n_dst]=nnz        */
    const int32_t *col_idx;   /* HOST [nnz], strictly increasing within a row, < n_src   */
    const float *val;         /* HOST [nnz] edge weights a_ij > 0; NULL => all 1 */
    dr_module module;
    /* Optional HOST inputs, each NULL => built / counted by the library:
     *  col_ptr [n_src+1], row_idx [nnz]: the CSC = CSR(A^T) of Alg. 2 stage 1
     *      ("Transpose A to CSC"), rows ascending within a column. Checked
     *      to equal the transpose of the CSR (DR_ERR_TRANSPOSE_MISMATCH) unless
     *      DR_GRAPH_SKIP_VALIDATION, in which case it is used as given.
     *  tval [nnz]: a_ij in CSC order (only with col_ptr; NULL => val transposed);
     *      checked against val like col_ptr / row_idx.
     *  deg_dst [n_dst], deg_src [n_src]: the degrees the normalisers use (e.g.
     *      those of a larger graph this one is a part of); >= 0, clamped to >= 1
     *      (Q12). The degree classes of the schedules always use the CSR's own
     *      counts.
     *  norm_dst [n_dst], norm_src [n_src]: c_i and s_j themselves (finite),
     *      overriding module + degrees for the SpMM and SSpMM of this relation. */
    const int64_t *col_ptr;
    const int32_t *row_idx;
    const float *tval;
    const int32_t *deg_dst, *deg_src;
    const float *norm_dst, *norm_src;
} dr_rel_desc;

typedef struct {
    void *(*alloc)(void *ctx, size_t bytes, void *stream);
    void (*free)(void *ctx, void *p, void *stream);
    void *ctx;
} dr_allocator;                              /* NULL => cudaMallocAsync / cudaFreeAsync */

#define DR_GRAPH_SKIP_VALIDATION 1u          /* trust the CSR invariants                 */
#define DR_GRAPH_ORDER_IDENTITY 2u           /* process rows in id order (no degree classes) */

/* Build the device-resident graph: validates each CSR (sorted, unique, in
 * range), checks rel[DR_PINNED] == rel[DR_PINS]^T, counts degrees and
 * normalisers, builds CSC = CSR(A^T) for the backward (Alg. 2 stage 1)
 * and the degree-binned processing orders (Alg. 1 stage 2). Host
 * work runs on n_threads worker threads, one relation each (§3.4, P:425;
 * 0 => 3); uploads are stream-ordered on `stream`, which this call
 * synchronises before returning. */
dr_status dr_graph_create(int32_t n_cell, int32_t n_net, const dr_rel_desc rel[3],
                          const dr_allocator *a, int32_t n_threads, uint32_t flags,
                          void *stream, dr_graph **out);
dr_status dr_graph_destroy(dr_graph *g);

typedef struct {
    int32_t n_cell, n_net;
    int64_t nnz[3];
    int32_t max_deg_dst[3], max_deg_src[3];
    int32_t hub_rows_dst[3], hub_rows_src[2];    /* rows routed to the CTA-per-row kernels */
    size_t device_bytes;
    /* tensor-core tiled SpMM (near only, unit weights, mean degree >= 8): tiles of
     * <= 128 rows and 64-id halo chunks of the CSR / CSC form; 0 => SIMT kernels */
    int32_t tiles[3], tiles_T[3];
    int64_t chunks[3], chunks_T[3];
} dr_graph_info_t;
dr_status dr_graph_info(const dr_graph *g, dr_graph_info_t *info);

/* ------------------------------------------------------------------ CBSR
 * Compressed Balanced Sparse Row: exactly k (value, index) pairs per
 * row, indices strictly ascending, values copied verbatim from the dense row.
 * val: DEVICE float [n*k]; idx: DEVICE uint8 [n*k] (idx_bytes must be 1). */
typedef struct {
    int64_t n;
    int32_t dim, k, idx_bytes;
    void *idx;
    float *val;
} dr_cbsr;

/* D-ReLU, Eq. 2-3: th_i = min(topk(X_i,:, k)); keep X_id >= th_i,
 * exactly k per row with ties at th_i broken towards the lowest column (Q5),
 * -0.0 == +0.0, values verbatim including negatives (Q6). x: DEVICE [n x dim]
 * with leading dimension ldx >= dim; out->n, dim, k set by the caller. */
dr_status dr_drelu_topk(const float *x, int64_t n, int32_t dim, int64_t ldx, dr_cbsr *out,
                        void *stream);

/* DR-SpMM forward of one relation, Eq. 5-7, Alg. 1,
 * W applied outside (Q9):  z[i,:] = c_i * sum_{j in N(i)} a_ij * s_j * densify(h_src[j]).
 * h_src->n must equal the relation's n_src; z: DEVICE [n_dst x h_src->dim]. */
dr_status dr_spmm_fwd(const dr_graph *g, dr_rel r, const dr_cbsr *h_src, float *z, void *stream);

/* DR-SpMM backward (SSpMM) of one relation, Eq. 10-11, Alg. 2
 * (P:316-345): the transposed product evaluated only at the forward-kept CBSR
 * indices of h_src (Alg. 2 stage 1 "Reuse preserved ... CBSR indices"):
 *   g[j,t] = sum_{i: j in N(i)} c_i * a_ij * s_j * dz[i, h_src.idx[j,t]].
 * dz = dL/dZ: DEVICE [n_dst x dim]. Outputs (either may be NULL, not both):
 *   g_kept: DEVICE [n_src x k];
 *   dx:     DEVICE [n_src x dim] dense D-ReLU mask gradient: g scattered to
 *           the kept indices, exact zeros elsewhere.
 * accumulate != 0 adds into g_kept / into dx's kept positions (dx's other
 * entries are then left untouched). Per-source-row ownership, no atomics (Q23). */
dr_status dr_spmm_bwd(const dr_graph *g, dr_rel r, const float *dz, const dr_cbsr *h_src,
                      float *g_kept, float *dx, int32_t accumulate, void *stream);

/* ------------------------------------------------------------------ HeteroConv layer
 * One HeteroConv block (Fig. 1; Eq. 4-9; reading Q1-Q3):
 *   H_c = drelu(X_c, k_cell), H_n = drelu(X_n, k_net)
 *   Z_psi = DR-SpMM_psi(H_src)                            (3 relations, 3 streams, §3.4)
 *   Y_near   = Z_near Wn_near + densify(H_c) Wr_near + b_near      (SageConv mean)
 *   Y_pinned = Z_pinned Wn_pinned + b_pinned                       (GraphConv)
 *   Y_net    = Z_pins Wn_pins + densify(H_n) Wr_pins + b_pins      (SageConv mean)
 *   Y_cell = max(Y_near, Y_pinned), M = [Y_near >= Y_pinned]      (Eq. 8, Eq. 14)
 * Weights are DEVICE fp32: wn[r] is d_in(src type of r) x d_out; wr[r] is
 * d_in(dst type of r) x d_out or NULL (no root term). wr[DR_PINNED] must be
 * NULL (GraphConv has no root weight; DR_ERR_UNSUPPORTED otherwise).
 * k_pins: per-edge-type k ("k_pinned, k_near, and k_pins"; reading Q27):
 * 0 = k_cell (per node type). Otherwise pins reads its own cell CBSR
 *   H_p = drelu(X_c, k_pins),  Z_pins = DR-SpMM_pins(H_p),
 * near and the near root keep H_c (k_near = k_cell), pinned and the pins root
 * keep H_n (k_pinned = k_net); the backward adds pins' D-ReLU mask gradient at
 * H_p's indices: dX_c = scatter(g_near + root, idx_c) + scatter(g_pins, idx_p).
 * Same restrictions as k_cell. */
typedef struct {
    int32_t d_cell, d_net, d_out, k_cell, k_net;
    dr_merge merge;
    const float *wn[3];
    const float *wr[3];
    const float *b[3];
    int32_t k_pins;
} dr_layer;
typedef struct {
    float *wn[3];
    float *wr[3];
    float *b[3];
} dr_layer_grad;                               /* same shapes; NULL where dr_layer's is NULL */

#define DR_FWD_SEQUENTIAL 1u  /* run the three relations on one stream (§4.4 breakdown)    */
#define DR_FWD_TAPS 2u        /* also keep Y_near / Y_pinned for teacher-forced parity      */
#define DR_FWD_INPUT_IN_TAPE 4u /* dr_heteroconv_fwd_chain: H_c / H_n are already in the tape */
#define DR_FWD_Y_SCRATCH 8u   /* dr_heteroconv_fwd_chain: y_cell / y_net may be left unwritten */
#define DR_FWD_NO_NET_OUT 16u /* Y_net not needed (last layer): no pins SpMM / net projection;
                                 y_net unwritten; the backward takes dy_net = NULL (zero) */

/* Bytes of the caller-allocated tape (forward activations reused by the
 * backward: CBSR of both types, Z_psi, merge-mask bits, taps) plus backward
 * scratch. */
dr_status dr_heteroconv_tape_bytes(const dr_graph *g, const dr_layer *L, uint32_t flags,
                                   size_t *bytes);
dr_status dr_heteroconv_fwd(const dr_graph *g, const dr_layer *L, const float *x_cell,
                            const float *x_net, float *y_cell, float *y_net, void *tape,
                            uint32_t flags, void *stream);
/* Layer forward with the NEXT layer's D-ReLU fused into this layer's projection
 * epilogue (row a5; Eq. 2-3, applied to this layer's output, which
 * is the next layer's input: "D-ReLU ... after the activation layer").
 * Same as dr_heteroconv_fwd, plus:
 *   next_L / next_tape (both or neither): the projection epilogues write
 *     drelu(Y_cell, next_L->k_cell) and drelu(Y_net, next_L->k_net) -- exactly
 *     k per row, ties to the lowest column, values verbatim, ascending indices;
 *     bit-identical to dr_drelu_topk on the written Y -- straight into
 *     next_tape's H_c / H_n (next_tape laid out for next_L with next_flags), so
 *     the next layer runs with DR_FWD_INPUT_IN_TAPE and Y is never re-read.
 *     next_L->d_cell == next_L->d_net == L->d_out (DR_ERR_SHAPE_MISMATCH);
 *     next_L->k_pins must be 0 or k_cell (DR_ERR_UNSUPPORTED).
 *   flags & DR_FWD_INPUT_IN_TAPE: this layer's H_c / H_n were written into
 *     `tape` by the previous layer's chained call; x_cell / x_net are ignored
 *     (may be NULL); L->k_pins must be 0 or k_cell.
 *   flags & DR_FWD_Y_SCRATCH: the caller does not need Y: where the epilogue
 *     is fused (k in {4, 8, 16, 32}, k <= d_out) y_cell / y_net are left
 *     unwritten; otherwise they are written and D-ReLU'd by a separate launch.
 *     y_cell / y_net must still be valid (n x d_out) buffers. */
dr_status dr_heteroconv_fwd_chain(const dr_graph *g, const dr_layer *L, const float *x_cell,
                                  const float *x_net, float *y_cell, float *y_net, void *tape,
                                  uint32_t flags, const dr_layer *next_L, void *next_tape,
                                  uint32_t next_flags, void *stream);
/* Backward (Eq. 10-14, Alg. 2): mask routing, dW = Z^T dY, dWr = H^T dY, db,
 * dZ = dY Wn^T, SSpMM per source type (cell: near + pins + root term; net:
 * pinned + root term) and the D-ReLU mask scatter. dx_cell == NULL and
 * dx_net == NULL skip the SSpMM (first layer). grads are overwritten.
 * dy_net == NULL means dY_net = 0 (after a DR_FWD_NO_NET_OUT forward): the
 * pins relation's terms are skipped and its gradients written as zeros. */
dr_status dr_heteroconv_bwd(const dr_graph *g, const dr_layer *L, void *tape,
                            const float *dy_cell, const float *dy_net, float *dx_cell,
                            float *dx_net, dr_layer_grad *grads, uint32_t flags, void *stream);
/* Device views into a tape after dr_heteroconv_fwd (for teacher-forced parity
 * tests): the CBSR of both node types, Z per relation, Y_near/Y_pinned taps
 * (NULL unless DR_FWD_TAPS) and the merge mask (uint32 words, row-major
 * n_cell x ceil(d_out/32), bit d%32 of word d/32 = M[i,d]). z_split[r] = 1:
 * Z of relation r is stored as rows of [hi | lo] bf16 halves (d_src values
 * each, 4 d_src bytes per row), Z = hi + lo -- the tensor-core operand format
 * the fused path uses when the widths allow (source width % 64 == 0). */
typedef struct {
    dr_cbsr h_cell, h_net;
    float *z[3];
    float *y_near, *y_pinned;
    uint32_t *mask;
    int32_t z_split[3];
    dr_cbsr h_pins;                 /* pins' source CBSR (== h_cell unless k_pins set) */
} dr_tape_view;
dr_status dr_heteroconv_tape_view(const dr_graph *g, const dr_layer *L, void *tape,
                                  uint32_t flags, dr_tape_view *view);

/* ------------------------------------------------------------------ NEXT-2: per-neighbour-group K
 * Alg. 1 stage 2 and P:346-350: "D-ReLU will apply respective
 * K-values to the NGs with respect to their sizes ... The more neighbors the NGs
 * have, the fewer features per neighbor are required to pass". Reading Q26
 * (DESIGN.md): a destination row with in-degree d keeps, from every neighbour,
 * the first K(d) entries of the neighbour's value-sorted CBSR row (its exact
 * top-K(d)), K(d) = kb[0] for d <= thr[0], kb[1] for d <= thr[1], kb[2] above;
 * k >= kb[0] >= kb[1] >= kb[2] >= 1. Runs on the SIMT kernels (all relations). */
typedef struct {
    int32_t thr[2];
    int32_t kb[3];
} dr_ng_sched;
/* D-ReLU with each row's k pairs in value-descending order (ties: lower column
 * first), so every prefix is an exact top-k'. k <= 32. Same arguments/errors as
 * dr_drelu_topk. */
dr_status dr_drelu_topk_sorted(const float *x, int64_t n, int32_t dim, int64_t ldx, dr_cbsr *out,
                               void *stream);
/* A schedule bound to one relation of one graph: validates `sched` (BadK unless
 * 32 >= kb[0] >= kb[1] >= kb[2] >= 1, InvalidArgument unless thr[0] <= thr[1])
 * and precomputes, on `stream`, K(deg of the destination) for every edge in the
 * relation's CSC order (nnz bytes of device memory from the graph's allocator),
 * so the backward reads it coalesced. The plan is immutable once created: any
 * number of streams may use it after `stream` has reached the creation point.
 * Destroy it before its graph. */
typedef struct dr_ng_plan dr_ng_plan;
dr_status dr_ng_plan_create(const dr_graph *g, dr_rel r, const dr_ng_sched *sched, void *stream,
                            dr_ng_plan **out);
dr_status dr_ng_plan_destroy(dr_ng_plan *p);
/* z[i,:] = c_i * sum_{j in N(i)} a_ij * s_j * densify(first K(deg_i) pairs of h_src[j]),
 * h_src value-sorted (dr_drelu_topk_sorted), for the plan's graph and relation.
 * Errors as dr_spmm_fwd, plus BadK when h_src->k < kb[0]. */
dr_status dr_spmm_fwd_ng(const dr_ng_plan *p, const dr_cbsr *h_src, float *z, void *stream);
/* Adjoint of dr_spmm_fwd_ng: g[j,t] = sum over i with j in N(i) and t < K(deg_i) of
 * c_i a_ij s_j dz[i, idx[j,t]]; outputs as dr_spmm_bwd (no accumulate). */
dr_status dr_spmm_bwd_ng(const dr_ng_plan *p, const float *dz, const dr_cbsr *h_src,
                         float *g_kept, float *dx, void *stream);

/* ------------------------------------------------------------------ training
 * The 2-layer model of P:464-466: HeteroConv x n_layers -> linear head on
 * cells -> MSE (Q14) -> backward -> [NCCL allreduce of the flat gradient] ->
 * Adam with coupled L2 weight decay (Q15). Flat parameter layout, per layer
 * l (d_c = d_in_cell, d_n = d_in_net for l = 0, else d_hidden; D = d_hidden):
 *   wn_near[d_c*D] wr_near[d_c*D] b_near[D] wn_pinned[d_n*D] b_pinned[D]
 *   wn_pins[d_c*D] wr_pins[d_n*D] b_pins[D]
 * then the head w_h[D] b_h[1]. */
typedef struct {
    int32_t n_layers, d_in_cell, d_in_net, d_hidden, k_cell, k_net;
    float lr, weight_decay, beta1, beta2, eps;
    int32_t k_pins;                 /* per-edge-type k of every layer (dr_layer.k_pins), 0 = k_cell */
} dr_train_cfg;
typedef struct dr_trainer dr_trainer;         /* opaque, single-threaded use */

int64_t dr_train_param_count(const dr_train_cfg *c);
/* params: DEVICE flat buffer (caller-owned, updated in place). nccl_comm: an
 * ncclComm_t from dr_nccl_comm_init, or NULL for one GPU. */
dr_status dr_trainer_create(const dr_train_cfg *c, float *params, int64_t n_params,
                            void *nccl_comm, const dr_allocator *a, dr_trainer **out);
/* One training step on `batch` (one design, or a disjoint union of designs,
 * Q24). x_cell/x_net/labels: DEVICE. If loss_host != NULL (pinned host float)
 * the step's mean loss is written there when the stream reaches it. If
 * grad_out != NULL (DEVICE [n_params]) the allreduced mean gradient is also
 * copied there (parity tests). */
dr_status dr_train_step(dr_trainer *t, const dr_graph *batch, const float *x_cell,
                        const float *x_net, const float *labels, float *loss_host,
                        float *grad_out, void *stream);
dr_status dr_trainer_destroy(dr_trainer *t);

/* NCCL bootstrap for data parallelism (north_star: one gradient allreduce per
 * step). The unique id (128 bytes) is made on rank 0 and broadcast by the
 * caller (e.g. through torch.distributed). NCCL is loaded at run time. */
dr_status dr_nccl_unique_id(void *id128);
dr_status dr_nccl_comm_init(const void *id128, int32_t nranks, int32_t rank, void **comm);
dr_status dr_nccl_comm_destroy(void *comm);

/* ------------------------------------------------------------------ single-graph multi-GPU
 * SURVEY §8 f4 (beyond the paper): one relation's DR-SpMM (Eq. 5-7) and SSpMM
 * (Eq. 10-11) split across `world` ranks by contiguous destination-row ranges
 * (1-D partition). Rank q owns destinations [dst_part[q], dst_part[q+1]) and
 * sources [src_part[q], src_part[q+1]). What crosses ranks is the compact
 * CBSR, not dense features: the forward allgathers every rank's CBSR rows
 * (k * 5 bytes per source row instead of dim * 4), the backward reduce-scatters
 * the per-source partial g (k * 4 bytes per row) to the source's owner.
 * Source rows live in a padded global space of world * max_src rows: global
 * source j owned by q sits at row q * max_src + (j - src_part[q]); each rank's
 * block is max_src rows, rows past its count are padding (no edge reads them).
 * Normalisers are the global ones (Q12), so the union of the ranks' z_local is
 * dr_spmm_fwd's Z and the sum of their g_part is dr_spmm_bwd's g. */
typedef struct dr_shard dr_shard;
typedef struct {
    int32_t world, rank, max_src;
    int64_t dst_begin, dst_end, src_begin, src_end, nnz_local;
    size_t device_bytes;
    int32_t tiles, tiles_T;         /* tensor-core tiled SpMM tiles of the block (0 => SIMT) */
} dr_shard_info_t;
/* Default partition (host only, no GPU): dst_part [world+1] balances edges
 * (boundaries at the first row whose row_ptr reaches q * nnz / world);
 * src_part [world+1] = dst_part for a square relation (n_dst == n_src), else
 * balances rows. */
dr_status dr_shard_plan(const dr_rel_desc *rel, int32_t world, int64_t *dst_part,
                        int64_t *src_part);
/* rel: the GLOBAL relation (HOST CSR, validated as in dr_graph_create).
 * dst_part / src_part: [world+1] non-decreasing from 0 to n_dst / n_src, or
 * NULL for dr_shard_plan's. Uploads this rank's row block on `stream`
 * (synchronised before returning). */
dr_status dr_shard_create(const dr_rel_desc *rel, int32_t world, int32_t rank,
                          const int64_t *dst_part, const int64_t *src_part, const dr_allocator *a,
                          void *stream, dr_shard **out);
dr_status dr_shard_destroy(dr_shard *s);
dr_status dr_shard_info(const dr_shard *s, dr_shard_info_t *info);
/* h_local: n = max_src (this rank's sources, padded); h_all: n = world * max_src,
 * same dim and k. NCCL allgather of val and idx on nccl_comm (a communicator of
 * `world` ranks in rank order, from dr_nccl_comm_init); NULL only when world == 1. */
dr_status dr_shard_allgather_cbsr(const dr_shard *s, const dr_cbsr *h_local, dr_cbsr *h_all,
                                  void *nccl_comm, void *stream);
/* z_local: DEVICE [dst_end - dst_begin x dim] = rows dst_begin.. of Z. */
dr_status dr_shard_spmm_fwd(const dr_shard *s, const dr_cbsr *h_all, float *z_local, void *stream);
/* dz_local: DEVICE [dst_end - dst_begin x dim] rows of dL/dZ; g_part: DEVICE
 * [world * max_src x k] this rank's contribution to every source's g. */
dr_status dr_shard_spmm_bwd(const dr_shard *s, const float *dz_local, const dr_cbsr *h_all,
                            float *g_part, void *stream);
/* g_local [max_src x k] = sum over ranks of their g_part rows for this rank's
 * sources (NCCL reduce-scatter; NULL comm only when world == 1). If dx_local
 * (DEVICE [max_src x dim]) is given, also writes the dense D-ReLU mask gradient:
 * g_local scattered to h_local's indices, zeros elsewhere. */
dr_status dr_shard_reduce_scatter_g(const dr_shard *s, const float *g_part,
                                    const dr_cbsr *h_local, float *g_local, float *dx_local,
                                    void *nccl_comm, void *stream);
/* ---- the exchange fused into the SpMM over peer memory (f4, beyond the paper).
 * Instead of an allgather of the CBSR and a reduce-scatter of g, the SIMT SpMM
 * kernels read every remote source row IN PLACE from its owner's buffer and the
 * backward writes every per-source contribution IN PLACE into the owner's inbox
 * -- over NVLink when the owner is another GPU (P2P loads / stores inside the
 * compute kernel, so the transfer overlaps the math row by row), plain loads
 * when ranks share a device. val[q] / idx[q]: rank q's LOCAL CBSR (max_src rows,
 * k pairs, idx uint8) as device pointers usable on this device (cudaIpc- or
 * symmetric-memory-mapped peers; `peer_buffers` in the Python binding). The
 * caller orders the ranks: every owner's CBSR written before any rank's
 * _fwd_peer / _bwd_peer reads it, every rank's _bwd_peer done before the owner's
 * _inbox_reduce (e.g. a barrier). world <= 8. */
typedef struct {
    int32_t world;
    const float *val[8];
    const void *idx[8];
} dr_peer_cbsr;
/* z_local as dr_shard_spmm_fwd (bit-identical to it on the allgathered CBSR). */
dr_status dr_shard_spmm_fwd_peer(const dr_shard *s, const dr_peer_cbsr *h, int32_t dim, int32_t k,
                                 float *z_local, void *stream);
/* inbox[q]: owner q's inbox, DEVICE [world x max_src x k] usable on this device;
 * this rank writes its contributions to owner q's sources into slot `rank`
 * (every slot row of every owner, zeros for sources without local edges). */
dr_status dr_shard_spmm_bwd_peer(const dr_shard *s, const float *dz_local, const dr_peer_cbsr *h,
                                 int32_t dim, int32_t k, float *const *inbox, void *stream);
/* g_local [max_src x k] = sum over slots p = 0 .. world-1 of inbox_local[p] in
 * that fixed order (deterministic); dx_local as dr_shard_reduce_scatter_g. */
dr_status dr_shard_inbox_reduce(const dr_shard *s, const float *inbox_local, const dr_cbsr *h_local,
                                float *g_local, float *dx_local, void *stream);

/* ---- a HeteroConv layer sharded by destination rows (f4, beyond the paper).
 * One rank owns cell rows [c0, c1) and net rows [n0, n1): its three dr_shard
 * must share one cell and one net partition -- near: cells -> cells (dst_part ==
 * src_part), pins: cells -> nets, pinned: nets -> cells (DR_ERR_SHAPE_MISMATCH
 * otherwise). The layer is Eq. 2-14 on the rank's rows; every exchange goes
 * through peer memory (dr_peer_cbsr, as dr_shard_spmm_*_peer):
 *   1. every rank: its local CBSR of cells and nets = dr_drelu_topk of its X rows
 *      (max_src rows each, zero rows past its range) -- h_cell / h_net.val[rank];
 *   2. (after all ranks' step 1) dr_shard_layer_fwd: the three SpMMs read remote
 *      CBSR rows in place, then the projections / max-merge on the local rows;
 *      y_cell [c1 - c0 x d_out], y_net [n1 - n0 x d_out];
 *   3. dr_shard_layer_bwd: dZ' and the Sage root terms on the local rows, the
 *      SSpMMs write every per-source sum into its owner's inbox (cells: [2 x
 *      world x max_src_cell x k_cell] = near, pins slots; nets: [world x
 *      max_src_net x k_net]), and this rank's rows' contribution to every weight
 *      gradient (the caller allreduces `grads` over ranks: dW is a sum over rows);
 *   4. (after all ranks' step 3) dr_shard_layer_dx: the owner adds up its inbox
 *      slots in a fixed order (+ its root terms) and scatters the D-ReLU mask
 *      gradient: dx_cell [c1 - c0 x d_cell], dx_net [n1 - n0 x d_net].
 * dy_net may not be NULL; no k_pins; the layer set borrows the shards. */
typedef struct dr_shard_layer dr_shard_layer;
dr_status dr_shard_layer_create(const dr_shard *near, const dr_shard *pins, const dr_shard *pinned,
                                dr_shard_layer **out);
dr_status dr_shard_layer_destroy(dr_shard_layer *sl);
dr_status dr_shard_layer_tape_bytes(const dr_shard_layer *sl, const dr_layer *L, uint32_t flags,
                                    size_t *bytes);
dr_status dr_shard_layer_fwd(const dr_shard_layer *sl, const dr_layer *L, const dr_peer_cbsr *h_cell,
                             const dr_peer_cbsr *h_net, float *y_cell, float *y_net, void *tape,
                             uint32_t flags, void *stream);
dr_status dr_shard_layer_bwd(const dr_shard_layer *sl, const dr_layer *L, void *tape,
                             const float *dy_cell, const float *dy_net, const dr_peer_cbsr *h_cell,
                             const dr_peer_cbsr *h_net, float *const *inbox_cell,
                             float *const *inbox_net, dr_layer_grad *grads, uint32_t flags,
                             void *stream);
dr_status dr_shard_layer_dx(const dr_shard_layer *sl, const dr_layer *L, void *tape,
                            const dr_peer_cbsr *h_cell, const dr_peer_cbsr *h_net,
                            const float *inbox_cell, const float *inbox_net, float *dx_cell,
                            float *dx_net, void *stream);

/* Per-kernel device timing: between dr_profile_begin and dr_profile_end every
 * libdr launch issued by this host thread is bracketed by CUDA events on the
 * stream it is launched on. dr_profile_end synchronises, aggregates by kernel
 * tag ("<kernel>.<relation or role>") and disables profiling; *n_out is the
 * number of distinct tags (entries beyond cap are dropped). While profiling,
 * layers run on the caller's stream (isolated kernel times) and training
 * steps run eagerly. Not for use inside CUDA-graph capture. */
typedef struct {
    char name[48];
    int64_t launches;
    double total_ms, max_ms;
} dr_profile_entry;
dr_status dr_profile_begin(void);
dr_status dr_profile_end(dr_profile_entry *out, int32_t cap, int32_t *n_out);

/* Experiment / test switches (read once from DR_* environment variables when
 * the library loads; never on a launch path). name is one of: nvtx, no_graph,
 * dense_simt, tspmm, ts_zerofill, ts_debug, tc2_debug, bwd_p, drelu_bs, drelu_tpr, tiles,
 * order_degree, warp_row_deg, ts_tile_w, ts_tile_w_bwd, ts_order_rr,
 * shard_tiles, shard_tiles_t (see csrc/knobs.cpp). Each selects between
 * parity-tested kernel paths or adds diagnostics; none changes a result beyond
 * rounding. Not synchronised with concurrent launches. DR_ERR_INVALID_ARGUMENT
 * for an unknown name. */
dr_status dr_debug_set(const char *name, int64_t value);

/* Number of kernels this library launched on this host thread since the last
 * reset (evidence for bench.py's gpu_launches). */
/* Bandwidth probe for the second roofline: reads the DEVICE
 * buffer `buf` (16-B aligned, `bytes` long) `reps` times with 128-bit loads on
 * `stream`, one float per CTA written to `sink` (DEVICE, >= 592 floats) so no
 * load is dead. The caller times it (read bytes = bytes x reps); a buffer of
 * about 1/4 of L2 gives the L2 read bandwidth. DR_ERR_INVALID_ARGUMENT on bad
 * arguments. Not part of the method; a measurement utility. */
dr_status dr_probe_read(const void *buf, int64_t bytes, int32_t reps, float *sink, void *stream);
int64_t dr_launch_count(void);
void dr_launch_count_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* DR_H_ */

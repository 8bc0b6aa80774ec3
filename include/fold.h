/*
 * fold.h — C ABI of the B200-native dynamic-batching hot path (arXiv 1702.02181,
 * "Deep Learning with Dynamic Computation Graphs", TensorFlow Fold, §2).
 *
 * Three calls carry the method:
 *   fold_schedule  — PAPER.md L40-44 (§2 bullets): depth per node, batching of all
 *                    nodes with the same (depth, operation), concatenation order, and
 *                    the gather indices ("the indices to gather encode the topology",
 *                    L30). Executor form: one append-only pool, so no pass-through
 *                    rows are materialised.
 *   fold_forward   — PAPER.md L47 (§2 loop model): per depth, gather child states,
 *                    run the batched operation once (embedding lookup at depth 1,
 *                    TreeRNN/TreeLSTM cell above), append the outputs to the pool.
 *   fold_backward  — PAPER.md L49: the gradient of gather/concat/loop, written out as
 *                    a reverse-level sweep with deterministic pull-reductions plus one
 *                    weight-gradient GEMM over all cells.
 * plus fold_sgd_update (the training step's optimizer).
 *
 * Conventions (all calls):
 *  - Every pointer named d_* / documented "device" is CUDA device memory, owned by the
 *    caller (the library never allocates or frees on these paths). Host pointers are
 *    documented "host".
 *  - `stream` is a cudaStream_t (CUstream) passed as void*. All work is stream-ordered.
 *    fold_schedule performs exactly one blocking device->host copy (status, depth count,
 *    level offsets) because launch shapes depend on it; forward/backward/sgd never sync.
 *  - No exceptions cross the ABI; every call returns fold_status. Data-dependent errors
 *    of fold_schedule report the smallest offending node id through
 *    fold_last_error_detail (graph id for FOLD_E_ROOT_RANGE).
 *  - Thread safety: calls on different streams with disjoint buffers may run concurrently;
 *    fold_last_error_detail is thread-local.
 *  - Int arrays are int32, row-major. Floats are IEEE fp32 unless stated.
 *
 * Environment (read once per process; tuning and test hooks, defaults are the measured
 * best):
 *   FOLD_FWD_NARROW_MAX   forward levels of at most this many rows after the last wider
 *                         level run in the weight-stationary narrow kernel (default 32; 0 off)
 *   FOLD_BWD_NARROW_MAX   same for the backward's first levels (default 64, used when at least 4
 *                         levels qualify; 0 off)
 *   FOLD_SCHED_SMALLN     fold_schedule runs as one block up to this many nodes (4096)
 *   FOLD_SCHED_PER_BLOCK  nodes per block of the cooperative scheduler above it (2048)
 *   FOLD_AUX_ORDER        0: embedding / db reductions on an auxiliary stream beside the
 *                         weight-gradient GEMM (default), 1: launched after it, 2: serial
 *   FOLD_DBG_FWD          1/2: per-tile forward timelines (fold_debug_fwd_trace)
 *   FOLD_DBG_BWD          1: per-tile timelines of the wide backward (fold_debug_bwd_trace)
 *   FOLD_DBG_SCHED        1: scheduler phase timeline (fold_debug_sched_trace)
 *   FOLD_DEBUG_SYNC       1: synchronize and check after every launch
 *   FOLD_FP32_SIMT        1: FP32 mode on the SIMT FFMA kernels (A/B measurement only)
 */
#ifndef FOLD_H
#define FOLD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FOLD_ABI_VERSION 6

typedef enum {
  FOLD_OK = 0,
  FOLD_E_INVALID = 1,       /* bad host-visible argument: null pointer, negative size,
                               unsupported S / cell / precision, schedule/model mismatch */
  FOLD_E_CHILD_RANGE = 2,   /* some child[n][k] not in [-1, n_nodes) */
  FOLD_E_ARITY = 3,         /* EMBED with a child, or CELL without two children */
  FOLD_E_TOKEN_RANGE = 4,   /* EMBED token not in [0, vocab) */
  FOLD_E_ROOT_RANGE = 5,    /* root[g] not in [0, n_nodes) (detail = g) */
  FOLD_E_CYCLE = 6,         /* the graph is not acyclic (PAPER.md L37 requires a DAG);
                               detail = smallest node that depends on a cycle */
  FOLD_E_WORKSPACE = 7,     /* workspace smaller than the *_workspace() query */
  FOLD_E_CUDA = 8,          /* a CUDA launch/copy failed */
  FOLD_E_MISMATCH = 9,      /* schedule and acts/model disagree (e.g. n_nodes) */
  FOLD_E_OP_RANGE = 10,     /* op[n] not in {FOLD_OP_EMBED, FOLD_OP_CELL} */
  FOLD_E_UNSUPPORTED = 11,  /* valid request this build does not implement
                               (e.g. not an sm_100 device) */
  FOLD_E_LEVEL = 12,        /* caller-fixed levels (fold_graphs.level) violate
                               level[n] in [1, n_nodes], level[EMBED] == 1,
                               level[CELL] > level[each child] */
} fold_status;

/* Operation ids = the enumeration order of PAPER.md L32/L43 ("all operations ... be
 * specified in advance, and it enumerates them"): a binary TreeRNN/TreeLSTM has two. */
enum { FOLD_OP_EMBED = 0, FOLD_OP_CELL = 1, FOLD_N_OPS = 2 };
/* Cell equations: DESIGN.md "Cell" (TreeRNN: Fig. 1 'RNN Cell', L67; TreeLSTM: Tai et
 * al. eqs 9-14 with x = 0, N = 2, cited at L301-304). */
enum { FOLD_CELL_TREERNN = 0, FOLD_CELL_TREELSTM = 1 };
/* FP32: states, gates, gradients fp32; the three GEMM passes on the tensor cores as
 *       3xTF32 (tcgen05 kind::tf32, x = hi + lo split, hi*hi + hi*lo + lo*hi, fp32
 *       accumulation in TMEM): fp32-class results (north_star bar 1e-5).
 * TF32: the FP32 mode's data and kernels with one kind::tf32 MMA per K step (operands
 *       read as TF32, 10 mantissa bits; north_star bar 1e-2).
 * BF16: states h, saved gates and GEMM operands in bf16, fp32 accumulation in TMEM
 *       (tcgen05), c / gradients / reductions in fp32 (the fused persistent kernels).  */
enum { FOLD_PREC_FP32 = 0, FOLD_PREC_TF32 = 1, FOLD_PREC_BF16 = 2 };

/* ----------------------------------------------------------------- input graphs
 * A batch of graphs = one disconnected DAG. Node n:
 *   op[n]            FOLD_OP_EMBED (leaf; consumes its depth-0 constant token[n]) or
 *                    FOLD_OP_CELL (consumes nodes child[2n], child[2n+1] = left, right).
 *   child[2n + k]    int32 node ids, -1 for "none" (EMBED: both -1).
 *   token[n]         int32 in [0, vocab) for EMBED; ignored for CELL.
 *   root[g]          int32 node whose state is graph g's result.
 * Any node order is accepted (children need not precede parents); DAG sharing and
 * child[2n] == child[2n+1] are allowed. All pointers are device.
 *   level[n]         OPTIONAL (NULL = dynamic batching). Caller-fixed schedule levels
 *                    that replace L40's depth: the "manual batching" baseline of
 *                    PAPER.md L83 / Table 1 ("we construct a static data-flow graph of
 *                    operations corresponding to the shape of the tree"), where every
 *                    tree position is its own operation, batched only across trees of
 *                    the same shape; with one tree it is the unbatched, node-at-a-time
 *                    evaluation. Requires level[n] in [1, n_nodes], == 1 for EMBED, and
 *                    level[n] > level[c] for each child c of a CELL (checked after
 *                    ROOT_RANGE, error FOLD_E_LEVEL, smallest offending node); levels
 *                    may skip values (empty levels are allowed). */
typedef struct {
  int32_t n_nodes, n_graphs, vocab;
  const int32_t *op, *child, *token, *root;
  const int32_t *level;
} fold_graphs;

/* ----------------------------------------------------------------- schedule
 * Executor-form schedule; all arrays device, caller-allocated with the sizes below
 * (N = n_nodes, G = n_graphs). Definitions (bit-exact with oracle/fold_oracle.c):
 *   depth[N]       PAPER.md L40: EMBED = 1 (its token constant is depth 0);
 *                  (with caller levels: depth[n] = level[n])
 *                  CELL = 1 + max(depth of children).
 *   perm[N]        pool row -> node: rows ordered by (depth, op, node id) (L42-43).
 *   rank[N]        node -> pool row (= perm^-1).
 *   gather[2N]     gather[2r + k] = rank[child[perm[r]][k]] for CELL rows, else -1 —
 *                  the edge label of L44 as a global pool row (the paper's per-depth
 *                  index i = gather - level_off[depth of child]).
 *   level_off[N+2] level_off[d] = #rows with depth < d, d = 0..n_levels+1.
 *   group_off[2N+3] group_off[k] = #rows with key < k, key = 2*depth + op, k = 0..2(D+1).
 *   cons_off[N+1], cons_edge[2N]
 *                  consumer CSR: for each pool row (ascending), the cell edges
 *                  e = 2c + k that read it, ascending; c = row - n_leaves is the cell
 *                  index (all EMBED rows precede all CELL rows).
 *   leaf_perm[N]   EMBED rows ordered by (token, row) (first n_leaves entries).
 *   tok_seg[N+1]   start of each distinct-token run of leaf_perm, + end sentinel
 *                  (first n_tok_segs + 1 entries).
 *   root_row[G]    rank[root[g]].
 *   root_perm[G]   graph ids ordered by (root_row, g) (deterministic seeding).
 *   leaf_token[N]  token of each EMBED row (first n_leaves entries): the depth-0
 *                  constants of PAPER.md L40/L47 ("int [] state", Fig. 1) in pool order.
 *   level_off_host host array [N+2]; receives level_off[0..n_levels+1].
 * Scalars n_levels (= max depth D), n_leaves, n_cells, n_tok_segs are outputs. */
typedef struct {
  int32_t *depth, *perm, *rank, *gather, *level_off, *group_off, *cons_off, *cons_edge,
          *leaf_perm, *tok_seg, *root_row, *root_perm, *leaf_token;
  int32_t *level_off_host;
  int32_t n_nodes, n_graphs, n_levels, n_leaves, n_cells, n_tok_segs;
  int32_t tree_like;  /* output: 1 if every pool row is read by at most one cell edge and the
                         rows read by none are exactly the (unconsumed) roots */
} fold_schedule_t;

/* Workspace bytes fold_schedule needs for n_nodes / n_graphs (device scratch). */
size_t fold_schedule_workspace(int32_t n_nodes, int32_t n_graphs);

/* Validate + schedule. Errors in this order (smallest offending id): CHILD_RANGE,
 * OP_RANGE, ARITY, TOKEN_RANGE, ROOT_RANGE, LEVEL (only with caller levels), CYCLE
 * (only without: strictly increasing levels exclude cycles). On error the schedule arrays are
 * unspecified. Exactly one blocking D2H copy (two if n_levels + 2 > 4096). */
fold_status fold_schedule(const fold_graphs *graphs, fold_schedule_t *sched,
                          void *d_workspace, size_t workspace_bytes, void *stream);

/* fold_schedule with a cap on the scheduler's grid (CTAs of its cooperative kernel; 0 = the
 * default sizing, values below 2 act as 2 on batches that need the cooperative kernel).
 * Same outputs, bit for bit, for any cap. For a schedule that runs BESIDE other work (the
 * next batch's schedule on a side stream overlapping this batch's weight-gradient GEMM,
 * SURVEY §8(f) NEXT-4): a few CTAs leave the GEMM its SMs (C4 B=1024 step
 * 21.5 -> 20.0-20.9 ms with 32 CTAs; C2 and C5 within noise). FOLD_E_INVALID if
 * max_blocks < 0. */
fold_status fold_schedule_ex(const fold_graphs *graphs, fold_schedule_t *sched,
                             void *d_workspace, size_t workspace_bytes, void *stream, int32_t max_blocks);

/* ----------------------------------------------------------------- model
 * Parameters are the caller's fp32 masters (device):
 *   U[gates*S][2S]  row-major, torch nn.Linear.weight order; gate row blocks
 *                   (i, f_L, f_R, o, u) for TreeLSTM, one block for TreeRNN; columns
 *                   [0,S) multiply h_L, [S,2S) multiply h_R.
 *   b[gates*S]      bias.
 *   E[vocab][S]     embedding table (leaf h = E[token], leaf c = 0).
 * BF16 mode converts U to bf16 inside fold_forward / fold_backward (workspace).
 * U, b and E must be 16-byte aligned (FOLD_E_INVALID otherwise). */
typedef struct {
  int32_t cell, prec, S, vocab;
  const float *U, *b, *E;
} fold_model;

/* ----------------------------------------------------------------- activations
 * One caller-owned device buffer holding everything the forward saves for the
 * backward (the pool of PAPER.md L47's loop state for every depth):
 *   H [N][ld] bf16 (BF16) or fp32 (FP32)  hidden state h per pool row (BF16: written only
 *                                         for rows without consumers; a consumed row's h
 *                                         lives in its consumers' A rows)
 *   C [N][ld] fp32                        cell state c per pool row (0 for TreeRNN; leaf
 *                                         rows are c = 0 by definition and are not
 *                                         materialised in BF16 mode)
 *   A_L, A_R [n_cells][ld] bf16 (BF16)    consumer-side operand planes: row c holds the h
 *                                         of cell c's left / right child (written by the
 *                                         producer of that child; read by the level GEMM
 *                                         and by the weight-gradient GEMM)
 *   G [n_cells][gates][ld] bf16 / fp32    saved gate activations (i, fL, fR, o, u)
 *                                         or h (TreeRNN) per cell; gate g of state
 *                                         column j at g*ld + j (every gate block starts
 *                                         16-byte aligned)
 * Offsets/strides come from fold_acts_layout; the buffer is otherwise opaque. */
typedef struct {
  size_t bytes;          /* total size of the buffer */
  size_t h_off, c_off, g_off;   /* byte offsets of H, C, G */
  int32_t ld;            /* row stride of H and C, in elements (>= S, multiple of 8) */
  int32_t h_elem_bytes;  /* 2 (bf16) or 4 (fp32) */
} fold_acts_layout_t;

fold_status fold_acts_layout(const fold_schedule_t *sched, const fold_model *model,
                             fold_acts_layout_t *layout);

size_t fold_forward_workspace(const fold_schedule_t *sched, const fold_model *model);

/* Forward over all levels. d_acts: buffer of fold_acts_layout().bytes.
 * d_h_root / d_c_root: [G][S] fp32 outputs (root h and c; either may be NULL). */
fold_status fold_forward(const fold_schedule_t *sched, const fold_model *model,
                         void *d_acts, float *d_h_root, float *d_c_root,
                         void *d_workspace, size_t workspace_bytes, void *stream);

/* ----------------------------------------------------------------- backward
 * Loss L = sum_g <dh_root[g], h_root(g)> + <dc_root[g], c_root(g)> (dc_root may be
 * NULL = 0). Outputs dU/db/dE with the layouts of U/b/E (device fp32). With
 * accumulate = 0 they are overwritten (dE rows of untouched tokens become 0);
 * with accumulate = 1 the gradients are added. Deterministic: bitwise-identical
 * results for identical inputs (no floating-point atomics). dU, db and dE must be
 * 16-byte aligned (FOLD_E_INVALID otherwise). */
typedef struct {
  float *dU, *db, *dE;
  int32_t accumulate;
  /* OPTIONAL (NULL = none): a cudaEvent_t recorded on the stream once the level sweep (the
   * dA GEMMs and pointwise steps) is enqueued, before the weight-gradient GEMM and the
   * embedding / bias reductions -- a caller may start independent work (e.g. the next
   * batch's fold_schedule on another stream) that overlaps them. */
  void *sweep_done_event;
} fold_grads;

size_t fold_backward_workspace(const fold_schedule_t *sched, const fold_model *model);

fold_status fold_backward(const fold_schedule_t *sched, const fold_model *model,
                          const void *d_acts, const float *d_dh_root, const float *d_dc_root,
                          fold_grads *grads, void *d_workspace, size_t workspace_bytes,
                          void *stream);

/* ----------------------------------------------------------------- §3.5 model (NEXT-2)
 * The sentiment model of PAPER.md L297-304: leaves h = TreeLSTM(Embedding(word), 0, 0)
 * (L300), internal nodes TreeLSTM(0, h_L, h_R) (L301), Tai et al. eqs 9-14 with N = 2
 * (L304), and a softmax classifier with cross-entropy at EVERY node ("every node has a
 * sentiment label", L297). Loss L = sum over all nodes n of -log softmax(Ws h_n + bs)[label].
 * The model's U, b, E are the fold_model's (cell must be FOLD_CELL_TREELSTM; prec FOLD_PREC_FP32
 * or FOLD_PREC_TF32, else FOLD_E_UNSUPPORTED); b's i, o, u blocks are shared by leaves and
 * cells. The leaf forget gates never contribute (c_L = c_R = 0, Tai eq 13), so there is no
 * W^(f). Roots play no special role (fold_graphs.root is only validated). All device:
 *   W[3S][S]         leaf input weights, row blocks (i, o, u); 16-byte aligned
 *   Ws[C][S], bs[C]  classifier; Ws 16-byte aligned
 *   label[n_nodes]   class of each node in NODE-ID order, in [0, C) (else the loss is NaN)
 *   n_classes        C in [1, 8] (5 for SST) */
typedef struct {
  const float *W, *Ws, *bs;
  const int32_t *label;
  int32_t n_classes;
} fold_sst;
/* gradients of W, Ws, bs (layouts as above), 16-byte aligned; fold_grads.accumulate applies */
typedef struct {
  float *dW, *dWs, *dbs;
} fold_sst_grads;

/* Activation buffer of the §3.5 model (its own layout; H / C fp32 for every pool row, saved
 * gates of leaves then cells at g_off) */
fold_status fold_sst_acts_layout(const fold_schedule_t *sched, const fold_model *model, const fold_sst *sst,
                                 fold_acts_layout_t *layout);
size_t fold_sst_forward_workspace(const fold_schedule_t *sched, const fold_model *model, const fold_sst *sst);
/* d_loss: device float[1] <- L. Per level a tcgen05 TF32 GEMM (the leaf level's A = the
 * embedding gather), a pointwise step, then the per-node classifier. */
fold_status fold_sst_forward(const fold_schedule_t *sched, const fold_model *model, const fold_sst *sst,
                             void *d_acts, float *d_loss, void *d_workspace, size_t workspace_bytes,
                             void *stream);
size_t fold_sst_backward_workspace(const fold_schedule_t *sched, const fold_model *model, const fold_sst *sst);
/* dL/d(U, b, E) into grads (sweep_done_event ignored) and dL/d(W, Ws, bs) into sst_grads. */
fold_status fold_sst_backward(const fold_schedule_t *sched, const fold_model *model, const fold_sst *sst,
                              const void *d_acts, fold_grads *grads, fold_sst_grads *sst_grads,
                              void *d_workspace, size_t workspace_bytes, void *stream);

/* ----------------------------------------------------------------- sparse dE exchange
 * (a data-parallel step needs only the embedding rows its
 * batch touched, so the ranks can all-gather those rows instead of all-reducing the whole
 * [V][S] table). All device pointers, stream-ordered, no host sync.
 *   fold_touched_rows    d_rows[0 .. n_tok_segs) = the batch's distinct tokens, ascending (one
 *                        per token segment of the schedule; n_tok_segs is the host count)
 *   fold_gather_rows     d_dst[i][0..S) = d_src[d_rows[i]][0..S)   (row stride ld of d_src;
 *                        d_rows[i] < 0: a zero row, i.e. padding)
 *   fold_scatter_add_rows d_dst[d_rows[i]][0..S) += d_src[i][0..S) (rows of one call must be
 *                        distinct; d_rows[i] < 0 skipped). Summing the ranks' packed rows
 *                        with one call per rank in rank order is deterministic. */
fold_status fold_touched_rows(const fold_schedule_t *sched, int32_t *d_rows, void *stream);
fold_status fold_gather_rows(const float *d_src, int64_t ld, const int32_t *d_rows, int32_t n, int32_t S,
                             float *d_dst, void *stream);
fold_status fold_scatter_add_rows(const float *d_src, const int32_t *d_rows, int32_t n, int32_t S,
                                  float *d_dst, int64_t ld, void *stream);

/* param[i] -= lr * grad[i], i < n (device fp32). SPEC S:L511 sgd_step. */
fold_status fold_sgd_update(float *d_param, const float *d_grad, int64_t n, float lr,
                            void *stream);

/* ----------------------------------------------------------------- misc */
const char *fold_status_string(fold_status s);
/* Detail of the last data-dependent error on this thread: the offending node (or
 * graph) id, -1 if none. */
int32_t fold_last_error_detail(void);
/* The persistent level kernels of fold_forward / fold_backward (BF16) leave n SMs free (rounded
 * up to CTA pairs; default 0) for work on other streams: the next batch's fold_schedule,
 * launched beside a small batch's latency-bound levels, then runs on those SMs instead of
 * waiting for the level kernels to finish. Process-wide, read at each launch;
 * returns the previous value; n < 0 acts as 0. Results stay deterministic for a given value;
 * across values they can differ in the last bits, because the backward's split-K choice for
 * latency-bound levels depends on the number of CTA pairs. */
int32_t fold_set_reserved_sms(int32_t n);

/* (node, depth, op) context of the last data-dependent fold_schedule error on this thread
 * (errors carry the depth and operation): node = the offending node (graph id
 * for FOLD_E_ROOT_RANGE); op = that node's op[] value as given (-1 for ROOT_RANGE); depth =
 * its caller-fixed level for FOLD_E_LEVEL, else -1 (every other class is detected before
 * depths exist: validation precedes depth propagation, and a cycle has none). Host pointers,
 * each may be NULL. Returns FOLD_OK if such an error is recorded, else FOLD_E_INVALID with
 * all three set to -1. */
fold_status fold_last_error_context(int32_t *node, int32_t *depth, int32_t *op);
int32_t fold_abi_version(void);
/* FOLD_OK if the current CUDA device is sm_100 (B200) and the kernels are loadable. */
fold_status fold_device_check(void);
/* Number of kernels this library launched on the calling thread since the last reset
 * (instrumentation for the bench's gpu_launches count). */
int64_t fold_launch_count(int32_t reset);

/* Instrumentation: with profiling on, every kernel class below is bracketed by a pair of
 * CUDA events recorded on the launch stream (calling thread only). fold_profile_enable
 * resets the records. fold_profile_read synchronizes on the recorded events and returns,
 * per class, the summed elapsed milliseconds and the number of bracketed launches.
 * Classes: 0 schedule (whole call), 1 embedding forward, 2 cell forward (the level sweep:
 * one bracket per call), 3 backward pointwise (BF16 tree path: the roots' seeded step),
 * 4 dA GEMM (the backward level sweep: one bracket per call; on the per-level paths it
 * includes each level's pointwise step), 5 dU GEMM, 6 embedding backward, 7 db column sum,
 * 8 SGD, 9 weight conversion, 10 root read-out. */
#define FOLD_PROF_NCLASS 11
void fold_profile_enable(int32_t on);
/* As fold_profile_enable(mask != 0), recording only the classes whose bit is set in mask
 * (bit c = class c): fewer events on the stream when one class is timed inside a long step. */
void fold_profile_enable_classes(uint32_t mask);
fold_status fold_profile_read(int32_t n_classes, double *ms, int64_t *launches);
/* Instrumentation: with FOLD_DBG_FWD=1 in the environment the BF16 forward kernel stamps
 * %globaltimer (ns) per pair tile at ten points: 0 producer starts the tile, 1 its
 * inputs are published, 2 its last MMA is issued, 3 its accumulator is ready in the
 * epilogue, 4 its outputs are published, 5 the epilogue may write its staging, 6 the
 * epilogue math is done, 7 the bulk stores have read the staging, 8 the bulk stores are
 * complete. Copies the first n_tiles stamps of each point into host[9][n_tiles] (tiles in
 * the kernel's order: levels ascending, row tile, column tile); returns the count, or -1
 * on a CUDA error. */
int32_t fold_debug_fwd_trace(unsigned long long *host, int32_t n_tiles);
/* Instrumentation: with FOLD_DBG_BWD=1 the wide backward kernel (k_bwd_levels) records
 * %globaltimer (ns) per pair tile at ten points: 0 producer starts the tile, 1 its inputs
 * (dZ rows, dCe) are published, 2 its accumulator is free, 3 its last MMA is issued, 4 the
 * accumulator is ready in the epilogue, 5 the epilogue has published, 6 the first epilogue
 * warp's first slab is in its transpose buffer, 7 that slab's pointwise rows are done,
 * 8 the tile's first pipeline stage has landed (MMA warp), 9 that warp's first row group
 * is done. Tiles in the kernel's order (levels descending from the first wide level, row
 * tile, column tile, k-half). Copies the first n_tiles stamps of each point into
 * host[10][n_tiles], then the SM clock64 values at points 8 and 3 into host[10..11][n_tiles]
 * (host holds 12 x n_tiles);
 * returns the count, or -1 on a CUDA error. */
int32_t fold_debug_bwd_trace(unsigned long long *host, int32_t n_tiles);
/* Instrumentation: with FOLD_DBG_SCHED=1, fold_schedule's block 0 stamps %globaltimer (ns)
 * at the start of phases P0..P11 and at its end; copies the 13 stamps into host[13] and
 * returns 13 (-1 on a CUDA error). */
int32_t fold_debug_sched_trace(unsigned long long *host);
/* Test hook: one tcgen05 TF32 GEMM of the FP32 / TF32 modes, C[M][N] (ldc) = A * B
 * (accumulate: +=). A is [M][K] row-major (a_mn = 0, K-major) or [K][M] (a_mn = 1); B is
 * [N][K] (b_mn = 0) or [K][N] (b_mn = 1); all device fp32, 16-byte aligned, ld % 4 == 0.
 * npass 1 = TF32, 3 = 3xTF32. ws: split-K scratch of fold_debug_gemm_tf32_ws(M, N, K)
 * floats (may be NULL: no split). */
fold_status fold_debug_gemm_tf32(const float *A, int64_t lda, int32_t a_mn, const float *B, int64_t ldb,
                                 int32_t b_mn, int32_t M, int32_t N, int32_t K, float *C, int64_t ldc,
                                 int32_t accumulate, int32_t npass, float *ws, int64_t ws_floats, void *stream);
int64_t fold_debug_gemm_tf32_ws(int32_t M, int32_t N, int32_t K);

#ifdef __cplusplus
}
#endif
#endif /* FOLD_H */

/*
 * fold_mo.h — C ABI of MULTI-OP dynamic batching: several operations
 * and tensor types per depth, §2 in full generality:
 *   L31  "dynamic batching schedules operations ... it enumerates them for scheduling
 *        purposes" — an op table, op id = enumeration position;
 *   L33  "The inputs and outputs of operations have tensor types ... fixed and fully
 *        specified in advance" — each op has an input and an output tensor type;
 *   L40  depth; L42 "Batch together all nodes invoking the same operation at the same
 *        depth"; L43 "Concatenate all outputs which have the same depth and tensor type.
 *        The order of concatenation corresponds to the order in which the dynamic batching
 *        operations were enumerated"; L44 edge labels (d, t, i);
 *   L47  the loop: per depth, every operation present runs once on its gathered inputs.
 * Conventions as in fold.h (caller-owned device buffers, void* stream, fold_status codes,
 * no exceptions, int32 row-major arrays, fp32 floats, thread-local error detail).
 *
 * Operation kinds (per op o; reading R30 in DESIGN.md):
 *   FOLD_MO_EMBED  arity 0:  h = E_o[token], c = 0                     (Fig. 1 embed lookup)
 *   FOLD_MO_LSTM   arity a:  N-ary TreeLSTM with x = 0 (Tai et al. eqs 9-14 as cited at
 *                  PAPER.md L301-304, N = a); in_type == out_type; U_o [(3+a) S][a S] with
 *                  row blocks (i, f_1..f_a, o, u) and column block k multiplying child k's h,
 *                  b_o [(3+a) S]:  c = i u + sum_k f_k c_k,  h = o tanh(c)
 *   FOLD_MO_RNN    arity a:  h = tanh(U_o [h_1; ..; h_a] + b_o), c = 0; U_o [S_out][a S_in]
 *                  (Fig. 1 "RNN Cell"; in_type != out_type makes it a typed projection)
 * a in {1, 2}. Every tensor type t carries (h, c) in R^{S_t}.
 */
#ifndef FOLD_MO_H
#define FOLD_MO_H

#include "fold.h"

#ifdef __cplusplus
extern "C" {
#endif

#define FOLD_MO_MAX_OPS 8
#define FOLD_MO_MAX_TYPES 4
enum { FOLD_MO_EMBED = 0, FOLD_MO_LSTM = 1, FOLD_MO_RNN = 2 };
/* additional status: a child's output type differs from its consumer's input type (L33) */
#define FOLD_E_TYPE 13

/* Op table (host struct). in_type is ignored for EMBED; vocab only for EMBED (> 0).
 * S[t] in [1, 4096]. Returns FOLD_E_INVALID from every call if malformed. */
typedef struct {
  int32_t n_ops, n_types;
  int32_t kind[FOLD_MO_MAX_OPS], arity[FOLD_MO_MAX_OPS], in_type[FOLD_MO_MAX_OPS],
          out_type[FOLD_MO_MAX_OPS], vocab[FOLD_MO_MAX_OPS];
  int32_t S[FOLD_MO_MAX_TYPES];
} fold_mo_table;

/* Input graphs (device): op[N] op ids; child[2N]: child[2n + k] for k < arity(op[n]), -1 in
 * the unused slots; token[N] (EMBED nodes); root[G]. Any node order, DAG sharing allowed. */
typedef struct {
  int32_t n_nodes, n_graphs;
  const int32_t *op, *child, *token, *root;
} fold_mo_graphs;

/* Schedule (all arrays device, caller-allocated with the capacities given; N = n_nodes,
 * G = n_graphs, K = n_ops, T = n_types). Definitional outputs, bit-exact with
 * oracle/fold_oracle_mo.c (oracle_mo_schedule):
 *   depth[N]          L40 (EMBED = 1; else 1 + max over children)
 *   group_off[(N+1)K+1] rows with key < k, key = depth*K + op: the batched operation
 *                     instances of L42 (first (D+1)K + 1 entries valid)
 *   type_off[T+1]     first row of each tensor type's pool in `pool`
 *   pool[N]           for t ascending: the nodes of output type t ordered by (depth, op, id)
 *                     (L43's concatenation per (depth, type), concatenated over depths)
 *   pool_row[N]       a node's row within its own type's pool
 *   tlevel_off[T(N+2)] compact [T][D+2]: rows of type t with depth < d
 *   label[6N]         edge (n, k) -> (d, t, i) of its child (L44), i = pool_row(child) -
 *                     tlevel_off[t][d]; (-1, -1, -1) for unused slots
 * Executor arrays:
 *   order[N]          nodes by (depth, op, id): group (d, o) = order[group_off[dK+o] ..)
 *   cons_off[N+1], cons_edge[2N]
 *                     consumers of each node by GLOBAL pool index (type_off[t] + pool_row):
 *                     edges e = 2 * (position of the consumer in order) + k, ascending
 *   root_off[N+1], root_graph[G]
 *                     graphs rooted at each node (by global pool index), ascending g
 *   leaf_seg[N+1], leaf_order[N], n_leaf_segs
 *                     EMBED nodes (as order positions) sorted by (op, token, position);
 *                     leaf_seg = start of each (op, token) run + end sentinel
 *   group_off_host    host [(N+1)K+1] capacity: receives group_off[0 .. (D+1)K]
 * Scalars: n_levels (= D), n_leaf_segs. fold_mo_schedule also records the input graphs'
 * device arrays (op, child, token, root): forward / backward read them, so they must stay
 * valid and unchanged while the schedule is used (schedules are immutable). */
typedef struct {
  int32_t *depth, *group_off, *type_off, *pool, *pool_row, *tlevel_off, *label;
  int32_t *order, *cons_off, *cons_edge, *root_off, *root_graph, *leaf_seg, *leaf_order;
  int32_t *group_off_host;
  int32_t n_nodes, n_graphs, n_levels, n_leaf_segs;
  const int32_t *op, *child, *token, *root;
} fold_mo_schedule_t;

size_t fold_mo_schedule_workspace(const fold_mo_table *table, int32_t n_nodes, int32_t n_graphs);

/* Validate + schedule. Errors in this order (smallest offending node id; graph id for
 * ROOT_RANGE): CHILD_RANGE, OP_RANGE, ARITY, TYPE, TOKEN_RANGE, ROOT_RANGE, CYCLE. One
 * blocking D2H copy (two when (D+1)K + 1 > 4096). */
fold_status fold_mo_schedule(const fold_mo_table *table, const fold_mo_graphs *graphs,
                             fold_mo_schedule_t *sched, void *d_workspace, size_t workspace_bytes,
                             void *stream);

/* Parameters (device fp32, 16-byte aligned): per op o, EMBED: E[o] [vocab][S_out];
 * LSTM / RNN: U[o] and b[o] in the layouts above. prec: FOLD_PREC_FP32 (3xTF32 tensor
 * cores, 1e-5 class) or FOLD_PREC_TF32 (1e-2 class); FOLD_PREC_BF16 -> FOLD_E_UNSUPPORTED. */
typedef struct {
  int32_t prec;
  const float *U[FOLD_MO_MAX_OPS], *b[FOLD_MO_MAX_OPS], *E[FOLD_MO_MAX_OPS];
} fold_mo_model;
typedef struct {
  float *dU[FOLD_MO_MAX_OPS], *db[FOLD_MO_MAX_OPS], *dE[FOLD_MO_MAX_OPS];  /* NULL for unused */
  int32_t accumulate;
} fold_mo_grads;

/* Activations (opaque device buffer): per type t the pool H_t, C_t [n_t][ld_t] fp32 (ld_t =
 * S_t rounded up to 4); per op its op-major slab of gathered inputs A_o [rows_o][a S_in] and
 * saved gates Z_o [rows_o][(3+a) S | S]. */
size_t fold_mo_acts_bytes(const fold_mo_table *table, const fold_mo_schedule_t *sched);
size_t fold_mo_forward_workspace(const fold_mo_table *table, const fold_mo_schedule_t *sched);

/* Forward over all levels: per depth ONE gather launch (all of the level's ops), ONE grouped
 * tcgen05 GEMM launch (every op's tiles) and ONE pointwise launch. d_h_root: [G][S_max] fp32
 * (graph g fills the first S_{type(root g)} entries, the rest 0), may be NULL. */
fold_status fold_mo_forward(const fold_mo_table *table, const fold_mo_schedule_t *sched,
                            const fold_mo_model *model, void *d_acts, float *d_h_root,
                            void *d_workspace, size_t workspace_bytes, void *stream);

size_t fold_mo_backward_workspace(const fold_mo_table *table, const fold_mo_schedule_t *sched);

/* Loss L = sum_g <dh_root[g][0 .. S_{type(root g)}), h_root(g)> (d_dh_root [G][S_max]).
 * Reverse sweep per depth (one pull-reduction + pointwise launch, one grouped dA GEMM), then
 * one grouped weight-gradient GEMM over every op's slab, fixed-order bias sums and the
 * per-(op, token) embedding reductions. Deterministic (no floating-point atomics). */
fold_status fold_mo_backward(const fold_mo_table *table, const fold_mo_schedule_t *sched,
                             const fold_mo_model *model, const void *d_acts, const float *d_dh_root,
                             fold_mo_grads *grads, void *d_workspace, size_t workspace_bytes,
                             void *stream);

#ifdef __cplusplus
}
#endif

#endif  /* FOLD_MO_H */

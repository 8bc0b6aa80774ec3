// exec.cuh — declarations shared by the executor translation units.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace fold {

// Consumer-side operand planes (BF16 path): the forward "gather" is done at production
// time — every produced row r is also written to the A operand row of each consumer edge
// e = 2c + k in cons(r): A_k[c] = h(r). Level d's GEMM then reads its A rows
// [c0, c0 + M_d) of A_L / A_R densely with TMA (no gather on the MMA critical path), and
// the weight-gradient GEMM reads the same planes as its dense B operand.
struct ScatterA {
  const int32_t *cons_off, *cons_edge;
  __nv_bfloat16 *AL, *AR;  // [n_cells][ld] each
  int ld;
};

// Activation / workspace layouts (pure functions of the schedule and model).
struct ActsLayout {
  size_t bytes, h_off, c_off, g_off, al_off, ar_off;
  int ld;       // H, C row stride (elements)
  int ld_g;     // G row stride (elements) = gates * ld; gate g at g * ld
  int helem;    // bytes per H / G element
};
ActsLayout acts_layout(const fold_schedule_t *s, const fold_model *m);

inline int gates_of(int cell) { return cell == FOLD_CELL_TREELSTM ? 5 : 1; }

// --- SIMT / shared kernels (exec.cu)
fold_status launch_embed_fwd(bool bf16, int r0, int r1, const int32_t *leaf_token, const float *E, int S, int ld,
                             void *H, float *C, const ScatterA *sc, cudaStream_t st);
fold_status launch_cell_fwd_simt(int cell, int r0, int r1, const int32_t *gather, int S, int ld,
                                 const float *U, const float *b, float *H, float *C, float *Gact, int ld_g,
                                 int nl, cudaStream_t st);
fold_status launch_root_out(bool bf16, int G, int S, int ld, int nl, const int32_t *root_row, const void *H,
                            const float *C, float *h_root, float *c_root, const ScatterA *sc, cudaStream_t st);
fold_status launch_cell_bwd_pw(bool bf16, int cell, int r0, int r1, int nl, int S, int ld, int ld_g,
                               const int32_t *cons_off, const int32_t *cons_edge, const int32_t *root_off,
                               const int32_t *root_perm, int G, const float *dh_root, const float *dc_root,
                               const int32_t *gather, const void *Gact, const float *C, const float *dA,
                               float *dCe, void *dZ, int ld_z, cudaStream_t st,
                               const int32_t *root_row = nullptr,  // root mode: rows = distinct root rows, [r0,r1)=[0,G)
                               const float *dh_node = nullptr,     // + per-node dh [N][S] (pool rows; §3.5 classifier)
                               bool leaf_c = false);               // leaves carry c (the §3.5 leaf cell)
// dA[rows][2S] (edge-indexed, fp32) = dZ[rows][gates*S] * U[gates*S][2S]
fold_status launch_gemm_dA_simt(int M, int S, int gates, const float *dZ, int ld_z, const float *U,
                                float *dA, cudaStream_t st);
// dU[gates*S][2S] (+)= sum_c dZ[c] (x) [H[gL(c)]; H[gR(c)]]
fold_status launch_gemm_dU_simt(int n_cells, int nl, int S, int gates, const float *dZ, int ld_z,
                                const int32_t *gather, const float *H, int ld, float *dU, int accumulate,
                                cudaStream_t st);
// db[j] (+)= sum_c dZ[c][j], fixed-order partials then fixed-order total
fold_status launch_colsum(bool bf16, int n_rows, int ncols, const void *dZ, int ld_z, float *partial,
                          int nsplit, float *db, int accumulate, cudaStream_t st);
fold_status launch_embed_bwd(int S, int nl, int n_tok_segs, const int32_t *tok_seg, const int32_t *leaf_perm,
                             const int32_t *leaf_token, const int32_t *cons_off,
                             const int32_t *cons_edge, const int32_t *root_off, const int32_t *root_perm, int G,
                             const float *dh_root, const float *dA, float *dE, cudaStream_t st);
fold_status launch_root_off(int N, int G, const int32_t *root_row, const int32_t *root_perm, int32_t *root_off,
                            cudaStream_t st);
fold_status launch_sgd(float *p, const float *g, int64_t n, float lr, cudaStream_t st);
fold_status launch_touched_rows(int n_seg, const int32_t *tok_seg, const int32_t *leaf_perm,
                                const int32_t *leaf_token, int32_t *rows, cudaStream_t st);
fold_status launch_gather_rows(const float *src, int64_t ld, const int32_t *rows, int n, int S, float *dst,
                               cudaStream_t st);
fold_status launch_scatter_add_rows(const float *src, const int32_t *rows, int n, int S, float *dst, int64_t ld,
                                    cudaStream_t st);
// exclusive int32 scan (sched.cu)
fold_status scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *sums, int32_t *total,
                           cudaStream_t st);
int64_t scan_sums_count(int64_t n);
// embedding gradient, segmented by token, long segments split into fixed pieces
constexpr int kEmbedPiece = 64;
struct EmbedBwdWs {
  int32_t *piece_cnt, *piece_off, *scan_sums;
  int32_t *piece_seg;  // [n_leaves / kEmbedPiece + n_tok_segs + 1]: segment of each piece
  float *partial;
};
fold_status launch_embed_bwd_pieces(int S, int n_leaves, int n_tok_segs, const int32_t *tok_seg,
                                    const int32_t *leaf_perm, const int32_t *leaf_token, const int32_t *cons_off,
                                    const int32_t *cons_edge, const int32_t *root_off, const int32_t *root_perm,
                                    const float *dh_root, const void *dA, bool dA_bf16, float *dE,
                                    const EmbedBwdWs &w, cudaStream_t st,
                                    const float *dX = nullptr);  // dense per-leaf gradient [nl][S] (§3.5)
fold_status launch_zero(void *p, size_t bytes, cudaStream_t st);

// --- tcgen05 path (exec_tc.cu)
// bf16 copies of U per call, [rows][ld_u] with K halves padded to Sp = round_up(S, 64)
// (ld_u = 2 Sp): natural row order for the backward's dA GEMM (MN-major B operand),
// gate-interleaved in 8-column blocks for the forward (K-major B operand, one TMA box).
int tc_ld_u(int S);
int tc_debug_fwd_trace(unsigned long long *host, int n);
int tc_debug_bwd_trace(unsigned long long *host, int n);
size_t tc_ut_bytes(int gates, int S);
size_t tc_weights_bytes(int gates, int S);
fold_status tc_prepare_U(int gates, int S, const float *U, __nv_bfloat16 *Ub, cudaStream_t st);
// the forward's gate-interleaved copy (Uil8, same size)
fold_status tc_prepare_Uil(int gates, int S, const float *U, __nv_bfloat16 *Uil, cudaStream_t st);
// All cell levels d = 2..D of the forward in one persistent launch.
struct TcFwdArgs {
  const int32_t *level_off;       // device
  const int32_t *level_off_host;  // host copy (tile count)
  int D, S, nl, n_cells, ld, ld_g, ld_u;
  const int32_t *gather;
  const __nv_bfloat16 *Ub;
  const float *b;
  __nv_bfloat16 *H, *Gact;
  float *C;
  ScatterA sc;
  int *rt_cnt;                     // [n_cells] per-row-tile counters (workspace)
  int32_t *tstart;                 // [n_cells] first cell of each cell's row tile (workspace)
};
fold_status tc_fwd_levels(int cell, const TcFwdArgs &a, cudaStream_t st);
// Tree-like schedules: the dA GEMM of every level in one persistent launch, each tile's
// epilogue running the children's backward pointwise step (dZ, dCe); dA kept for leaves.
struct TcBwdArgs {
  const int32_t *level_off, *level_off_host;
  int D, S, nl, n_cells, ld, ld_g, ld_z;
  const int32_t *gather;
  const float *U;        // fp32 master (the narrow backward's transposed copy is made from it)
  __nv_bfloat16 *Ut;     // workspace [2 Sp][gates*S] for that copy
  const __nv_bfloat16 *Ub, *Gact;
  const float *C;
  float *dA, *dCe;
  __nv_bfloat16 *dZ;
  int *rt_cnt;       // [n_cells] per-row-tile completion counters (keyed by a tile's first cell)
  int32_t *tstart;   // [n_cells] first cell of each cell's row tile
  float *ks_ring;    // [kKsRing][kKsSlotFloats] split-K hand-over slots (k_bwd_levels)
  int *ks_cnt;       // [2 * kKsRing] their written / read counts (zeroed by tc_bwd_prelude)
  int *lvl_tab;      // [tc_bwd_lvl_tab_ints(D)] per-level tile tables of k_bwd_levels
};
// per level d <= D: three int4 (critical units, deferred tiles run inline, deferred tiles run
// at the end) and one flag word, + the total
inline int64_t tc_bwd_lvl_tab_ints(int64_t D) { return (D + 2) * 13 + 8; }
// split-K hand-over ring of the wide backward (see k_bwd_levels)
constexpr int kKsRing = 256;
constexpr int kKsSlotFloats = 2 * 128 * 128;
inline size_t tc_ks_ring_bytes() { return (size_t)kKsRing * kKsSlotFloats * 4; }
// tile bookkeeping (zero counters, tstart, roots' pre-credit); before the seeded pass
fold_status tc_bwd_prelude(const TcBwdArgs &a, const int32_t *cons_off, cudaStream_t st);
fold_status tc_bwd_levels(int cell, const TcBwdArgs &a, cudaStream_t st);
fold_status tc_gemm_dA(int c0, int M, int n_cells, int S, int gates, const __nv_bfloat16 *dZ, int ld_z,
                       const __nv_bfloat16 *Ub, float *dA, cudaStream_t st);
// split-K over cells into split_ws [splits][gates*S][2S] (fp32), then a fixed-order sum
int tc_dU_splits(int n_cells, int gates, int S);
int set_reserved_sms(int n);  // fold_set_reserved_sms
fold_status tc_gemm_dU(int n_cells, int S, int gates, const __nv_bfloat16 *dZ, int ld_z, const ScatterA &sc,
                       float *dU, int accumulate, float *split_ws, float *db, float *db_ws,
                       cudaStream_t st);

// out[i] = (accumulate ? out[i] : 0) + sum_{s < nsplit} part[s][i] in fixed order
fold_status launch_reduce_splits(int64_t n, int nsplit, const float *part, float *out, int accumulate,
                                 cudaStream_t st);

// --- tcgen05 TF32 GEMM (gemm_tf32.cu): the FP32 (3xTF32) and TF32 modes' contractions.
// An operand is a row-major fp32 matrix in global memory read either K-major (rows = M or
// N, K contiguous) or MN-major (rows = K, M or N contiguous); ld in elements, ld * 4 and the
// base 16-byte aligned (TMA).
struct TfOperand {
  const float *p;
  int64_t ld;
  int mn_major;
};
// C[M][N] (ldc) = A * B (accumulate: C +=) with fp32 accumulation in TMEM. npass = 1: one
// kind::tf32 MMA per K step (TF32 mode); npass = 3: 3xTF32 (A_hi B_hi + A_hi B_lo +
// A_lo B_hi, the lo parts split in shared memory): fp32-class accuracy (FP32 mode).
// split_ws (nullable, split_ws_floats capacity): split-K partials for small tile counts,
// reduced in fixed order (deterministic).
fold_status gemm_tf32(const TfOperand &A, const TfOperand &B, int M, int N, int K, float *C, int64_t ldc,
                      int accumulate, int npass, float *split_ws, int64_t split_ws_floats, cudaStream_t st);
int64_t gemm_tf32_split_floats(int M, int N, int K);
// Grouped TF32 GEMM (multi-op levels, fold_mo.h): up to kTfGroupMax independent problems
// C_i = A_i * B_i in ONE launch (problems with M or N <= 0 are skipped); split-K partials of
// the problems that use them go to split_ws (gemm_tf32_grouped_ws_floats floats).
constexpr int kTfGroupMax = 8;
struct TfProblem {
  TfOperand A, B;
  int M, N, K;
  float *C;
  int64_t ldc;
  int accumulate;
};
struct alignas(64) TfGroupArgs {
  CUtensorMap ta[kTfGroupMax], tb[kTfGroupMax];
  int a_mn[kTfGroupMax], b_mn[kTfGroupMax], M[kTfGroupMax], N[kTfGroupMax], K[kTfGroupMax];
  int kbps[kTfGroupMax], nsplit[kTfGroupMax], ntn[kTfGroupMax], accumulate[kTfGroupMax];
  float *C[kTfGroupMax];
  int64_t ldc[kTfGroupMax], split_stride[kTfGroupMax];
  int tile_start[kTfGroupMax + 1];
  int n;
};
fold_status gemm_tf32_grouped(const TfProblem *q, int n, int npass, float *split_ws, int64_t split_ws_floats,
                              cudaStream_t st);
int64_t gemm_tf32_grouped_ws_floats(const TfProblem *q, int n, int npass);
// FP32 / TF32 mode level helpers (gemm_tf32.cu)
// Acat[c][0:S] = H[gather[2r]], Acat[c][S:2S] = H[gather[2r+1]] for rows r in [r0, r1), c = r - nl
fold_status launch_gather_cat(int r0, int r1, int nl, int S, int ld, const int32_t *gather, const float *H,
                              float *Acat, int64_t ld_a, cudaStream_t st);
// Z rows of the level are in Gact (gate g of column j at g*ld + j): gates, c, h in place
fold_status launch_cell_fwd_pw(int cell, int r0, int r1, int nl, int S, int ld, int ld_g, const int32_t *gather,
                               const float *b, float *H, float *C, float *Gact, cudaStream_t st);
// U copies for the TF32 GEMMs: fwd rows gate-padded (row g*ld + j <- U row g*S + j, zero for
// j >= S), bwd rows natural; both [rows][ld_u] with ld_u = round_up(2S, 4)
int64_t tf_ld_u(int S);
fold_status launch_prep_U_tf(int gates, int S, int ld, const float *U, float *Ufwd, float *Ubwd, cudaStream_t st);

}  // namespace fold

// abi.cu — the extern "C" entry points declared in include/fold.h: argument checks,
// workspace carving and launch sequencing of the level loop (one
// iteration per depth) forward and in reverse for the backward (L49).
#include <cstring>

#include "../../include/fold_mo.h"
#include "exec.cuh"

namespace fold {

fold_status run_schedule(const fold_graphs *gr, fold_schedule_t *s, void *ws, size_t ws_bytes, int max_blocks,
                         cudaStream_t st);
int debug_sched_trace(unsigned long long *host);
size_t schedule_workspace(int64_t N, int64_t G);
size_t mo_schedule_workspace(const fold_mo_table *t, int64_t N, int64_t G);
fold_status run_mo_schedule(const fold_mo_table *t, const fold_mo_graphs *gr, fold_mo_schedule_t *s, void *ws,
                            size_t ws_bytes, cudaStream_t st);
size_t mo_acts_bytes(const fold_mo_table *t, const fold_mo_schedule_t *s);
size_t mo_forward_workspace(const fold_mo_table *t, const fold_mo_schedule_t *s);
size_t mo_backward_workspace(const fold_mo_table *t, const fold_mo_schedule_t *s);
fold_status mo_forward(const fold_mo_table *t, const fold_mo_schedule_t *s, const fold_mo_model *model, void *acts,
                       float *h_root, void *ws, size_t ws_bytes, cudaStream_t st);
fold_status mo_backward(const fold_mo_table *t, const fold_mo_schedule_t *s, const fold_mo_model *model,
                        const void *acts, const float *dh_root, fold_mo_grads *gr, void *ws, size_t ws_bytes,
                        cudaStream_t st);
extern thread_local int32_t g_last_detail;
extern thread_local int32_t g_last_ctx[3];

namespace {

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

fold_status check_model(const fold_model *m) {
  if (!m || !m->U || !m->b || !m->E) return FOLD_E_INVALID;
  if (m->cell != FOLD_CELL_TREERNN && m->cell != FOLD_CELL_TREELSTM) return FOLD_E_INVALID;
  if (m->prec != FOLD_PREC_FP32 && m->prec != FOLD_PREC_TF32 && m->prec != FOLD_PREC_BF16) return FOLD_E_INVALID;
  if (m->S <= 0 || m->S > 8192 || m->vocab <= 0) return FOLD_E_INVALID;
  // vectorised loads: parameter arrays must be 16-byte aligned
  if (((uintptr_t)m->U | (uintptr_t)m->b | (uintptr_t)m->E) & 15) return FOLD_E_INVALID;
  return FOLD_OK;
}

fold_status check_sched(const fold_schedule_t *s) {
  if (!s || s->n_nodes < 0 || s->n_levels < 0 || !s->level_off_host) return FOLD_E_INVALID;
  if (s->n_nodes > 0 && (!s->perm || !s->gather || !s->cons_off || !s->cons_edge)) return FOLD_E_INVALID;
  return FOLD_OK;
}

// FOLD_FP32_SIMT=1 (A/B measurements only): the FP32 mode's contractions on the previous
// SIMT FFMA kernels instead of the 3xTF32 tensor-core GEMMs
bool simt_fp32() {
  static const bool v = [] { const char *e = getenv("FOLD_FP32_SIMT"); return e && atoi(e) != 0; }();
  return v;
}
size_t tf_u_bytes(int gates, int S) {
  return a256((size_t)gates * ld_of(S) * tf_ld_u(S) * 4);
}
inline int npass_of(int prec) { return prec == FOLD_PREC_TF32 ? 1 : 3; }
inline int64_t tf_ld_a(int S) { return round_up(2 * (int64_t)S, 8); }

// backward workspace carve
struct BwdWs {
  float *dA, *dCe, *partial, *dU_split;
  int32_t *root_off;
  int *rt_cnt;      // [n_cells] row-tile counters of the fused backward
  int32_t *tstart;  // [n_cells]
  float *ks_ring;   // its split-K hand-over slots (BF16 path)
  int *ks_cnt;
  int *lvl_tab;     // the wide backward's per-level tile tables (tc_bwd_lvl_tab_ints)
  EmbedBwdWs emb;
  void *dZ;
  __nv_bfloat16 *Ub, *Ut;
  float *Utf;               // FP32 / TF32 modes: the natural-row U copy (MN-major B of dA)
  int64_t tf_split_floats;  // their dU GEMM's split-K partials
  int ld_z, nsplit;
  size_t bytes;
};

BwdWs bwd_layout(void *base, const fold_schedule_t *s, const fold_model *m) {
  BwdWs b{};
  const int64_t nc = s->n_cells, S = m->S;
  const int gates = gates_of(m->cell);
  const bool bf16 = m->prec == FOLD_PREC_BF16;
  b.ld_z = (int)round_up((int64_t)gates * S, 8);
  b.nsplit = (int)(nc / 128 < 1 ? 1 : (nc / 128 > 256 ? 256 : nc / 128));
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = a256(off + bytes); return o; };
  size_t o_dA = take((size_t)(2 * nc + 1) * S * 4);
  size_t o_dCe = take(gates == 5 ? (size_t)(2 * nc + 1) * S * 4 : 256);
  size_t o_dZ = take((size_t)(nc + 1) * b.ld_z * (bf16 ? 2 : 4));
  size_t o_part = take((size_t)b.nsplit * gates * S * 4);
  size_t o_roff = take((size_t)(s->n_nodes + 2) * 4);
  size_t o_rtc = take((size_t)(nc + 1) * 4), o_ts = take((size_t)(nc + 1) * 4);
  const int64_t nseg = s->n_tok_segs;
  const int64_t max_pieces = s->n_leaves / kEmbedPiece + nseg + 1;
  size_t o_pc = take((size_t)(nseg + 2) * 4), o_po = take((size_t)(nseg + 2) * 4);
  size_t o_ss = take((size_t)scan_sums_count(nseg + 1) * 4);
  size_t o_psg = take((size_t)max_pieces * 4);
  size_t o_ep = take((size_t)max_pieces * S * 4);
  const bool tf = !bf16 && !simt_fp32();
  size_t o_w = take(bf16 ? tc_weights_bytes(gates, (int)S) : tf ? tf_u_bytes(gates, (int)S) : 0);
  size_t o_ut = take(bf16 ? tc_ut_bytes(gates, (int)S) : 0);
  const int splits = bf16 ? tc_dU_splits((int)nc, gates, (int)S) : 1;
  const int64_t tf_split = tf ? gemm_tf32_split_floats(gates * (int)S, 2 * (int)S, (int)nc) : 0;
  b.tf_split_floats = tf_split;
  size_t o_spl = take(splits > 1 ? (size_t)splits * gates * S * 2 * S * 4 : (size_t)tf_split * 4);
  size_t o_ksr = take(bf16 ? tc_ks_ring_bytes() : 0), o_ksc = take(bf16 ? (size_t)2 * kKsRing * 4 : 0);
  size_t o_lvt = take(bf16 ? (size_t)tc_bwd_lvl_tab_ints(s->n_levels) * 4 : 0);
  b.bytes = off;
  if (base) {
    char *p = (char *)base;
    b.dA = (float *)(p + o_dA);
    b.dCe = (float *)(p + o_dCe);
    b.dZ = p + o_dZ;
    b.partial = (float *)(p + o_part);
    b.root_off = (int32_t *)(p + o_roff);
    b.rt_cnt = (int *)(p + o_rtc);
    b.tstart = (int32_t *)(p + o_ts);
    b.emb.piece_cnt = (int32_t *)(p + o_pc);
    b.emb.piece_off = (int32_t *)(p + o_po);
    b.emb.scan_sums = (int32_t *)(p + o_ss);
    b.emb.piece_seg = (int32_t *)(p + o_psg);
    b.emb.partial = (float *)(p + o_ep);
    b.dU_split = (splits > 1 || tf_split > 0) ? (float *)(p + o_spl) : nullptr;
    b.Ub = bf16 ? (__nv_bfloat16 *)(p + o_w) : nullptr;
    b.Utf = tf ? (float *)(p + o_w) : nullptr;
    b.Ut = bf16 ? (__nv_bfloat16 *)(p + o_ut) : nullptr;
    b.ks_ring = bf16 ? (float *)(p + o_ksr) : nullptr;
    b.ks_cnt = bf16 ? (int *)(p + o_ksc) : nullptr;
    b.lvl_tab = bf16 ? (int *)(p + o_lvt) : nullptr;
  }
  return b;
}

// Library-owned auxiliary stream (one per host thread and device), used to overlap
// independent memory-bound kernels with tensor-bound ones inside one ABI call; ordering
// with the caller's stream is by events, so the call stays stream-ordered for the caller.
struct AuxStream {
  bool ok = false;
  int dev = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
AuxStream &aux_stream() {
  static thread_local AuxStream ax[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) {
    static AuxStream none;
    return none;
  }
  AuxStream &a = ax[dev];
  if (!a.ok) {
    a.ok = cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming) == cudaSuccess;
    a.dev = dev;
  }
  return a;
}

// forward workspace (BF16 path): bf16 U, then the row-tile counters and tile starts
size_t fwd_ws_bytes(const fold_schedule_t *s, const fold_model *m) {
  if (m->prec != FOLD_PREC_BF16) return simt_fp32() ? 256 : tf_u_bytes(gates_of(m->cell), m->S);
  return tc_weights_bytes(gates_of(m->cell), m->S) + 2 * a256((size_t)(s->n_cells + 1) * sizeof(int));
}

}  // namespace

ActsLayout acts_layout(const fold_schedule_t *s, const fold_model *m) {
  ActsLayout L{};
  const int64_t N = s->n_nodes, nc = s->n_cells, S = m->S;
  const int gates = gates_of(m->cell);
  L.helem = m->prec == FOLD_PREC_BF16 ? 2 : 4;
  L.ld = ld_of((int)S);
  L.ld_g = gates * L.ld;  // G row = gates blocks of ld (16-byte aligned gate blocks)
  size_t off = 0;
  L.h_off = off; off = a256(off + (size_t)(N + 1) * L.ld * L.helem);
  L.c_off = off; off = a256(off + (size_t)(N + 1) * L.ld * 4);
  L.g_off = off; off = a256(off + (size_t)(nc + 1) * L.ld_g * L.helem);
  const bool planes = m->prec == FOLD_PREC_BF16;
  // BF16: the two push-gathered operand planes A_L / A_R; FP32 / TF32: one gathered fp32
  // plane Acat [n_cells][round_up(2S, 8)] (the level GEMMs' A, the dU GEMM's B)
  const bool cat = !planes && !simt_fp32();
  L.al_off = off;
  off = a256(off + (planes ? (size_t)(nc + 1) * L.ld * 2 : cat ? (size_t)(nc + 1) * tf_ld_a((int)S) * 4 : 0));
  L.ar_off = off; off = a256(off + (planes ? (size_t)(nc + 1) * L.ld * 2 : 0));
  L.bytes = off;
  return L;
}

}  // namespace fold

using namespace fold;

extern "C" {

size_t fold_schedule_workspace(int32_t n_nodes, int32_t n_graphs) {
  return schedule_workspace(n_nodes < 0 ? 0 : n_nodes, n_graphs < 0 ? 0 : n_graphs);
}

fold_status fold_schedule(const fold_graphs *graphs, fold_schedule_t *sched, void *ws, size_t ws_bytes,
                          void *stream) {
  ProfScope ps(K_SCHED, (cudaStream_t)stream);
  return run_schedule(graphs, sched, ws, ws_bytes, 0, (cudaStream_t)stream);
}

fold_status fold_schedule_ex(const fold_graphs *graphs, fold_schedule_t *sched, void *ws, size_t ws_bytes,
                             void *stream, int32_t max_blocks) {
  ProfScope ps(K_SCHED, (cudaStream_t)stream);
  if (max_blocks < 0) return FOLD_E_INVALID;
  return run_schedule(graphs, sched, ws, ws_bytes, max_blocks, (cudaStream_t)stream);
}

fold_status fold_acts_layout(const fold_schedule_t *s, const fold_model *m, fold_acts_layout_t *out) {
  FOLD_TRY(check_sched(s));
  FOLD_TRY(check_model(m));
  if (!out) return FOLD_E_INVALID;
  ActsLayout L = acts_layout(s, m);
  out->bytes = L.bytes; out->h_off = L.h_off; out->c_off = L.c_off; out->g_off = L.g_off;
  out->ld = L.ld; out->h_elem_bytes = L.helem;
  return FOLD_OK;
}

size_t fold_forward_workspace(const fold_schedule_t *s, const fold_model *m) {
  if (check_sched(s) != FOLD_OK || check_model(m) != FOLD_OK) return 0;
  return fwd_ws_bytes(s, m);
}

// Forward level loop: depth 1 = embedding lookup, depth d >= 2 = one
// batched cell invocation over the level's contiguous pool rows [lo[d], lo[d+1]).
fold_status fold_forward(const fold_schedule_t *s, const fold_model *m, void *acts, float *h_root, float *c_root,
                         void *ws, size_t ws_bytes, void *stream) {
  FOLD_TRY(check_sched(s));
  FOLD_TRY(check_model(m));
  if (!acts && s->n_nodes > 0) return FOLD_E_INVALID;
  if (ws_bytes < fwd_ws_bytes(s, m) || (!ws && m->prec == FOLD_PREC_BF16)) return FOLD_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = s->n_nodes, S = m->S, D = s->n_levels, nl = s->n_leaves, G = s->n_graphs;
  if (N == 0) return FOLD_OK;
  if (!s->leaf_token || !s->root_row) return FOLD_E_INVALID;
  const bool bf16 = m->prec == FOLD_PREC_BF16;
  const int gates = gates_of(m->cell);
  ActsLayout L = acts_layout(s, m);
  char *a = (char *)acts;
  void *H = a + L.h_off;
  float *C = (float *)(a + L.c_off);
  void *Gact = a + L.g_off;
  const int32_t *lo = s->level_off_host;
  ScatterA sc{s->cons_off, s->cons_edge, (__nv_bfloat16 *)(a + L.al_off), (__nv_bfloat16 *)(a + L.ar_off), L.ld};
  {
    ProfScope ps(K_EMBED_FWD, st);
    FOLD_TRY(launch_embed_fwd(bf16, lo[1], lo[2], s->leaf_token, m->E, S, L.ld, H, C, bf16 ? &sc : nullptr, st));
  }
  if (bf16) {
    __nv_bfloat16 *Ub = (__nv_bfloat16 *)ws;
    if (D >= 2) {
      {
        ProfScope ps(K_PREP, st);
        FOLD_TRY(tc_prepare_Uil(gates, S, m->U, Ub, st));
      }
      TcFwdArgs fa{};
      fa.level_off = s->level_off; fa.level_off_host = lo;
      fa.D = D; fa.S = S; fa.nl = nl; fa.n_cells = s->n_cells; fa.ld = L.ld; fa.ld_g = L.ld_g; fa.ld_u = tc_ld_u(S);
      fa.gather = s->gather; fa.Ub = Ub; fa.b = m->b;
      fa.H = (__nv_bfloat16 *)H; fa.Gact = (__nv_bfloat16 *)Gact; fa.C = C; fa.sc = sc;
      fa.rt_cnt = (int *)((char *)ws + tc_weights_bytes(gates, S));
      fa.tstart = (int32_t *)((char *)fa.rt_cnt + a256((size_t)(s->n_cells + 1) * sizeof(int)));
      ProfScope ps(K_CELL_FWD, st);
      FOLD_TRY(tc_fwd_levels(m->cell, fa, st));
    }
  } else if (simt_fp32()) {
    ProfScope ps(K_CELL_FWD, st);  // one bracket around the level sweep
    for (int d = 2; d <= D; d++) {
      FOLD_TRY(launch_cell_fwd_simt(m->cell, lo[d], lo[d + 1], s->gather, S, L.ld, m->U, m->b, (float *)H, C,
                                    (float *)Gact, L.ld_g, nl, st));
    }
  } else if (D >= 2) {
    // FP32 (3xTF32) / TF32: per level gather -> tcgen05 GEMM -> pointwise
    // append; Z lands in the level's saved-gate rows (gate blocks at g*ld: the forward U copy
    // has gate-padded rows) and the pointwise step turns it into the gates in place
    float *Uf = (float *)ws;
    {
      ProfScope ps(K_PREP, st);
      FOLD_TRY(launch_prep_U_tf(gates, S, L.ld, m->U, Uf, nullptr, st));
    }
    float *Acat = (float *)(a + L.al_off);
    const int64_t lda = tf_ld_a(S);
    const int npass = npass_of(m->prec);
    ProfScope ps(K_CELL_FWD, st);  // one bracket around the level sweep (fewer events in the step)
    for (int d = 2; d <= D; d++) {
      const int r0 = lo[d], r1 = lo[d + 1], M = r1 - r0, c0 = r0 - nl;
      if (M <= 0) continue;
      FOLD_TRY(launch_gather_cat(r0, r1, nl, S, L.ld, s->gather, (const float *)H, Acat, lda, st));
      FOLD_TRY(gemm_tf32(TfOperand{Acat + (int64_t)c0 * lda, lda, 0}, TfOperand{Uf, tf_ld_u(S), 0}, M, gates * L.ld,
                         2 * S, (float *)Gact + (int64_t)c0 * L.ld_g, L.ld_g, 0, npass, nullptr, 0, st));
      FOLD_TRY(launch_cell_fwd_pw(m->cell, r0, r1, nl, S, L.ld, L.ld_g, s->gather, m->b, (float *)H, C,
                                  (float *)Gact, st));
    }
  }
  ProfScope ps(K_ROOT, st);
  FOLD_TRY(launch_root_out(bf16, G, S, L.ld, nl, s->root_row, H, C, h_root, c_root, bf16 ? &sc : nullptr, st));
  return FOLD_OK;
}

size_t fold_backward_workspace(const fold_schedule_t *s, const fold_model *m) {
  if (check_sched(s) != FOLD_OK || check_model(m) != FOLD_OK) return 0;
  return bwd_layout(nullptr, s, m).bytes;
}

// Reverse level sweep: for d = D..2 pull-reduce the consumers' edge
// gradients, form dz, and produce this level's edge gradients dA = dz U; then the
// embedding gradient at depth 1 and one weight-gradient GEMM over all cells.
fold_status fold_backward(const fold_schedule_t *s, const fold_model *m, const void *acts, const float *dh_root,
                          const float *dc_root, fold_grads *grads, void *ws, size_t ws_bytes, void *stream) {
  FOLD_TRY(check_sched(s));
  FOLD_TRY(check_model(m));
  if (!grads || !grads->dU || !grads->db || !grads->dE) return FOLD_E_INVALID;
  // vectorised stores / read-modify-writes: gradient arrays must be 16-byte aligned
  if (((uintptr_t)grads->dU | (uintptr_t)grads->db | (uintptr_t)grads->dE) & 15) return FOLD_E_INVALID;
  if (s->n_graphs > 0 && !dh_root) return FOLD_E_INVALID;
  BwdWs b = bwd_layout(ws, s, m);
  if (!ws || ws_bytes < b.bytes) return FOLD_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = s->n_nodes, S = m->S, D = s->n_levels, nl = s->n_leaves, G = s->n_graphs, nc = s->n_cells;
  const int gates = gates_of(m->cell);
  const bool bf16 = m->prec == FOLD_PREC_BF16;
  const int acc = grads->accumulate ? 1 : 0;
  if (!acc) FOLD_TRY(launch_zero(grads->dE, (size_t)m->vocab * S * 4, st));
  if (N > 0) FOLD_TRY(launch_root_off(N, G, s->root_row, s->root_perm, b.root_off, st));
  if (N == 0 || nc == 0) {
    if (!acc) {
      FOLD_TRY(launch_zero(grads->dU, (size_t)gates * S * 2 * S * 4, st));
      FOLD_TRY(launch_zero(grads->db, (size_t)gates * S * 4, st));
    }
    if (N > 0)
      FOLD_TRY(launch_embed_bwd(S, nl, s->n_tok_segs, s->tok_seg, s->leaf_perm, s->leaf_token, s->cons_off,
                                s->cons_edge, b.root_off, s->root_perm, G, dh_root, b.dA, grads->dE, st));
    return FOLD_OK;
  }
  if (!acts) return FOLD_E_INVALID;
  ActsLayout L = acts_layout(s, m);
  const char *a = (const char *)acts;
  const void *H = a + L.h_off;
  const float *C = (const float *)(a + L.c_off);
  const void *Gact = a + L.g_off;
  const int32_t *lo = s->level_off_host;
  if (bf16) {
    ProfScope ps(K_PREP, st);
    FOLD_TRY(tc_prepare_U(gates, S, m->U, b.Ub, st));
  } else if (b.Utf) {
    ProfScope ps(K_PREP, st);
    FOLD_TRY(launch_prep_U_tf(gates, S, L.ld, m->U, nullptr, b.Utf, st));
  }
  const bool fused_tree = bf16 && s->tree_like && (S & 1) == 0;  // (leaf dA in bf16 on this path)
  if (fused_tree) {
    // tree-like: roots' seeded pointwise step, then every level's dA GEMM with the
    // children's pointwise step fused into its epilogue (one persistent launch)
    TcBwdArgs ba{};
    ba.level_off = s->level_off; ba.level_off_host = lo;
    ba.D = D; ba.S = S; ba.nl = nl; ba.n_cells = nc; ba.ld = L.ld; ba.ld_g = L.ld_g; ba.ld_z = b.ld_z;
    ba.gather = s->gather; ba.Ub = b.Ub; ba.U = m->U; ba.Ut = b.Ut; ba.Gact = (const __nv_bfloat16 *)Gact; ba.C = C;
    ba.dA = b.dA; ba.dCe = b.dCe; ba.dZ = (__nv_bfloat16 *)b.dZ; ba.rt_cnt = b.rt_cnt; ba.tstart = b.tstart;
    ba.ks_ring = b.ks_ring; ba.ks_cnt = b.ks_cnt; ba.lvl_tab = b.lvl_tab;
    {
      ProfScope ps(K_BWD_PW, st);
      FOLD_TRY(launch_cell_bwd_pw(bf16, m->cell, 0, G, nl, S, L.ld, L.ld_g, s->cons_off, s->cons_edge, b.root_off,
                                  s->root_perm, G, dh_root, dc_root, s->gather, Gact, C, b.dA, b.dCe, b.dZ, b.ld_z,
                                  st, s->root_row));
      FOLD_TRY(tc_bwd_prelude(ba, s->cons_off, st));
    }
    ProfScope ps(K_GEMM_DA, st);
    FOLD_TRY(tc_bwd_levels(m->cell, ba, st));
  } else {
  ProfScope ps(K_GEMM_DA, st);  // the backward level sweep (pointwise + dA GEMM per level), one bracket
  for (int d = D; d >= 2; d--) {
    const int r0 = lo[d], r1 = lo[d + 1], M = r1 - r0, c0 = r0 - nl;
    if (M <= 0) continue;
    FOLD_TRY(launch_cell_bwd_pw(bf16, m->cell, r0, r1, nl, S, L.ld, L.ld_g, s->cons_off, s->cons_edge, b.root_off,
                                s->root_perm, G, dh_root, dc_root, s->gather, Gact, C, b.dA, b.dCe, b.dZ, b.ld_z, st));
    float *dA_lvl = b.dA + (size_t)2 * c0 * S;
    if (bf16)
      FOLD_TRY(tc_gemm_dA(c0, M, nc, S, gates, (const __nv_bfloat16 *)b.dZ, b.ld_z, b.Ub, b.dA, st));
    else if (b.Utf)  // dA = dZ U: A = the level's dZ rows (K-major), B = U [gates*S][2S] (MN-major)
      FOLD_TRY(gemm_tf32(TfOperand{(const float *)b.dZ + (int64_t)c0 * b.ld_z, b.ld_z, 0},
                         TfOperand{b.Utf, tf_ld_u(S), 1}, M, 2 * S, gates * S, dA_lvl, 2 * S, 0,
                         npass_of(m->prec), nullptr, 0, st));
    else
      FOLD_TRY(launch_gemm_dA_simt(M, S, gates, (const float *)b.dZ + (size_t)c0 * b.ld_z, b.ld_z, m->U, dA_lvl, st));
  }
  }
  // The embedding gradient and db only need dA / dZ, the weight-gradient GEMM only dZ and
  // the A planes: run the two memory-bound reductions on an auxiliary stream beside the
  // tensor-bound dU GEMM, then join.
  if (grads->sweep_done_event) FOLD_CUDA_TRY(cudaEventRecord((cudaEvent_t)grads->sweep_done_event, st));
  // FOLD_AUX_ORDER (experiments): 0 = reductions on the aux stream launched before the
  // GEMM (default), 1 = after it, 2 = everything serial on the caller's stream
  static const int aux_order = [] { const char *e = getenv("FOLD_AUX_ORDER"); return e ? atoi(e) : 0; }();
  static AuxStream serial;  // ok == false: everything on the caller's stream
  AuxStream &ax = aux_order == 2 ? serial : aux_stream();
  cudaStream_t s2 = ax.ok ? ax.s : st;
  if (ax.ok) {
    FOLD_CUDA_TRY(cudaEventRecord(ax.fork, st));
    FOLD_CUDA_TRY(cudaStreamWaitEvent(s2, ax.fork, 0));
  }
  auto run_du = [&]() -> fold_status {
    ProfScope ps(K_GEMM_DU, st);
    if (bf16)
      FOLD_TRY(tc_gemm_dU(nc, S, gates, (const __nv_bfloat16 *)b.dZ, b.ld_z,
                          ScatterA{s->cons_off, s->cons_edge, (__nv_bfloat16 *)(a + L.al_off),
                                   (__nv_bfloat16 *)(a + L.ar_off), L.ld},
                          grads->dU, acc, b.dU_split, grads->db, b.partial, st));  // (+ db, fused)
    else if (b.Utf)  // dU = dZ^T Acat: both operands MN-major (cells are the reduction)
      FOLD_TRY(gemm_tf32(TfOperand{(const float *)b.dZ, b.ld_z, 1},
                         TfOperand{(const float *)(a + L.al_off), tf_ld_a(S), 1}, gates * S, 2 * S, nc, grads->dU,
                         2 * S, acc, npass_of(m->prec), b.dU_split, b.tf_split_floats, st));
    else
      FOLD_TRY(launch_gemm_dU_simt(nc, nl, S, gates, (const float *)b.dZ, b.ld_z, s->gather, (const float *)H, L.ld,
                                   grads->dU, acc, st));
    return FOLD_OK;
  };
  if (aux_order == 1) FOLD_TRY(run_du());
  {
    ProfScope ps(K_EMBED_BWD, s2);
    FOLD_TRY(launch_embed_bwd_pieces(S, nl, s->n_tok_segs, s->tok_seg, s->leaf_perm, s->leaf_token, s->cons_off,
                                     s->cons_edge, b.root_off, s->root_perm, dh_root, b.dA, fused_tree, grads->dE,
                                     b.emb, s2));
  }
  if (!bf16) {  // (BF16: db is summed inside the dU GEMM from its dZ stage tiles)
    ProfScope ps(K_COLSUM, s2);
    FOLD_TRY(launch_colsum(bf16, nc, gates * S, b.dZ, b.ld_z, b.partial, b.nsplit, grads->db, acc, s2));
  }
  if (aux_order != 1) FOLD_TRY(run_du());
  if (ax.ok) {
    FOLD_CUDA_TRY(cudaEventRecord(ax.join, s2));
    FOLD_CUDA_TRY(cudaStreamWaitEvent(st, ax.join, 0));
  }
  return FOLD_OK;
}

fold_status fold_sgd_update(float *p, const float *g, int64_t n, float lr, void *stream) {
  if (n < 0 || (n > 0 && (!p || !g))) return FOLD_E_INVALID;
  ProfScope ps(K_SGD, (cudaStream_t)stream);
  return launch_sgd(p, g, n, lr, (cudaStream_t)stream);
}

fold_status fold_touched_rows(const fold_schedule_t *s, int32_t *d_rows, void *stream) {
  if (!s || (s->n_tok_segs > 0 && (!d_rows || !s->tok_seg || !s->leaf_perm || !s->leaf_token))) return FOLD_E_INVALID;
  return launch_touched_rows(s->n_tok_segs, s->tok_seg, s->leaf_perm, s->leaf_token, d_rows, (cudaStream_t)stream);
}
fold_status fold_gather_rows(const float *d_src, int64_t ld, const int32_t *d_rows, int32_t n, int32_t S,
                             float *d_dst, void *stream) {
  if (n < 0 || S < 0 || ld < S || (n > 0 && (!d_src || !d_rows || !d_dst))) return FOLD_E_INVALID;
  return launch_gather_rows(d_src, ld, d_rows, n, S, d_dst, (cudaStream_t)stream);
}
fold_status fold_scatter_add_rows(const float *d_src, const int32_t *d_rows, int32_t n, int32_t S, float *d_dst,
                                  int64_t ld, void *stream) {
  if (n < 0 || S < 0 || ld < S || (n > 0 && (!d_src || !d_rows || !d_dst))) return FOLD_E_INVALID;
  return launch_scatter_add_rows(d_src, d_rows, n, S, d_dst, ld, (cudaStream_t)stream);
}

const char *fold_status_string(fold_status s) {
  switch (s) {
    case FOLD_OK: return "FOLD_OK";
    case FOLD_E_INVALID: return "FOLD_E_INVALID";
    case FOLD_E_CHILD_RANGE: return "FOLD_E_CHILD_RANGE";
    case FOLD_E_ARITY: return "FOLD_E_ARITY";
    case FOLD_E_TOKEN_RANGE: return "FOLD_E_TOKEN_RANGE";
    case FOLD_E_ROOT_RANGE: return "FOLD_E_ROOT_RANGE";
    case FOLD_E_CYCLE: return "FOLD_E_CYCLE";
    case FOLD_E_WORKSPACE: return "FOLD_E_WORKSPACE";
    case FOLD_E_CUDA: return "FOLD_E_CUDA";
    case FOLD_E_MISMATCH: return "FOLD_E_MISMATCH";
    case FOLD_E_OP_RANGE: return "FOLD_E_OP_RANGE";
    case FOLD_E_UNSUPPORTED: return "FOLD_E_UNSUPPORTED";
    case FOLD_E_LEVEL: return "FOLD_E_LEVEL";
  }
  if ((int)s == FOLD_E_TYPE) return "FOLD_E_TYPE";
  return "FOLD_E_UNKNOWN";
}

int32_t fold_last_error_detail(void) { return g_last_detail; }
fold_status fold_last_error_context(int32_t *node, int32_t *depth, int32_t *op) {
  if (node) *node = g_last_ctx[0];
  if (depth) *depth = g_last_ctx[1];
  if (op) *op = g_last_ctx[2];
  return g_last_ctx[0] >= 0 ? FOLD_OK : FOLD_E_INVALID;
}
int32_t fold_abi_version(void) { return FOLD_ABI_VERSION; }

int32_t fold_set_reserved_sms(int32_t n) { return set_reserved_sms(n); }

// ----------------------------------------------------------------- multi-op (fold_mo.h)
size_t fold_mo_schedule_workspace(const fold_mo_table *table, int32_t n_nodes, int32_t n_graphs) {
  return fold::mo_schedule_workspace(table, n_nodes, n_graphs);
}
fold_status fold_mo_schedule(const fold_mo_table *table, const fold_mo_graphs *graphs, fold_mo_schedule_t *sched,
                             void *ws, size_t ws_bytes, void *stream) {
  fold::ProfScope ps(fold::K_SCHED, (cudaStream_t)stream);
  return fold::run_mo_schedule(table, graphs, sched, ws, ws_bytes, (cudaStream_t)stream);
}
size_t fold_mo_acts_bytes(const fold_mo_table *table, const fold_mo_schedule_t *sched) {
  return fold::mo_acts_bytes(table, sched);
}
size_t fold_mo_forward_workspace(const fold_mo_table *table, const fold_mo_schedule_t *sched) {
  return fold::mo_forward_workspace(table, sched);
}
fold_status fold_mo_forward(const fold_mo_table *table, const fold_mo_schedule_t *sched, const fold_mo_model *model,
                            void *acts, float *h_root, void *ws, size_t ws_bytes, void *stream) {
  fold::ProfScope ps(fold::K_CELL_FWD, (cudaStream_t)stream);
  return fold::mo_forward(table, sched, model, acts, h_root, ws, ws_bytes, (cudaStream_t)stream);
}
size_t fold_mo_backward_workspace(const fold_mo_table *table, const fold_mo_schedule_t *sched) {
  return fold::mo_backward_workspace(table, sched);
}
fold_status fold_mo_backward(const fold_mo_table *table, const fold_mo_schedule_t *sched, const fold_mo_model *model,
                             const void *acts, const float *dh_root, fold_mo_grads *grads, void *ws, size_t ws_bytes,
                             void *stream) {
  fold::ProfScope ps(fold::K_GEMM_DA, (cudaStream_t)stream);
  return fold::mo_backward(table, sched, model, acts, dh_root, grads, ws, ws_bytes, (cudaStream_t)stream);
}

/* instrumentation: per-phase timeline of the last FOLD_DBG_SCHED=1 schedule (block 0) */
int32_t fold_debug_sched_trace(unsigned long long *host) { return fold::debug_sched_trace(host); }

/* instrumentation: per-tile forward timeline of the last FOLD_DBG_FWD=1 run */
int32_t fold_debug_fwd_trace(unsigned long long *host, int32_t n_tiles) {
  return fold::tc_debug_fwd_trace(host, n_tiles);
}

/* instrumentation: per-tile timeline of the wide backward kernel in the last FOLD_DBG_BWD=1 run */
int32_t fold_debug_bwd_trace(unsigned long long *host, int32_t n_tiles) {
  return fold::tc_debug_bwd_trace(host, n_tiles);
}

/* instrumentation / tests: one k_gemm_tf32 GEMM (the FP32 / TF32 modes' contraction) */
fold_status fold_debug_gemm_tf32(const float *A, int64_t lda, int32_t a_mn, const float *B, int64_t ldb,
                                 int32_t b_mn, int32_t M, int32_t N, int32_t K, float *C, int64_t ldc,
                                 int32_t accumulate, int32_t npass, float *ws, int64_t ws_floats, void *stream) {
  if (M < 0 || N < 0 || K < 0 || !A || !B || !C) return FOLD_E_INVALID;
  return fold::gemm_tf32(fold::TfOperand{A, lda, a_mn}, fold::TfOperand{B, ldb, b_mn}, M, N, K, C, ldc, accumulate,
                         npass, ws, ws_floats, (cudaStream_t)stream);
}
int64_t fold_debug_gemm_tf32_ws(int32_t M, int32_t N, int32_t K) { return fold::gemm_tf32_split_floats(M, N, K); }

fold_status fold_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FOLD_E_CUDA;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return FOLD_E_CUDA;
  if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return FOLD_E_CUDA;
  return (major == 10 && minor == 0) ? FOLD_OK : FOLD_E_UNSUPPORTED;
}

int64_t fold_launch_count(int32_t reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

}  // extern "C"


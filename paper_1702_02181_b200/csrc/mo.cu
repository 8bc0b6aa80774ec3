// mo.cu — multi-op level executor (fold_mo.h): several operations and
// tensor types per depth, §2 in full generality.
//
// Layout (reading R30 / DESIGN.md §13):
//   * per tensor type t a pool H_t, C_t [n_t][ld_t] fp32 whose rows are the L43 concatenation
//     (depth, op enumeration, id) of every node of output type t (pool_row from the schedule);
//   * per operation o an op-major SLAB: its nodes in (depth, id) order, one row each: A_o
//     (the gathered inputs [h_1 | .. | h_a], the "gather" of L30 materialised as the dense GEMM
//     operand and kept for the weight gradient) and Z_o (pre-activations, then the saved gate
//     activations). Group (d, o) of L42 is the contiguous slab range [sstart, sstart + cnt).
// Forward, per depth d (L47: "each iteration of the loop will evaluate all of the operations
// at a particular depth"): ONE gather launch over every group of the level, ONE grouped
// tcgen05 TF32 / 3xTF32 GEMM launch (every op's tiles, gemm_tf32.cu), ONE pointwise launch.
// Backward, per depth D..1: ONE pull-reduction + pointwise launch (each node sums its consumer
// edges' dA / dCe rows in ascending edge order and its root seeds: deterministic, no float
// atomics), ONE grouped dA GEMM; then one grouped weight-gradient GEMM over every op's whole
// slab, fixed-order bias sums and the (op, token)-segmented embedding reduction.
#include <cstring>
#include <vector>

#include "../../include/fold_mo.h"
#include "exec.cuh"

namespace fold {

bool mo_table_ok(const fold_mo_table *t);

namespace {

constexpr int kMoGroups = FOLD_MO_MAX_OPS;  // groups per level: at most one per op

inline int ld4(int64_t x) { return (int)round_up(x, 4); }

struct MoDims {  // host-side shapes of one (table, schedule)
  int K, T, N, G, D, Smax;
  int S[FOLD_MO_MAX_TYPES], ldS[FOLD_MO_MAX_TYPES];
  int64_t ntype[FOLD_MO_MAX_TYPES];
  int kin[FOLD_MO_MAX_OPS], nout[FOLD_MO_MAX_OPS], ldK[FOLD_MO_MAX_OPS], ldN[FOLD_MO_MAX_OPS];
  int64_t rows[FOLD_MO_MAX_OPS];
  // acts offsets (floats)
  int64_t h_off[FOLD_MO_MAX_TYPES], c_off[FOLD_MO_MAX_TYPES], a_off[FOLD_MO_MAX_OPS], z_off[FOLD_MO_MAX_OPS];
  int64_t acts_floats;
};

bool is_cell(const fold_mo_table *t, int o) { return t->kind[o] != FOLD_MO_EMBED; }

MoDims mo_dims(const fold_mo_table *t, const fold_mo_schedule_t *s) {
  MoDims m{};
  m.K = t->n_ops; m.T = t->n_types; m.N = s->n_nodes; m.G = s->n_graphs; m.D = s->n_levels;
  for (int i = 0; i < m.T; i++) { m.S[i] = t->S[i]; m.ldS[i] = ld4(t->S[i]); m.Smax = std::max(m.Smax, t->S[i]); }
  for (int o = 0; o < m.K; o++) {
    int64_t r = 0;
    for (int d = 0; d <= m.D; d++) r += s->group_off_host[d * m.K + o + 1] - s->group_off_host[d * m.K + o];
    m.rows[o] = r;
    m.ntype[t->out_type[o]] += r;
    const int So = t->S[t->out_type[o]];
    if (is_cell(t, o)) {
      m.kin[o] = t->arity[o] * t->S[t->in_type[o]];
      m.nout[o] = t->kind[o] == FOLD_MO_LSTM ? (3 + t->arity[o]) * So : So;
      m.ldK[o] = ld4(m.kin[o]);
      m.ldN[o] = ld4(m.nout[o]);
    }
  }
  int64_t off = 0;
  for (int i = 0; i < m.T; i++) {
    m.h_off[i] = off; off += round_up(m.ntype[i] * m.ldS[i], 64);
    m.c_off[i] = off; off += round_up(m.ntype[i] * m.ldS[i], 64);
  }
  for (int o = 0; o < m.K; o++) {
    if (!is_cell(t, o)) continue;
    m.a_off[o] = off; off += round_up(m.rows[o] * m.ldK[o], 64);
    m.z_off[o] = off; off += round_up(m.rows[o] * m.ldN[o], 64);
  }
  m.acts_floats = off;
  return m;
}

// per-level group descriptors (kernel parameters)
struct MoLevel {
  int n;
  int op[kMoGroups], gstart[kMoGroups], sstart[kMoGroups], cnt[kMoGroups], row0[kMoGroups];
  int64_t rows_total;
};

MoLevel level_groups(const fold_mo_table *t, const fold_mo_schedule_t *s, const int64_t *sstart_op, int d,
                     std::vector<int64_t> &sacc) {
  MoLevel L{};
  const int K = t->n_ops;
  for (int o = 0; o < K; o++) {
    const int c = s->group_off_host[d * K + o + 1] - s->group_off_host[d * K + o];
    if (c <= 0) continue;
    L.op[L.n] = o;
    L.gstart[L.n] = s->group_off_host[d * K + o];
    L.sstart[L.n] = (int)(sstart_op ? sstart_op[o] + sacc[o] : sacc[o]);
    L.cnt[L.n] = c;
    L.row0[L.n] = (int)L.rows_total;
    L.rows_total += c;
    L.n++;
    sacc[o] += c;
  }
  return L;
}

// Kernel-side view of the model / acts (by value)
struct MoView {
  int K, N, Smax;
  int kind[FOLD_MO_MAX_OPS], arity[FOLD_MO_MAX_OPS], in_t[FOLD_MO_MAX_OPS], out_t[FOLD_MO_MAX_OPS];
  int S[FOLD_MO_MAX_TYPES], ldS[FOLD_MO_MAX_TYPES];
  int kin[FOLD_MO_MAX_OPS], nout[FOLD_MO_MAX_OPS], ldK[FOLD_MO_MAX_OPS], ldN[FOLD_MO_MAX_OPS];
  float *H[FOLD_MO_MAX_TYPES], *C[FOLD_MO_MAX_TYPES];
  float *A[FOLD_MO_MAX_OPS], *Z[FOLD_MO_MAX_OPS];
  const float *b[FOLD_MO_MAX_OPS], *E[FOLD_MO_MAX_OPS];
  const int32_t *op, *child, *token, *order, *pool_row, *type_off;
  // push-gather (forward): a node's h goes straight into the A slab rows of its consumers
  const int32_t *cons_off, *cons_edge, *slab_of_pos;
};

// h of node n (type t, global pool index gp) at state column j -> the A rows of every
// consumer edge e = 2 p + k (consumer at order position p, input slot k): the gather of
// PAPER.md L30 / L47 performed by the producer (as in the BF16 path), so no gather launch
__device__ __forceinline__ void push_h(const MoView &v, int gp, int S, int j, float h) {
  for (int e = v.cons_off[gp]; e < v.cons_off[gp + 1]; e++) {
    const int ed = v.cons_edge[e], pm = ed >> 1, k = ed & 1;
    const int om = v.op[v.order[pm]];
    v.A[om][(int64_t)v.slab_of_pos[pm] * v.ldK[om] + k * S + j] = h;
  }
}

// find the group of a level-row index (rows of the level's groups concatenated)
__device__ __forceinline__ int grp_of(const MoLevel &L, int64_t r) {
  int g = 0;
  while (g + 1 < L.n && r >= L.row0[g + 1]) g++;
  return g;
}

// ---------------------------------------------------------------- forward kernels
// depth 1: EMBED groups, h = E_o[token], c = 0 (Fig. 1 "embed lookup")
__global__ void k_mo_embed(MoView v, MoLevel L) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = L.rows_total * v.Smax;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / v.Smax;
    const int col = (int)(i % v.Smax);
    const int g = grp_of(L, r), o = L.op[g];
    const int t = v.out_t[o], S = v.S[t];
    if (col >= S) continue;
    const int n = v.order[L.gstart[g] + (r - L.row0[g])];
    const int64_t row = v.pool_row[n];
    const float h = v.E[o][(int64_t)v.token[n] * S + col];
    v.H[t][row * v.ldS[t] + col] = h;
    v.C[t][row * v.ldS[t] + col] = 0.f;
    push_h(v, v.type_off[t] + (int)row, S, col, h);
  }
}

// cell pointwise step on Z = A U^T (the grouped GEMM's output): LSTM gates (i, f_1..f_a, o, u)
// -> c = i u + sum_k f_k c_k, h = o tanh(c); RNN h = tanh(z + b). The activations replace the
// pre-activations in Z (the backward's saved gates).
__global__ void k_mo_cell_fwd(MoView v, MoLevel L) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = L.rows_total * v.Smax;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / v.Smax;
    const int j = (int)(i % v.Smax);
    const int g = grp_of(L, r), o = L.op[g];
    const int t = v.out_t[o], S = v.S[t];
    if (j >= S) continue;
    const int64_t jr = r - L.row0[g];
    const int n = v.order[L.gstart[g] + jr];
    float *z = v.Z[o] + (L.sstart[g] + jr) * v.ldN[o];
    const float *b = v.b[o];
    const int64_t row = v.pool_row[n];
    if (v.kind[o] == FOLD_MO_RNN) {
      const float h = tanhf(z[j] + b[j]);
      z[j] = h;
      v.H[t][row * v.ldS[t] + j] = h;
      v.C[t][row * v.ldS[t] + j] = 0.f;
      push_h(v, v.type_off[t] + (int)row, S, j, h);
      continue;
    }
    const int a = v.arity[o];
    const float ig = 1.f / (1.f + expf(-(z[j] + b[j])));
    const float og = 1.f / (1.f + expf(-(z[(1 + a) * S + j] + b[(1 + a) * S + j])));
    const float ug = tanhf(z[(2 + a) * S + j] + b[(2 + a) * S + j]);
    float cc = ig * ug;
    for (int k = 0; k < a; k++) {
      const float f = 1.f / (1.f + expf(-(z[(1 + k) * S + j] + b[(1 + k) * S + j])));
      const int ch = v.child[2 * n + k];
      cc += f * v.C[t][(int64_t)v.pool_row[ch] * v.ldS[t] + j];
      z[(1 + k) * S + j] = f;
    }
    z[j] = ig; z[(1 + a) * S + j] = og; z[(2 + a) * S + j] = ug;
    v.C[t][row * v.ldS[t] + j] = cc;
    const float h = og * tanhf(cc);
    v.H[t][row * v.ldS[t] + j] = h;
    push_h(v, v.type_off[t] + (int)row, S, j, h);
  }
}

// h_root[g][0..S_t) = H_t[pool row of root g], the rest 0
__global__ void k_mo_root_out(MoView v, const int32_t *root, int G, float *h_root) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)G * v.Smax; i += stride) {
    const int g = (int)(i / v.Smax), j = (int)(i % v.Smax);
    const int n = root[g], t = v.out_t[v.op[n]];
    h_root[i] = j < v.S[t] ? v.H[t][(int64_t)v.pool_row[n] * v.ldS[t] + j] : 0.f;
  }
}

// U_o -> padded copy Up [nout][ldK] (16-byte rows for the tensor maps)
__global__ void k_mo_pad(const float *U, int rows, int cols, int ld, float *Up) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)rows * ld; i += stride) {
    const int64_t r = i / ld;
    const int c = (int)(i % ld);
    Up[i] = c < cols ? U[r * cols + c] : 0.f;
  }
}

// ---------------------------------------------------------------- backward kernels
struct MoBwdView {
  float *dZ[FOLD_MO_MAX_OPS], *dA[FOLD_MO_MAX_OPS], *dCe[FOLD_MO_MAX_OPS];
  const int32_t *cons_off, *cons_edge, *root_off, *root_graph;
  const int32_t *slab_of_pos;  // order position -> slab row within its op
  const float *dh_root;
  float *dh_leaf;  // [n_leaves][Smax]: leaves' dh (order position - l0)
  int l0;
};

// the node's (dh, dc) pulled from its consumers in ascending edge order, then root seeds;
// then its pointwise backward step:
//   EMBED: dh -> dh_leaf (the embedding gradient's input)
//   RNN:   dz = dh (1 - h^2)
//   LSTM:  tc = tanh(c), dc' = dc + dh o (1 - tc^2), dz_i = dc' u i(1-i),
//          dz_fk = dc' c_k f_k(1-f_k), dz_o = dh tc o(1-o), dz_u = dc' i (1-u^2),
//          dCe[own slab row][k] = dc' f_k (what child k pulls as its dc)
__global__ void k_mo_cell_bwd(MoView v, MoBwdView w, MoLevel L) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = L.rows_total * v.Smax;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / v.Smax;
    const int j = (int)(i % v.Smax);
    const int g = grp_of(L, r), o = L.op[g];
    const int t = v.out_t[o], S = v.S[t];
    if (j >= S) continue;
    const int64_t jr = r - L.row0[g];
    const int p = L.gstart[g] + (int)jr;
    const int n = v.order[p];
    const int gp = v.type_off[t] + v.pool_row[n];
    float dh = 0.f, dc = 0.f;
    for (int e = w.cons_off[gp]; e < w.cons_off[gp + 1]; e++) {
      const int ed = w.cons_edge[e], pm = ed >> 1, k = ed & 1;
      const int om = v.op[v.order[pm]];
      const int64_t srow = w.slab_of_pos[pm];
      dh += w.dA[om][srow * v.ldK[om] + k * S + j];
      if (v.kind[om] == FOLD_MO_LSTM) dc += w.dCe[om][srow * v.ldK[om] + k * S + j];
    }
    for (int q = w.root_off[gp]; q < w.root_off[gp + 1]; q++) dh += w.dh_root[(int64_t)w.root_graph[q] * v.Smax + j];
    if (v.kind[o] == FOLD_MO_EMBED) {
      w.dh_leaf[(int64_t)(p - w.l0) * v.Smax + j] = dh;
      continue;
    }
    const int64_t srow = L.sstart[g] + jr;
    const float *z = v.Z[o] + srow * v.ldN[o];
    float *dz = w.dZ[o] + srow * v.ldN[o];
    if (v.kind[o] == FOLD_MO_RNN) {
      dz[j] = dh * (1.f - z[j] * z[j]);
      continue;
    }
    const int a = v.arity[o];
    const float ig = z[j], og = z[(1 + a) * S + j], ug = z[(2 + a) * S + j];
    const float tc = tanhf(v.C[t][(int64_t)v.pool_row[n] * v.ldS[t] + j]);
    const float dcc = dc + dh * og * (1.f - tc * tc);
    dz[j] = dcc * ug * ig * (1.f - ig);
    for (int k = 0; k < a; k++) {
      const float f = z[(1 + k) * S + j];
      const float ck = v.C[t][(int64_t)v.pool_row[v.child[2 * n + k]] * v.ldS[t] + j];
      dz[(1 + k) * S + j] = dcc * ck * f * (1.f - f);
      w.dCe[o][srow * v.ldK[o] + k * S + j] = dcc * f;
    }
    dz[(1 + a) * S + j] = dh * tc * og * (1.f - og);
    dz[(2 + a) * S + j] = dcc * ig * (1.f - ug * ug);
  }
}

// order position -> slab row within its op (sstart of its (depth, op) group + offset)
__global__ void k_mo_slab_index(int N, int K, int ngroups, const int32_t *group_off, const int64_t *gsstart,
                                int32_t *slab_of_pos) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N; p += stride) {
    int lo = 0, hi = ngroups;  // last key with group_off[key] <= p among non-empty keys
    while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (group_off[mid] <= p) lo = mid; else hi = mid; }
    slab_of_pos[p] = (int32_t)(gsstart[lo] + (p - group_off[lo]));
  }
}

// dE_o[token] = sum over the (op, token) segment of the leaves' dh (every row of dE_o first
// zeroed unless accumulating). One block per (segment, 32-column chunk): warp w sums the
// segment's leaves w, w + 8, w + 16, ... in order (lane = column), then warp 0 adds the eight
// partials in warp order — a fixed order (deterministic), and a Zipf-heavy token's thousands of
// leaves no longer run on one thread.
__global__ void __launch_bounds__(256) k_mo_embed_bwd(MoView v, const int32_t *leaf_seg, const int32_t *leaf_order,
                                                      int l0, const float *dh_leaf, float *const *dE) {
  __shared__ float part[8][33];
  const int sg = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.y * 32 + lane;
  const int q0 = leaf_seg[sg], q1 = leaf_seg[sg + 1];
  const int n0 = v.order[leaf_order[q0]], o = v.op[n0];
  const int S = v.S[v.out_t[o]];
  if ((int)blockIdx.y * 32 >= S || !dE[o]) return;  // (uniform over the block)
  float acc = 0.f;
  if (j < S)
    for (int q = q0 + warp; q < q1; q += 8) acc += dh_leaf[(int64_t)(leaf_order[q] - l0) * v.Smax + j];
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && j < S) {
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; w++) tot += part[w][lane];
    dE[o][(int64_t)v.token[n0] * S + j] += tot;
  }
}

unsigned blocks_for(int64_t n) {
  int64_t b = cdiv(n, 256);
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)b;
}

MoView make_view(const fold_mo_table *t, const fold_mo_schedule_t *s, const MoDims &m, float *acts,
                 const fold_mo_model *model, const int32_t *op, const int32_t *child, const int32_t *token) {
  MoView v{};
  v.K = m.K; v.N = m.N; v.Smax = m.Smax;
  for (int o = 0; o < m.K; o++) {
    v.kind[o] = t->kind[o]; v.arity[o] = t->arity[o]; v.in_t[o] = t->in_type[o]; v.out_t[o] = t->out_type[o];
    v.kin[o] = m.kin[o]; v.nout[o] = m.nout[o]; v.ldK[o] = m.ldK[o]; v.ldN[o] = m.ldN[o];
    if (is_cell(t, o)) { v.A[o] = acts + m.a_off[o]; v.Z[o] = acts + m.z_off[o]; v.b[o] = model->b[o]; }
    else v.E[o] = model->E[o];
  }
  for (int i = 0; i < m.T; i++) {
    v.S[i] = m.S[i]; v.ldS[i] = m.ldS[i];
    v.H[i] = acts + m.h_off[i]; v.C[i] = acts + m.c_off[i];
  }
  v.op = op; v.child = child; v.token = token;
  v.order = s->order; v.pool_row = s->pool_row; v.type_off = s->type_off;
  return v;
}

// per-op slab start of each (depth, op) group: sstart[d][o] (host)
std::vector<int64_t> slab_starts(const fold_mo_schedule_t *s, int K, int D) {
  std::vector<int64_t> ss((size_t)(D + 1) * K, 0), acc(K, 0);
  for (int d = 0; d <= D; d++)
    for (int o = 0; o < K; o++) {
      ss[(size_t)d * K + o] = acc[o];
      acc[o] += s->group_off_host[d * K + o + 1] - s->group_off_host[d * K + o];
    }
  return ss;
}

// workspace layouts (bytes, 256-aligned)
struct MoFwdWs {
  float *Up[FOLD_MO_MAX_OPS];
  float *split;
  int64_t split_floats;
  int32_t *slab_of_pos;
  int64_t *gsstart;
  size_t bytes;
};
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

int64_t fwd_split_floats(const fold_mo_table *t, const MoDims &m, int npass) {
  // the largest level's problems bound every level's split partials (per-problem splits
  // depend on M, N, K only; M <= rows of the op)
  std::vector<TfProblem> q;
  for (int o = 0; o < m.K; o++) {
    if (!is_cell(t, o) || m.rows[o] == 0) continue;
    TfProblem p{};
    p.M = (int)m.rows[o]; p.N = m.nout[o]; p.K = m.kin[o];
    q.push_back(p);
  }
  return q.empty() ? 0 : gemm_tf32_grouped_ws_floats(q.data(), (int)q.size(), npass) + 64;
}

MoFwdWs fwd_ws(const fold_mo_table *t, const MoDims &m, int npass, void *base) {
  MoFwdWs w{};
  size_t off = 0;
  char *b = (char *)base;
  for (int o = 0; o < m.K; o++) {
    if (!is_cell(t, o)) continue;
    const size_t n = (size_t)m.nout[o] * m.ldK[o] * 4;
    if (b) w.Up[o] = (float *)(b + off);
    off = a256(off + n);
  }
  w.split_floats = fwd_split_floats(t, m, npass);
  if (b) w.split = (float *)(b + off);
  off = a256(off + (size_t)w.split_floats * 4);
  if (b) w.slab_of_pos = (int32_t *)(b + off);
  off = a256(off + (size_t)(m.N + 1) * 4);
  if (b) w.gsstart = (int64_t *)(b + off);
  off = a256(off + (size_t)((m.D + 1) * m.K + 1) * 8);
  w.bytes = off;
  return w;
}

struct MoBwdWs {
  MoFwdWs f;
  float *dZ[FOLD_MO_MAX_OPS], *dA[FOLD_MO_MAX_OPS], *dCe[FOLD_MO_MAX_OPS];
  float *dh_leaf, *colsum, *dU_split;
  int64_t dU_split_floats;
  int32_t *slab_of_pos;
  int64_t *gsstart;
  float **dE_dev;
  size_t bytes;
};

int colsum_splits(int64_t rows) {
  int64_t sp = rows / 512;
  return (int)(sp < 1 ? 1 : sp > 64 ? 64 : sp);
}

MoBwdWs bwd_ws(const fold_mo_table *t, const fold_mo_schedule_t *s, const MoDims &m, int npass, void *base) {
  MoBwdWs w{};
  w.f = fwd_ws(t, m, npass, base);
  size_t off = w.f.bytes;
  char *b = (char *)base;
  auto take = [&](size_t bytes) { size_t o = off; off = a256(off + bytes); return b ? (void *)(b + o) : nullptr; };
  std::vector<TfProblem> q;
  for (int o = 0; o < m.K; o++) {
    if (!is_cell(t, o)) continue;
    w.dZ[o] = (float *)take((size_t)m.rows[o] * m.ldN[o] * 4);
    w.dA[o] = (float *)take((size_t)m.rows[o] * m.ldK[o] * 4);
    w.dCe[o] = t->kind[o] == FOLD_MO_LSTM ? (float *)take((size_t)m.rows[o] * m.ldK[o] * 4) : nullptr;
    TfProblem p{};
    p.M = m.nout[o]; p.N = m.kin[o]; p.K = (int)m.rows[o];
    q.push_back(p);
  }
  const int64_t nl = s->group_off_host[2 * m.K] - s->group_off_host[m.K];
  w.dh_leaf = (float *)take((size_t)(nl + 1) * m.Smax * 4);
  int64_t cs = 0;
  for (int o = 0; o < m.K; o++)
    if (is_cell(t, o)) cs = std::max<int64_t>(cs, (int64_t)colsum_splits(m.rows[o]) * m.nout[o]);
  w.colsum = (float *)take((size_t)(cs + 1) * 4);
  w.dU_split_floats = q.empty() ? 0 : gemm_tf32_grouped_ws_floats(q.data(), (int)q.size(), npass);
  w.dU_split = (float *)take((size_t)(w.dU_split_floats + 1) * 4);
  w.slab_of_pos = (int32_t *)take((size_t)(m.N + 1) * 4);
  w.gsstart = (int64_t *)take((size_t)((m.D + 1) * m.K + 1) * 8);
  w.dE_dev = (float **)take(sizeof(float *) * FOLD_MO_MAX_OPS);
  w.bytes = off;
  return w;
}

fold_status check_common(const fold_mo_table *t, const fold_mo_schedule_t *s) {
  if (!mo_table_ok(t) || !s || !s->group_off_host) return FOLD_E_INVALID;
  if (s->n_nodes < 0 || s->n_levels < 0) return FOLD_E_INVALID;
  return FOLD_OK;
}

int npass_of(int prec) { return prec == FOLD_PREC_FP32 ? 3 : prec == FOLD_PREC_TF32 ? 1 : 0; }

}  // namespace

size_t mo_acts_bytes(const fold_mo_table *t, const fold_mo_schedule_t *s) {
  if (check_common(t, s) != FOLD_OK) return 0;
  return (size_t)mo_dims(t, s).acts_floats * 4;
}
// (split-K partial sizes depend on the pass count: the query covers both precisions)
size_t mo_forward_workspace(const fold_mo_table *t, const fold_mo_schedule_t *s) {
  if (check_common(t, s) != FOLD_OK) return 0;
  const MoDims m = mo_dims(t, s);
  return std::max(fwd_ws(t, m, 3, nullptr).bytes, fwd_ws(t, m, 1, nullptr).bytes);
}
size_t mo_backward_workspace(const fold_mo_table *t, const fold_mo_schedule_t *s) {
  if (check_common(t, s) != FOLD_OK) return 0;
  const MoDims m = mo_dims(t, s);
  return std::max(bwd_ws(t, s, m, 3, nullptr).bytes, bwd_ws(t, s, m, 1, nullptr).bytes);
}

static fold_status check_model(const fold_mo_table *t, const fold_mo_model *model) {
  if (!model) return FOLD_E_INVALID;
  if (model->prec == FOLD_PREC_BF16) return FOLD_E_UNSUPPORTED;
  if (!npass_of(model->prec)) return FOLD_E_INVALID;
  for (int o = 0; o < t->n_ops; o++) {
    if (is_cell(t, o)) {
      if (!model->U[o] || !model->b[o] || ((uintptr_t)model->U[o] & 15)) return FOLD_E_INVALID;
    } else if (!model->E[o]) {
      return FOLD_E_INVALID;
    }
  }
  return FOLD_OK;
}

fold_status mo_forward(const fold_mo_table *t, const fold_mo_schedule_t *s, const fold_mo_model *model, void *acts,
                       float *h_root, void *ws, size_t ws_bytes, cudaStream_t st) {
  const int32_t *op = s ? s->op : nullptr, *child = s ? s->child : nullptr, *token = s ? s->token : nullptr;
  const int32_t *root = s ? s->root : nullptr;
  FOLD_TRY(check_common(t, s));
  FOLD_TRY(check_model(t, model));
  if (s->n_nodes == 0) return FOLD_OK;
  if (!acts || !op || !child || !token) return FOLD_E_INVALID;
  const int npass = npass_of(model->prec);
  const MoDims m = mo_dims(t, s);
  MoFwdWs w = fwd_ws(t, m, npass, ws);
  if (!ws || ws_bytes < w.bytes) return FOLD_E_WORKSPACE;
  MoView v = make_view(t, s, m, (float *)acts, model, op, child, token);
  for (int o = 0; o < m.K; o++) {
    if (!is_cell(t, o)) continue;
    k_mo_pad<<<blocks_for((int64_t)m.nout[o] * m.ldK[o]), 256, 0, st>>>(model->U[o], m.nout[o], m.kin[o], m.ldK[o],
                                                                       w.Up[o]);
    FOLD_LAUNCH_CHECK();
  }
  {  // order position -> slab row, for the push-gather
    const std::vector<int64_t> ss = slab_starts(s, m.K, m.D);
    const int ngroups = (m.D + 1) * m.K;
    FOLD_CUDA_TRY(cudaMemcpyAsync(w.gsstart, ss.data(), (size_t)ngroups * 8, cudaMemcpyHostToDevice, st));
    k_mo_slab_index<<<blocks_for(m.N), 256, 0, st>>>(m.N, m.K, ngroups, s->group_off, w.gsstart, w.slab_of_pos);
    FOLD_LAUNCH_CHECK();
  }
  v.cons_off = s->cons_off; v.cons_edge = s->cons_edge; v.slab_of_pos = w.slab_of_pos;
  std::vector<int64_t> sacc(m.K, 0);
  for (int d = 1; d <= m.D; d++) {
    MoLevel L = level_groups(t, s, nullptr, d, sacc);
    if (L.n == 0) continue;
    if (d == 1) {  // only EMBED operations have depth 1
      k_mo_embed<<<blocks_for(L.rows_total * m.Smax), 256, 0, st>>>(v, L);
      FOLD_LAUNCH_CHECK();
      continue;
    }
    // (the level's A slab rows were filled by their producers' push-gather)
    TfProblem q[kMoGroups];
    for (int g = 0; g < L.n; g++) {
      const int o = L.op[g];
      q[g] = TfProblem{};
      q[g].A = TfOperand{v.A[o] + (int64_t)L.sstart[g] * m.ldK[o], m.ldK[o], 0};
      q[g].B = TfOperand{w.Up[o], m.ldK[o], 0};
      q[g].M = L.cnt[g]; q[g].N = m.nout[o]; q[g].K = m.kin[o];
      q[g].C = v.Z[o] + (int64_t)L.sstart[g] * m.ldN[o];
      q[g].ldc = m.ldN[o];
      q[g].accumulate = 0;
    }
    FOLD_TRY(gemm_tf32_grouped(q, L.n, npass, w.split, w.split_floats, st));
    k_mo_cell_fwd<<<blocks_for(L.rows_total * m.Smax), 256, 0, st>>>(v, L);
    FOLD_LAUNCH_CHECK();
  }
  if (h_root && m.G > 0) {
    if (!root) return FOLD_E_INVALID;
    k_mo_root_out<<<blocks_for((int64_t)m.G * m.Smax), 256, 0, st>>>(v, root, m.G, h_root);
    FOLD_LAUNCH_CHECK();
  }
  return FOLD_OK;
}

fold_status mo_backward(const fold_mo_table *t, const fold_mo_schedule_t *s, const fold_mo_model *model,
                        const void *acts, const float *dh_root, fold_mo_grads *gr, void *ws, size_t ws_bytes,
                        cudaStream_t st) {
  const int32_t *op = s ? s->op : nullptr, *child = s ? s->child : nullptr, *token = s ? s->token : nullptr;
  FOLD_TRY(check_common(t, s));
  FOLD_TRY(check_model(t, model));
  if (!gr) return FOLD_E_INVALID;
  const int npass = npass_of(model->prec);
  const MoDims m = mo_dims(t, s);
  // zero the gradients (or keep them: accumulate)
  if (!gr->accumulate) {
    for (int o = 0; o < m.K; o++) {
      const int So = m.S[t->out_type[o]];
      if (is_cell(t, o)) {
        if (gr->dU[o]) FOLD_TRY(launch_zero(gr->dU[o], (size_t)m.nout[o] * m.kin[o] * 4, st));
        if (gr->db[o]) FOLD_TRY(launch_zero(gr->db[o], (size_t)m.nout[o] * 4, st));
      } else if (gr->dE[o]) {
        FOLD_TRY(launch_zero(gr->dE[o], (size_t)t->vocab[o] * So * 4, st));
      }
    }
  }
  if (s->n_nodes == 0) return FOLD_OK;
  if (!acts || !op || !child || !token || (m.G > 0 && !dh_root)) return FOLD_E_INVALID;
  MoBwdWs w = bwd_ws(t, s, m, npass, ws);
  if (!ws || ws_bytes < w.bytes) return FOLD_E_WORKSPACE;
  MoView v = make_view(t, s, m, (float *)const_cast<void *>(acts), model, op, child, token);
  for (int o = 0; o < m.K; o++) {
    if (!is_cell(t, o)) continue;
    k_mo_pad<<<blocks_for((int64_t)m.nout[o] * m.ldK[o]), 256, 0, st>>>(model->U[o], m.nout[o], m.kin[o], m.ldK[o],
                                                                       w.f.Up[o]);
    FOLD_LAUNCH_CHECK();
  }
  // order position -> slab row (per (depth, op) group: its slab start)
  const std::vector<int64_t> ss = slab_starts(s, m.K, m.D);
  const int ngroups = (m.D + 1) * m.K;
  FOLD_CUDA_TRY(cudaMemcpyAsync(w.gsstart, ss.data(), (size_t)ngroups * 8, cudaMemcpyHostToDevice, st));
  k_mo_slab_index<<<blocks_for(m.N), 256, 0, st>>>(m.N, m.K, ngroups, s->group_off, w.gsstart, w.slab_of_pos);
  FOLD_LAUNCH_CHECK();
  MoBwdView bv{};
  for (int o = 0; o < m.K; o++) { bv.dZ[o] = w.dZ[o]; bv.dA[o] = w.dA[o]; bv.dCe[o] = w.dCe[o]; }
  bv.cons_off = s->cons_off; bv.cons_edge = s->cons_edge; bv.root_off = s->root_off; bv.root_graph = s->root_graph;
  bv.slab_of_pos = w.slab_of_pos; bv.dh_root = dh_root; bv.dh_leaf = w.dh_leaf;
  bv.l0 = s->group_off_host[m.K];
  // reverse sweep: levels D..1
  for (int d = m.D; d >= 1; d--) {
    std::vector<int64_t> sacc(m.K, 0);
    for (int o = 0; o < m.K; o++) sacc[o] = ss[(size_t)d * m.K + o];
    MoLevel L = level_groups(t, s, nullptr, d, sacc);
    if (L.n == 0) continue;
    k_mo_cell_bwd<<<blocks_for(L.rows_total * m.Smax), 256, 0, st>>>(v, bv, L);
    FOLD_LAUNCH_CHECK();
    if (d == 1) continue;
    TfProblem q[kMoGroups];
    int nq = 0;
    for (int g = 0; g < L.n; g++) {
      const int o = L.op[g];
      TfProblem &p = q[nq++];
      p = TfProblem{};
      p.A = TfOperand{w.dZ[o] + (int64_t)L.sstart[g] * m.ldN[o], m.ldN[o], 0};  // dZ [cnt][nout] (K-major)
      p.B = TfOperand{w.f.Up[o], m.ldK[o], 1};                                  // U [nout][kin] as K x N (MN-major)
      p.M = L.cnt[g]; p.N = m.kin[o]; p.K = m.nout[o];
      p.C = w.dA[o] + (int64_t)L.sstart[g] * m.ldK[o];
      p.ldc = m.ldK[o];
    }
    FOLD_TRY(gemm_tf32_grouped(q, nq, npass, w.f.split, w.f.split_floats, st));
  }
  // weight gradients: dU_o = dZ_o^T A_o over the op's whole slab (one grouped launch)
  {
    TfProblem q[kMoGroups];
    int nq = 0;
    for (int o = 0; o < m.K; o++) {
      if (!is_cell(t, o) || m.rows[o] == 0 || !gr->dU[o]) continue;
      TfProblem &p = q[nq++];
      p = TfProblem{};
      p.A = TfOperand{w.dZ[o], m.ldN[o], 1};  // dZ^T: K = rows, M = nout (MN-major)
      p.B = TfOperand{v.A[o], m.ldK[o], 1};   // A: K = rows, N = kin (MN-major)
      p.M = m.nout[o]; p.N = m.kin[o]; p.K = (int)m.rows[o];
      p.C = gr->dU[o]; p.ldc = m.kin[o]; p.accumulate = 1;  // zeroed above unless accumulating
    }
    FOLD_TRY(gemm_tf32_grouped(q, nq, npass, w.dU_split, w.dU_split_floats, st));
  }
  for (int o = 0; o < m.K; o++) {
    if (!is_cell(t, o) || m.rows[o] == 0 || !gr->db[o]) continue;
    const int sp = colsum_splits(m.rows[o]);
    FOLD_TRY(launch_colsum(false, (int)m.rows[o], m.nout[o], w.dZ[o], m.ldN[o], w.colsum, sp, gr->db[o], 1, st));
  }
  if (s->n_leaf_segs > 0) {
    float *dEh[FOLD_MO_MAX_OPS] = {};
    for (int o = 0; o < m.K; o++) dEh[o] = is_cell(t, o) ? nullptr : gr->dE[o];
    FOLD_CUDA_TRY(cudaMemcpyAsync(w.dE_dev, dEh, sizeof(dEh), cudaMemcpyHostToDevice, st));
    k_mo_embed_bwd<<<dim3((unsigned)s->n_leaf_segs, (unsigned)cdiv(m.Smax, 32)), 256, 0, st>>>(
        v, s->leaf_seg, s->leaf_order, bv.l0, w.dh_leaf, w.dE_dev);
    FOLD_LAUNCH_CHECK();
  }
  return FOLD_OK;
}

}  // namespace fold

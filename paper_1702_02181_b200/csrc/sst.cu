// sst.cu — NEXT-2: the §3.5 sentiment model on the level executor.
//
//   h_word = TreeLSTM(Embedding(word), 0, 0)      leaves: one more GEMM level (K = S) whose
//                                                 A operand is the embedding gather
//   h_{left,right} = TreeLSTM(0, h_left, h_right) internal levels: the executor's cells
//   every node: 5-way softmax + cross-entropy     "every node has a sentiment label" (L297)
//
// Runs in the FP32 (3xTF32) and TF32 precision modes on the per-level path: per level a
// gather, one tcgen05 TF32 GEMM (gemm_tf32.cu) and a pointwise step; the leaf level is the
// same GEMM with A = the leaves' embedding rows and B = W (its f-gate rows zero: at a leaf
// c_L = c_R = 0, so the forget gates never contribute, Tai eq 13). The classifier (K = S,
// N = 5) is a warp-per-row dot-product kernel fused with the log-softmax, the loss and the
// logit gradient p - e_y; its weight gradient dWs = (p - e_y)^T H runs on the TF32 GEMM.
// Saved gates of leaves and cells share one [N][gates*ld] array (leaves first), so the
// backward's pointwise kernel serves the leaf level too (rows below n_leaves have no
// children). Deterministic throughout: fixed-order reductions, no float atomics.
#include <cstring>

#include "exec.cuh"

namespace fold {

namespace {

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr int kSstLd = 8;      // row stride of the per-node logit gradients (TMA: 32 B rows)
constexpr int kMaxClasses = 8;
constexpr int kDwsRows = 2048;  // rows per fp64 partial of the classifier gradient

inline int npass_of(int prec) { return prec == FOLD_PREC_TF32 ? 1 : 3; }
inline int64_t ld_a_of(int S) { return round_up(2 * (int64_t)S, 8); }
inline int64_t ld_w_of(int S) { return round_up((int64_t)S, 4); }

fold_status check(const fold_schedule_t *s, const fold_model *m, const fold_sst *q) {
  if (!s || !m || !q || !s->level_off_host) return FOLD_E_INVALID;
  if (m->cell != FOLD_CELL_TREELSTM) return FOLD_E_UNSUPPORTED;
  if (m->prec != FOLD_PREC_FP32 && m->prec != FOLD_PREC_TF32) return FOLD_E_UNSUPPORTED;
  if (!m->U || !m->b || !m->E || !q->W || !q->Ws || !q->bs || (s->n_nodes > 0 && !q->label)) return FOLD_E_INVALID;
  if (m->S <= 0 || m->S > 8192 || q->n_classes < 1 || q->n_classes > kMaxClasses) return FOLD_E_INVALID;
  if (((uintptr_t)m->U | (uintptr_t)m->b | (uintptr_t)m->E | (uintptr_t)q->W | (uintptr_t)q->Ws) & 15)
    return FOLD_E_INVALID;
  return FOLD_OK;
}

// activations of the §3.5 model (one caller buffer)
struct SstActs {
  size_t h, c, g, acat, x, dlog, rowloss, bytes;
  int ld, ld_g;
};
SstActs acts_of(const fold_schedule_t *s, const fold_model *m) {
  SstActs L{};
  const int64_t N = s->n_nodes, nc = s->n_cells, nl = s->n_leaves, S = m->S;
  L.ld = ld_of((int)S);
  L.ld_g = 5 * L.ld;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o = a256(o + b); return r; };
  L.h = take((size_t)(N + 1) * L.ld * 4);
  L.c = take((size_t)(N + 1) * L.ld * 4);
  L.g = take((size_t)(N + 1) * L.ld_g * 4);  // leaves' then cells' saved gates
  L.acat = take((size_t)(nc + 1) * ld_a_of((int)S) * 4);
  L.x = take((size_t)(nl + 1) * L.ld * 4);   // the leaves' inputs E[word]
  L.dlog = take((size_t)(N + 1) * kSstLd * 4);
  L.rowloss = take((size_t)(N + 1) * 4);
  L.bytes = o;
  return L;
}

struct SstFwdWs {
  float *Uf, *Wf;
  size_t bytes;
};
SstFwdWs fwd_ws(void *base, const fold_model *m) {
  SstFwdWs w{};
  const int S = m->S, ld = ld_of(S);
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o = a256(o + b); return r; };
  const size_t ou = take((size_t)5 * ld * tf_ld_u(S) * 4);
  const size_t ow = take((size_t)5 * ld * ld_w_of(S) * 4);
  w.bytes = o;
  if (base) { w.Uf = (float *)((char *)base + ou); w.Wf = (float *)((char *)base + ow); }
  return w;
}

struct SstBwdWs {
  float *Ub, *Wb, *dA, *dCe, *dZ, *part, *dH, *dX, *dW5, *split;
  double *dws;  // classifier-gradient partials (fp64)
  int32_t *root_off;
  EmbedBwdWs emb;
  int ld_z, nsplit;
  int64_t split_floats;
  size_t bytes;
};
SstBwdWs bwd_ws(void *base, const fold_schedule_t *s, const fold_model *m, const fold_sst *q) {
  SstBwdWs w{};
  const int64_t N = s->n_nodes, nc = s->n_cells, nl = s->n_leaves, S = m->S;
  w.ld_z = (int)round_up(5 * S, 8);
  w.nsplit = (int)(N / 128 < 1 ? 1 : (N / 128 > 256 ? 256 : N / 128));
  int64_t sp = gemm_tf32_split_floats(5 * (int)S, 2 * (int)S, (int)nc);
  const int64_t sp2 = gemm_tf32_split_floats(5 * (int)S, (int)S, (int)nl);
  if (sp2 > sp) sp = sp2;
  w.split_floats = sp;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o = a256(o + b); return r; };
  const size_t oub = take((size_t)5 * S * tf_ld_u((int)S) * 4), owb = take((size_t)5 * S * ld_w_of((int)S) * 4);
  const size_t oda = take((size_t)(2 * nc + 1) * S * 4), odc = take((size_t)(2 * nc + 1) * S * 4);
  const size_t odz = take((size_t)(N + 1) * w.ld_z * 4), opa = take((size_t)w.nsplit * 5 * S * 4);
  const size_t odh = take((size_t)(N + 1) * S * 4), odx = take((size_t)(nl + 1) * S * 4);
  const size_t odw = take((size_t)5 * S * S * 4), osp = take((size_t)sp * 4);
  const size_t oro = take((size_t)(N + 2) * 4);
  const size_t ows = take((size_t)cdiv(N < 1 ? 1 : N, kDwsRows) * q->n_classes * (S + 1) * 8);
  const int64_t nseg = s->n_tok_segs, max_pieces = nl / kEmbedPiece + nseg + 1;
  const size_t opc = take((size_t)(nseg + 2) * 4), opo = take((size_t)(nseg + 2) * 4);
  const size_t oss = take((size_t)scan_sums_count(nseg + 1) * 4), oep = take((size_t)max_pieces * S * 4);
  const size_t opsg = take((size_t)max_pieces * 4);
  w.bytes = o;
  if (base) {
    char *p = (char *)base;
    w.Ub = (float *)(p + oub); w.Wb = (float *)(p + owb); w.dA = (float *)(p + oda); w.dCe = (float *)(p + odc);
    w.dZ = (float *)(p + odz); w.part = (float *)(p + opa); w.dH = (float *)(p + odh); w.dX = (float *)(p + odx);
    w.dws = (double *)(p + ows);
    w.dW5 = (float *)(p + odw); w.split = sp > 0 ? (float *)(p + osp) : nullptr; w.root_off = (int32_t *)(p + oro);
    w.emb.piece_cnt = (int32_t *)(p + opc); w.emb.piece_off = (int32_t *)(p + opo);
    w.emb.scan_sums = (int32_t *)(p + oss); w.emb.partial = (float *)(p + oep);
    w.emb.piece_seg = (int32_t *)(p + opsg);
  }
  return w;
}

// W [3S][S] (row blocks i, o, u) -> the 5-gate layouts the GEMMs read: Wf rows gate-padded
// (row g*ld + j, the forward's K-major B: output columns = the saved-gate layout), Wb rows
// natural (g*S + j, the backward's MN-major B); f-gate rows (g = 1, 2) zero
__global__ void k_prep_W(int S, int ld, int64_t ld_w, const float *__restrict__ W, float *__restrict__ Wf,
                         float *__restrict__ Wb) {
  const int64_t total = (int64_t)5 * ld * ld_w;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t row = i / ld_w, k = i % ld_w;
    const int g = (int)(row / ld), j = (int)(row % ld);
    const int blk = g == 0 ? 0 : g == 3 ? 1 : g == 4 ? 2 : -1;
    const float v = (blk >= 0 && j < S && k < S) ? W[((int64_t)blk * S + j) * S + k] : 0.f;
    if (Wf) Wf[i] = v;
    if (Wb && j < S) Wb[((int64_t)g * S + j) * ld_w + k] = v;
  }
}

// Per pool row r: logits l = Ws h_r + bs (C <= 8; one warp, fixed-order butterfly sums),
// p = softmax(l), rowloss[r] = logsumexp(l) - l[y], dlog[r] = p - e_y, y = label[perm[r]].
__global__ void k_sst_classify(int N, int S, int ld, int C, const float *__restrict__ H, const float *__restrict__ Ws,
                               const float *__restrict__ bs, const int32_t *__restrict__ label,
                               const int32_t *__restrict__ perm, float *__restrict__ dlog,
                               float *__restrict__ rowloss) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < N; r += nw) {
    float l[kMaxClasses];
#pragma unroll
    for (int k = 0; k < kMaxClasses; k++) l[k] = 0.f;
    const float *h = H + r * ld;
    for (int j = lane; j < S; j += 32) {
      const float hv = h[j];
#pragma unroll
      for (int k = 0; k < kMaxClasses; k++)
        if (k < C) l[k] = fmaf(Ws[(int64_t)k * S + j], hv, l[k]);
    }
#pragma unroll
    for (int k = 0; k < kMaxClasses; k++)
      for (int o = 16; o; o >>= 1) l[k] += __shfl_xor_sync(0xffffffffu, l[k], o);
    if (lane == 0) {
      const int y = label[perm[r]];
      float mx = -INFINITY;
      for (int k = 0; k < C; k++) { l[k] += bs[k]; mx = fmaxf(mx, l[k]); }
      float se = 0.f;
      for (int k = 0; k < C; k++) se += expf(l[k] - mx);
      const float lse = mx + logf(se);
      float ly = NAN;  // (labels outside [0, C): NaN loss, no one-hot term)
      for (int k = 0; k < C; k++) if (k == y) ly = l[k];
      rowloss[r] = lse - ly;
      for (int k = 0; k < kSstLd; k++) dlog[r * kSstLd + k] = k < C ? expf(l[k] - lse) - (k == y ? 1.f : 0.f) : 0.f;
    }
  }
}

// loss = sum_r rowloss[r]: one block, each thread a fixed strided run, then a fixed tree
__global__ void k_sum_fixed(int64_t n, const float *__restrict__ x, float *__restrict__ out) {
  __shared__ float red[1024];
  float a = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += 1024) a += x[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 512; o; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// dH[r][j] = sum_k dlog[r][k] Ws[k][j]: the classifier's contribution to every node's dh
__global__ void k_sst_dh(int64_t N, int S, int C, const float *__restrict__ dlog, const float *__restrict__ Ws,
                         float *__restrict__ dH) {
  const int64_t total = N * S, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / S;
    const int j = (int)(i % S);
    float a = 0.f;
    for (int k = 0; k < C; k++) a = fmaf(dlog[r * kSstLd + k], Ws[(int64_t)k * S + j], a);
    dH[i] = a;
  }
}

// Classifier weight gradient dWs[k][j] = sum_r dlog[r][k] H[r][j], dbs[k] = sum_r dlog[r][k]:
// a K = N reduction of a random-walk sum (labels are independent of h), so it accumulates in
// fp64 (fp32 accumulation alone would carry ~eps sqrt(N) relative error); split over row
// chunks (fixed), partials [split][C][S + 1] (column S = dbs), summed in order by k_sst_dws_final.
__global__ void k_sst_dws_part(int64_t N, int S, int C, int ld, const float *__restrict__ dlog,
                               const float *__restrict__ H, double *__restrict__ part) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;  // column (j == S: the bias column)
  if (j > S) return;
  const int64_t r0 = (int64_t)blockIdx.y * kDwsRows, r1 = min(N, r0 + kDwsRows);
  double acc[kMaxClasses];
#pragma unroll
  for (int k = 0; k < kMaxClasses; k++) acc[k] = 0.0;
  for (int64_t r = r0; r < r1; r++) {
    const double h = j < S ? (double)H[r * ld + j] : 1.0;
#pragma unroll
    for (int k = 0; k < kMaxClasses; k++)
      if (k < C) acc[k] += (double)dlog[r * kSstLd + k] * h;
  }
  for (int k = 0; k < C; k++) part[((int64_t)blockIdx.y * C + k) * (S + 1) + j] = acc[k];
}
__global__ void k_sst_dws_final(int nsplit, int S, int C, const double *__restrict__ part, float *__restrict__ dWs,
                                float *__restrict__ dbs, int accumulate) {
  const int64_t total = (int64_t)C * (S + 1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / (S + 1)), j = (int)(i % (S + 1));
    double a = 0.0;
    for (int sp = 0; sp < nsplit; sp++) a += part[((int64_t)sp * C + k) * (S + 1) + j];
    float *dst = j < S ? dWs + (int64_t)k * S + j : dbs + k;
    *dst = accumulate ? *dst + (float)a : (float)a;
  }
}

// dW[b][j][k] (+)= dW5[blk(b) * S + j][k], blk = (0, 3, 4): the i, o, u rows
__global__ void k_take_iou(int S, const float *__restrict__ dW5, float *__restrict__ dW, int accumulate) {
  const int64_t total = (int64_t)3 * S * S, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t b = i / ((int64_t)S * S), rest = i % ((int64_t)S * S);
    const int64_t blk = b == 0 ? 0 : b == 1 ? 3 : 4;
    const float v = dW5[blk * S * S + rest];
    dW[i] = accumulate ? dW[i] + v : v;
  }
}

unsigned grid_of(int64_t work, int per = 256) {
  int64_t b = cdiv(work < 1 ? 1 : work, per);
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)b;
}

}  // namespace

}  // namespace fold

using namespace fold;

extern "C" {

fold_status fold_sst_acts_layout(const fold_schedule_t *s, const fold_model *m, const fold_sst *q,
                                 fold_acts_layout_t *out) {
  FOLD_TRY(check(s, m, q));
  if (!out) return FOLD_E_INVALID;
  SstActs L = acts_of(s, m);
  out->bytes = L.bytes; out->h_off = L.h; out->c_off = L.c; out->g_off = L.g;
  out->ld = L.ld; out->h_elem_bytes = 4;
  return FOLD_OK;
}

size_t fold_sst_forward_workspace(const fold_schedule_t *s, const fold_model *m, const fold_sst *q) {
  if (check(s, m, q) != FOLD_OK) return 0;
  return fwd_ws(nullptr, m).bytes;
}

size_t fold_sst_backward_workspace(const fold_schedule_t *s, const fold_model *m, const fold_sst *q) {
  if (check(s, m, q) != FOLD_OK) return 0;
  return bwd_ws(nullptr, s, m, q).bytes;
}

// Forward (PAPER.md L47 loop with the §3.5 cells): depth 1 = the leaf cell on E[word], depth
// d >= 2 the x = 0 cell; then every node's classifier and the summed cross-entropy.
fold_status fold_sst_forward(const fold_schedule_t *s, const fold_model *m, const fold_sst *q, void *acts,
                             float *loss, void *ws, size_t ws_bytes, void *stream) {
  FOLD_TRY(check(s, m, q));
  cudaStream_t st = (cudaStream_t)stream;
  SstFwdWs w = fwd_ws(ws, m);
  if (!ws || ws_bytes < w.bytes) return FOLD_E_WORKSPACE;
  const int N = s->n_nodes, S = m->S, D = s->n_levels, nl = s->n_leaves, C = q->n_classes;
  if (!loss) return FOLD_E_INVALID;
  if (N == 0) return launch_zero(loss, 4, st);
  if (!acts || !s->leaf_token || !s->perm) return FOLD_E_INVALID;
  SstActs L = acts_of(s, m);
  char *a = (char *)acts;
  float *H = (float *)(a + L.h), *Cm = (float *)(a + L.c), *G = (float *)(a + L.g);
  float *Acat = (float *)(a + L.acat), *X = (float *)(a + L.x);
  float *Gc = G + (int64_t)nl * L.ld_g;  // cell-indexed view (rows below 0 are the leaves')
  const int npass = npass_of(m->prec);
  const int32_t *lo = s->level_off_host;
  {
    ProfScope ps(K_PREP, st);
    FOLD_TRY(launch_prep_U_tf(5, S, L.ld, m->U, w.Uf, nullptr, st));
    k_prep_W<<<grid_of((int64_t)5 * L.ld * ld_w_of(S)), 256, 0, st>>>(S, L.ld, ld_w_of(S), q->W, w.Wf, nullptr);
    FOLD_LAUNCH_CHECK();
  }
  {
    // depth 1: x = E[word] (the embedding gather), z = W x + b, then the cell with no children
    ProfScope ps(K_EMBED_FWD, st);
    FOLD_TRY(launch_embed_fwd(false, 0, nl, s->leaf_token, m->E, S, L.ld, X, Cm, nullptr, st));
    FOLD_TRY(gemm_tf32(TfOperand{X, L.ld, 0}, TfOperand{w.Wf, ld_w_of(S), 0}, nl, 5 * L.ld, S, G, L.ld_g, 0, npass,
                       nullptr, 0, st));
    FOLD_TRY(launch_cell_fwd_pw(FOLD_CELL_TREELSTM, 0, nl, nl, S, L.ld, L.ld_g, s->gather, m->b, H, Cm, Gc, st));
  }
  const int64_t lda = ld_a_of(S);
  {
  ProfScope ps(K_CELL_FWD, st);  // one bracket around the level sweep (fewer events in the step)
  for (int d = 2; d <= D; d++) {
    const int r0 = lo[d], r1 = lo[d + 1], M = r1 - r0, c0 = r0 - nl;
    if (M <= 0) continue;
    FOLD_TRY(launch_gather_cat(r0, r1, nl, S, L.ld, s->gather, H, Acat, lda, st));
    FOLD_TRY(gemm_tf32(TfOperand{Acat + (int64_t)c0 * lda, lda, 0}, TfOperand{w.Uf, tf_ld_u(S), 0}, M, 5 * L.ld,
                       2 * S, Gc + (int64_t)c0 * L.ld_g, L.ld_g, 0, npass, nullptr, 0, st));
    FOLD_TRY(launch_cell_fwd_pw(FOLD_CELL_TREELSTM, r0, r1, nl, S, L.ld, L.ld_g, s->gather, m->b, H, Cm, Gc, st));
  }
  }
  ProfScope ps(K_ROOT, st);
  float *dlog = (float *)(a + L.dlog), *rowloss = (float *)(a + L.rowloss);
  k_sst_classify<<<grid_of((int64_t)N * 32), 256, 0, st>>>(N, S, L.ld, C, H, q->Ws, q->bs, q->label, s->perm, dlog,
                                                           rowloss);
  FOLD_LAUNCH_CHECK();
  k_sum_fixed<<<1, 1024, 0, st>>>(N, rowloss, loss);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

// Backward of the summed cross-entropy (seed dL = 1): classifier -> every node's dh; the
// reverse level sweep over cells and then the leaf level; the leaf input
// gradient dX = dz W reaches dE through the token-segmented reduction; dU / dW / dWs on
// the TF32 GEMM, db / dbs as fixed-order column sums.
fold_status fold_sst_backward(const fold_schedule_t *s, const fold_model *m, const fold_sst *q, const void *acts,
                              fold_grads *grads, fold_sst_grads *sg, void *ws, size_t ws_bytes, void *stream) {
  FOLD_TRY(check(s, m, q));
  if (!grads || !grads->dU || !grads->db || !grads->dE || !sg || !sg->dW || !sg->dWs || !sg->dbs)
    return FOLD_E_INVALID;
  if (((uintptr_t)grads->dU | (uintptr_t)grads->db | (uintptr_t)grads->dE | (uintptr_t)sg->dW | (uintptr_t)sg->dWs |
       (uintptr_t)sg->dbs) & 15)
    return FOLD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  SstBwdWs w = bwd_ws(ws, s, m, q);
  if (!ws || ws_bytes < w.bytes) return FOLD_E_WORKSPACE;
  const int N = s->n_nodes, S = m->S, D = s->n_levels, nl = s->n_leaves, nc = s->n_cells, C = q->n_classes;
  const int acc = grads->accumulate ? 1 : 0;
  if (!acc) {
    FOLD_TRY(launch_zero(grads->dU, (size_t)5 * S * 2 * S * 4, st));
    FOLD_TRY(launch_zero(grads->db, (size_t)5 * S * 4, st));
    FOLD_TRY(launch_zero(grads->dE, (size_t)m->vocab * S * 4, st));
    FOLD_TRY(launch_zero(sg->dW, (size_t)3 * S * S * 4, st));
    FOLD_TRY(launch_zero(sg->dWs, (size_t)C * S * 4, st));
    FOLD_TRY(launch_zero(sg->dbs, (size_t)C * 4, st));
  }
  if (N == 0) return FOLD_OK;
  if (!acts) return FOLD_E_INVALID;
  SstActs L = acts_of(s, m);
  const char *a = (const char *)acts;
  const float *H = (const float *)(a + L.h), *Cm = (const float *)(a + L.c), *G = (const float *)(a + L.g);
  const float *Acat = (const float *)(a + L.acat), *X = (const float *)(a + L.x);
  const float *dlog = (const float *)(a + L.dlog);
  const float *Gc = G + (int64_t)nl * L.ld_g;
  float *dZc = w.dZ + (int64_t)nl * w.ld_z;  // cell-indexed view
  const int npass = npass_of(m->prec);
  const int32_t *lo = s->level_off_host;
  {
    ProfScope ps(K_PREP, st);
    FOLD_TRY(launch_prep_U_tf(5, S, L.ld, m->U, nullptr, w.Ub, st));
    k_prep_W<<<grid_of((int64_t)5 * L.ld * ld_w_of(S)), 256, 0, st>>>(S, L.ld, ld_w_of(S), q->W, nullptr, w.Wb);
    FOLD_LAUNCH_CHECK();
    FOLD_TRY(launch_root_off(N, 0, s->root_row, s->root_perm, w.root_off, st));  // no root seeds
    k_sst_dh<<<grid_of((int64_t)N * S), 256, 0, st>>>(N, S, C, dlog, q->Ws, w.dH);
    FOLD_LAUNCH_CHECK();
  }
  auto pw = [&](int r0, int r1) {
    return launch_cell_bwd_pw(false, FOLD_CELL_TREELSTM, r0, r1, nl, S, L.ld, L.ld_g, s->cons_off, s->cons_edge,
                              w.root_off, s->root_perm, 0, nullptr, nullptr, s->gather, Gc, Cm, w.dA, w.dCe, dZc,
                              w.ld_z, st, nullptr, w.dH, true);
  };
  {
  ProfScope ps(K_GEMM_DA, st);  // the backward level sweep (pointwise + dA GEMM per level)
  for (int d = D; d >= 2; d--) {
    const int r0 = lo[d], r1 = lo[d + 1], M = r1 - r0, c0 = r0 - nl;
    if (M <= 0) continue;
    FOLD_TRY(pw(r0, r1));
    FOLD_TRY(gemm_tf32(TfOperand{dZc + (int64_t)c0 * w.ld_z, w.ld_z, 0}, TfOperand{w.Ub, tf_ld_u(S), 1}, M, 2 * S,
                       5 * S, w.dA + (int64_t)2 * c0 * S, 2 * S, 0, npass, nullptr, 0, st));
  }
  }
  {
    // depth 1: the leaf cells (no children), then their input gradient dX = dz W -> dE
    ProfScope ps(K_EMBED_BWD, st);
    FOLD_TRY(pw(0, nl));
    FOLD_TRY(gemm_tf32(TfOperand{w.dZ, w.ld_z, 0}, TfOperand{w.Wb, ld_w_of(S), 1}, nl, S, 5 * S, w.dX, S, 0, npass,
                       nullptr, 0, st));
    FOLD_TRY(launch_embed_bwd_pieces(S, nl, s->n_tok_segs, s->tok_seg, s->leaf_perm, s->leaf_token, s->cons_off,
                                     s->cons_edge, w.root_off, s->root_perm, nullptr, nullptr, false, grads->dE, w.emb,
                                     st, w.dX));
  }
  ProfScope ps(K_GEMM_DU, st);
  // dU = dZ_cells^T Acat; dW = the (i, o, u) rows of dZ_leaves^T X; dWs = dlog^T H
  FOLD_TRY(gemm_tf32(TfOperand{dZc, w.ld_z, 1}, TfOperand{Acat, ld_a_of(S), 1}, 5 * S, 2 * S, nc, grads->dU, 2 * S,
                     acc, npass, w.split, w.split_floats, st));
  FOLD_TRY(gemm_tf32(TfOperand{w.dZ, w.ld_z, 1}, TfOperand{X, L.ld, 1}, 5 * S, S, nl, w.dW5, S, 0, npass, w.split,
                     w.split_floats, st));
  k_take_iou<<<grid_of((int64_t)3 * S * S), 256, 0, st>>>(S, w.dW5, sg->dW, acc);
  FOLD_LAUNCH_CHECK();
  {
    const int nsp = (int)cdiv(N, kDwsRows);
    k_sst_dws_part<<<dim3((unsigned)cdiv(S + 1, 128), (unsigned)nsp), 128, 0, st>>>(N, S, C, L.ld, dlog, H, w.dws);
    FOLD_LAUNCH_CHECK();
    k_sst_dws_final<<<grid_of((int64_t)C * (S + 1)), 256, 0, st>>>(nsp, S, C, w.dws, sg->dWs, sg->dbs, acc);
    FOLD_LAUNCH_CHECK();
  }
  // db over leaves and cells (a leaf's f-gate dz is 0: c_L = c_R = 0)
  FOLD_TRY(launch_colsum(false, N, 5 * S, w.dZ, w.ld_z, w.part, w.nsplit, grads->db, acc, st));
  return FOLD_OK;
}

}  // extern "C"

// exec.cu — level executor kernels other than the tcgen05 GEMMs:
//   embedding level (Fig. 1 "embed lookup", L67), the fp32 SIMT cell kernel
//   (FOLD_PREC_FP32 mode), root read-out, the backward pointwise pull-reduce kernel,
//   fp32 SIMT GEMMs for the backward, deterministic column sums (db), the segmented
//   embedding gradient, and SGD.
// Cell equations: DESIGN.md "Cell" (TreeLSTM = Tai et al. eqs 9-14 with x=0, N=2,
// cited at PAPER.md L301-304; TreeRNN = tanh(W[h_L;h_R]+b), Fig. 1 "RNN Cell").
#include "exec.cuh"

namespace fold {

namespace {

inline unsigned grid_cap(int64_t blocks) {
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 32) blocks = 148 * 32;
  return (unsigned)blocks;
}

// ---------------------------------------------------------------- embedding forward
// H[r] = E[leaf_token[r]], C[r] = 0 for the level-1 rows [r0, r1). One warp per row.
// BF16 path (sc != null): h is also pushed to the A-operand row of every consumer edge.
template <typename T>
__global__ void k_embed_fwd(int r0, int r1, const int32_t *__restrict__ leaf_token,
                            const float *__restrict__ E, int S, int ld, T *__restrict__ H, float *__restrict__ C,
                            ScatterA sc, int has_sc) {
  int lane = threadIdx.x & 31;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = r0 + w; r < r1; r += nw) {
    int tok = leaf_token[r];
    const float *e = E + (int64_t)tok * S;
    T *h = H + r * ld;
    float *c = C + r * ld;
    int e0 = 0, e1 = 0;
    if (has_sc) { e0 = sc.cons_off[r]; e1 = sc.cons_off[r + 1]; }
    if (sizeof(T) == 2 && has_sc && (S & 3) == 0) {
      // BF16 push path: the (usually one) consumer rows resolved once, four float4 loads in
      // flight per lane before the stores
      __nv_bfloat16 *d0 = nullptr;
      if (e1 > e0) {
        const int ed = sc.cons_edge[e0];
        d0 = ((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld;
      }
      for (int jb = lane * 4; jb < S; jb += 512) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (jb + 128 * u < S) v[u] = *reinterpret_cast<const float4 *>(e + jb + 128 * u);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int j = jb + 128 * u;
          if (j >= S) break;
          __nv_bfloat162 a = __floats2bfloat162_rn(v[u].x, v[u].y), b2 = __floats2bfloat162_rn(v[u].z, v[u].w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t *>(&a);
          pk.y = *reinterpret_cast<uint32_t *>(&b2);
          // the pool row only for leaves nobody consumes (roots); consumers read the pushed
          // copy in their A rows
          if (e1 == e0) *reinterpret_cast<uint2 *>(h + j) = pk;
          else *reinterpret_cast<uint2 *>(d0 + j) = pk;
          for (int q = e0 + 1; q < e1; q++) {
            const int ed = sc.cons_edge[q];
            __nv_bfloat16 *dst = ((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld + j;
            *reinterpret_cast<uint2 *>(dst) = pk;
          }
        }
      }
    } else if ((S & 3) == 0) {
      for (int j = lane * 4; j < S; j += 128) {
        float4 v = *reinterpret_cast<const float4 *>(e + j);
        if constexpr (sizeof(T) == 2) {
          __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b2 = __floats2bfloat162_rn(v.z, v.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t *>(&a);
          pk.y = *reinterpret_cast<uint32_t *>(&b2);
          // BF16: the pool row only for leaves nobody consumes (roots); consumers read the
          // pushed copy in their A rows
          if (e1 == e0) *reinterpret_cast<uint2 *>(h + j) = pk;
          for (int q = e0; q < e1; q++) {
            int ed = sc.cons_edge[q];
            __nv_bfloat16 *dst = ((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld + j;
            *reinterpret_cast<uint2 *>(dst) = pk;
          }
        } else {
          *reinterpret_cast<float4 *>(h + j) = v;
        }
        if (!has_sc) *reinterpret_cast<float4 *>(c + j) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      for (int j = lane; j < S; j += 32) {
        T hv = from_f<T>(e[j]);
        if (sizeof(T) == 4 || e1 == e0) h[j] = hv;
        if (!has_sc) c[j] = 0.f;
        if constexpr (sizeof(T) == 2) {
          for (int q = e0; q < e1; q++) {
            int ed = sc.cons_edge[q];
            (((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld)[j] = hv;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- fp32 SIMT cell forward
// Block tile: 32 rows x 32 state columns x all GATES gate blocks; K = 2S in chunks of 32.
// A row m = [H[gL] | H[gR]] gathered on the fly (gather -> op -> concat,
// the concat being the append into rows [r0, r1) of the pool).
template <int GATES>
__global__ void __launch_bounds__(256) k_cell_fwd_simt(int r0, int r1, const int32_t *__restrict__ gather,
                                                       int S, int ld, const float *__restrict__ U,
                                                       const float *__restrict__ bias, float *__restrict__ H,
                                                       float *__restrict__ C, float *__restrict__ Gact, int ld_g,
                                                       int nl) {
  constexpr int BM = 32, BW = 32, BK = 32;
  __shared__ float As[BK][BM + 1];
  __shared__ float Bs[GATES][BK][BW + 1];
  __shared__ int gl[BM], gr[BM];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;  // ty: 0..7
  const int m0 = r0 + blockIdx.x * BM, j0 = blockIdx.y * BW;
  const int M = r1 - r0;
  if (tid < BM) {
    int r = m0 + tid;
    bool ok = r < r1;
    gl[tid] = ok ? gather[2 * (int64_t)r] : 0;
    gr[tid] = ok ? gather[2 * (int64_t)r + 1] : 0;
  }
  __syncthreads();
  float acc[4][GATES];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int g = 0; g < GATES; g++) acc[i][g] = 0.f;
  const int K = 2 * S;
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int it = 0; it < (BM * BK) / 256; it++) {
      int idx = tid + it * 256, kk = idx & 31, mm = idx >> 5;
      int k = k0 + kk;
      float v = 0.f;
      if (k < K && (m0 - r0) + mm < M) {
        int row = k < S ? gl[mm] : gr[mm];
        v = H[(int64_t)row * ld + (k < S ? k : k - S)];
      }
      As[kk][mm] = v;
    }
#pragma unroll
    for (int g = 0; g < GATES; g++)
#pragma unroll
      for (int it = 0; it < (BW * BK) / 256; it++) {
        int idx = tid + it * 256, kk = idx & 31, jj = idx >> 5;
        int k = k0 + kk, j = j0 + jj;
        Bs[g][kk][jj] = (k < K && j < S) ? U[((int64_t)g * S + j) * K + k] : 0.f;
      }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; kk++) {
      float a[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int g = 0; g < GATES; g++) {
        float bv = Bs[g][kk][tx];
#pragma unroll
        for (int i = 0; i < 4; i++) acc[i][g] = fmaf(a[i], bv, acc[i][g]);
      }
    }
    __syncthreads();
  }
  const int j = j0 + tx;
  if (j >= S) return;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int mm = ty * 4 + i;
    int64_t r = m0 + mm;
    if (r >= r1) continue;
    int64_t c = r - nl;
    if constexpr (GATES == 1) {
      float h = tanhf(acc[i][0] + bias[j]);
      H[r * ld + j] = h;
      C[r * ld + j] = 0.f;
      Gact[c * ld_g + j] = h;
    } else {
      float zi = acc[i][0] + bias[j], zfl = acc[i][1] + bias[S + j], zfr = acc[i][2] + bias[2 * S + j];
      float zo = acc[i][3] + bias[3 * S + j], zu = acc[i][4] + bias[4 * S + j];
      float ig = 1.f / (1.f + expf(-zi)), fl = 1.f / (1.f + expf(-zfl)), fr = 1.f / (1.f + expf(-zfr));
      float og = 1.f / (1.f + expf(-zo)), ug = tanhf(zu);
      float cl = C[(int64_t)gl[mm] * ld + j], cr = C[(int64_t)gr[mm] * ld + j];
      float cc = ig * ug + fl * cl + fr * cr;
      H[r * ld + j] = og * tanhf(cc);
      C[r * ld + j] = cc;
      float *ga = Gact + c * ld_g;
      ga[j] = ig; ga[ld + j] = fl; ga[2 * ld + j] = fr; ga[3 * ld + j] = og; ga[4 * ld + j] = ug;
    }
  }
}

// ---------------------------------------------------------------- roots out
// BF16 path: cell rows that have consumers keep h only in their consumers' A-operand
// rows (the pool row is written for consumer-free rows), so a consumed root reads it there.
template <typename T>
__global__ void k_root_out(int G, int S, int ld, int nl, const int32_t *__restrict__ root_row,
                           const T *__restrict__ H, const float *__restrict__ C, float *__restrict__ h_root,
                           float *__restrict__ c_root, ScatterA sc, int has_sc) {
  int64_t total = (int64_t)G * S;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    int64_t g = i / S, j = i - g * S;
    int64_t r = root_row[g];
    const T *src = H + r * ld;
    if (has_sc && sc.cons_off[r + 1] > sc.cons_off[r]) {  // consumed (leaf or cell): its pushed copy
      int ed = sc.cons_edge[sc.cons_off[r]];
      src = reinterpret_cast<const T *>(((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld);
    }
    if (h_root) h_root[i] = to_f(src[j]);
    if (c_root) c_root[i] = r >= nl ? C[r * ld + j] : 0.f;
  }
}

// ---------------------------------------------------------------- backward pointwise
// Per cell row r of one level (one warp per row):
//   dh = sum_{roots g at r, ascending g} dh_root[g] + sum_{e in cons(r), ascending} dA[e]
//   dc = sum_{roots} dc_root[g] + sum_{e} dCe[e]                 (pull, no atomics)
//   TreeLSTM: tc = tanh(c); do = dh*tc; dc += dh*o*(1-tc^2)
//             dz = [dc*u*i(1-i), dc*cL*fL(1-fL), dc*cR*fR(1-fR), do*o(1-o), dc*i*(1-u^2)]
//             dCe[2c] = dc*fL, dCe[2c+1] = dc*fR
//   TreeRNN:  dz = dh*(1-h^2)
template <typename T, int V> struct VecIO;
template <> struct VecIO<float, 1> {
  static __device__ __forceinline__ void ld(const float *p, float *v) { v[0] = *p; }
  static __device__ __forceinline__ void st(float *p, const float *v) { *p = v[0]; }
};
template <> struct VecIO<float, 4> {
  static __device__ __forceinline__ void ld(const float *p, float *v) {
    float4 x = *reinterpret_cast<const float4 *>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
  static __device__ __forceinline__ void st(float *p, const float *v) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct VecIO<__nv_bfloat16, 1> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16 *p, float *v) { v[0] = __bfloat162float(*p); }
  static __device__ __forceinline__ void st(__nv_bfloat16 *p, const float *v) { *p = __float2bfloat16_rn(v[0]); }
};
template <> struct VecIO<__nv_bfloat16, 4> {
  static __device__ __forceinline__ void ld(const __nv_bfloat16 *p, float *v) {
    uint2 x = *reinterpret_cast<const uint2 *>(p);
    float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162 *>(&x.x));
    float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162 *>(&x.y));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  static __device__ __forceinline__ void st(__nv_bfloat16 *p, const float *v) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 x;
    x.x = *reinterpret_cast<uint32_t *>(&a);
    x.y = *reinterpret_cast<uint32_t *>(&b);
    *reinterpret_cast<uint2 *>(p) = x;
  }
};

// VEC consecutive state columns per lane (VEC = 4 needs S % 4 == 0: 16-byte fp32 and
// 8-byte bf16 accesses stay aligned since every row stride is a multiple of 8 elements).
template <typename T, int GATES, int VEC>
__global__ void k_cell_bwd_pw(int r0, int r1, int nl, int S, int ld, int ld_g, const int32_t *__restrict__ cons_off,
                              const int32_t *__restrict__ cons_edge, const int32_t *__restrict__ root_off,
                              const int32_t *__restrict__ root_perm, int G, const float *__restrict__ dh_root,
                              const float *__restrict__ dc_root, const int32_t *__restrict__ gather,
                              const T *__restrict__ Gact, const float *__restrict__ C, const float *__restrict__ dA,
                              float *__restrict__ dCe, T *__restrict__ dZ, int ld_z, const int32_t *__restrict__ root_row,
                              const float *__restrict__ dh_node, int c_rows0) {
  using IT = VecIO<T, VEC>;
  using IF = VecIO<float, VEC>;
  int lane = threadIdx.x & 31;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // warp task = (row, block of 32*VEC columns): narrow levels still spread over all SMs.
  // Root mode (root_row != null): the rows are the distinct cell root rows, visited in
  // root_perm order (index i in [r0, r1) = [0, G)).
  const int nblk = (int)cdiv(S, 32 * VEC);
  const int64_t ntask = (int64_t)(r1 - r0) * nblk;
  for (int64_t task = w; task < ntask; task += nw) {
    int64_t r = r0 + task / nblk;
    if (root_row) {
      const int q = (int)r;
      r = root_row[root_perm[q]];
      if (r < nl || (q > 0 && root_row[root_perm[q - 1]] == r)) continue;
    }
    const int j = (int)(task % nblk) * 32 * VEC + lane * VEC;
    int64_t c = r - nl;
    int e0 = cons_off[r], e1 = cons_off[r + 1];
    // roots seeded at this row: root_perm[root_off[r] .. root_off[r+1]) (ascending g)
    const int rs0 = root_off[r], rs1 = root_off[r + 1];
    const T *ga = Gact + c * ld_g;
    T *dz = dZ + c * ld_z;
    int64_t gL = gather[2 * r], gR = gather[2 * r + 1];
    if (j < S) {
      float dh[VEC], dc[VEC], t[VEC];
#pragma unroll
      for (int u = 0; u < VEC; u++) { dh[u] = 0.f; dc[u] = 0.f; }
      for (int q = rs0; q < rs1; q++) {
        int g = root_perm[q];
        IF::ld(dh_root + (int64_t)g * S + j, t);
#pragma unroll
        for (int u = 0; u < VEC; u++) dh[u] += t[u];
        if (dc_root) {
          IF::ld(dc_root + (int64_t)g * S + j, t);
#pragma unroll
          for (int u = 0; u < VEC; u++) dc[u] += t[u];
        }
      }
      if (dh_node) {  // a per-node loss term (§3.5 classifier), pool-row indexed [N][S]
        IF::ld(dh_node + r * S + j, t);
#pragma unroll
        for (int u = 0; u < VEC; u++) dh[u] += t[u];
      }
      for (int e = e0; e < e1; e++) {
        int64_t ed = cons_edge[e];
        IF::ld(dA + ed * S + j, t);
#pragma unroll
        for (int u = 0; u < VEC; u++) dh[u] += t[u];
        if (GATES == 5) {
          IF::ld(dCe + ed * S + j, t);
#pragma unroll
          for (int u = 0; u < VEC; u++) dc[u] += t[u];
        }
      }
      if constexpr (GATES == 1) {
        float h[VEC], o[VEC];
        IT::ld(ga + j, h);
#pragma unroll
        for (int u = 0; u < VEC; u++) o[u] = dh[u] * (1.f - h[u] * h[u]);
        IT::st(dz + j, o);
      } else {
        float ig[VEC], fl[VEC], fr[VEC], og[VEC], ug[VEC], cc[VEC], cl[VEC], cr[VEC];
        IT::ld(ga + j, ig); IT::ld(ga + ld + j, fl); IT::ld(ga + 2 * ld + j, fr);
        IT::ld(ga + 3 * ld + j, og); IT::ld(ga + 4 * ld + j, ug);
        IF::ld(C + r * ld + j, cc);
        // children below row c_rows0 have c = 0: the R1 model's leaves (c_rows0 = nl; their C
        // rows are not materialised in BF16 mode); the §3.5 leaf cells have c (c_rows0 = 0)
#pragma unroll
        for (int u = 0; u < VEC; u++) { cl[u] = 0.f; cr[u] = 0.f; }
        if (gL >= c_rows0) IF::ld(C + gL * ld + j, cl);
        if (gR >= c_rows0) IF::ld(C + gR * ld + j, cr);
        float z0[VEC], z1[VEC], z2[VEC], z3[VEC], z4[VEC], eL[VEC], eR[VEC];
#pragma unroll
        for (int u = 0; u < VEC; u++) {
          float tc = tanhf(cc[u]);
          float dO = dh[u] * tc;
          float dcc = dc[u] + dh[u] * og[u] * (1.f - tc * tc);
          z0[u] = dcc * ug[u] * ig[u] * (1.f - ig[u]);
          z1[u] = dcc * cl[u] * fl[u] * (1.f - fl[u]);
          z2[u] = dcc * cr[u] * fr[u] * (1.f - fr[u]);
          z3[u] = dO * og[u] * (1.f - og[u]);
          z4[u] = dcc * ig[u] * (1.f - ug[u] * ug[u]);
          eL[u] = dcc * fl[u];
          eR[u] = dcc * fr[u];
        }
        IT::st(dz + j, z0); IT::st(dz + S + j, z1); IT::st(dz + 2 * S + j, z2);
        IT::st(dz + 3 * S + j, z3); IT::st(dz + 4 * S + j, z4);
        if (c >= 0) {  // (rows below nl: §3.5 leaf cells, no children)
          IF::st(dCe + (2 * c) * S + j, eL);
          IF::st(dCe + (2 * c + 1) * S + j, eR);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- fp32 SIMT GEMMs
// dA[m][n] = sum_k dZ[m][k] U[k][n];  M rows, N = 2S, K = gates*S. 64x64 tiles, BK 16.
__global__ void __launch_bounds__(256) k_gemm_dA_simt(int M, int N, int K, const float *__restrict__ A, int lda,
                                                      const float *__restrict__ B, int ldb, float *__restrict__ Cm,
                                                      int ldc) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int it = 0; it < 4; it++) {
      int idx = tid + it * 256, kk = idx & 15, mm = idx >> 4;
      int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? A[(int64_t)m * lda + k] : 0.f;
      int nn = idx & 63, kb = idx >> 6;
      int n = n0 + nn, k2 = k0 + kb;
      Bs[kb][nn] = (n < N && k2 < K) ? B[(int64_t)k2 * ldb + n] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; kk++) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[i][q] = fmaf(a[i], b[q], acc[i][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      int n = n0 + tx * 4 + q;
      if (n < N) Cm[(int64_t)m * ldc + n] = acc[i][q];
    }
  }
}

// dU[i][j] = sum_c dZ[c][i] * Acat(c, j), Acat(c, j) = H[gather[2(nl+c) + (j >= S)]][j mod S].
// M = gates*S (i), N = 2S (j), K = n_cells (c, fixed ascending order per output).
__global__ void __launch_bounds__(256) k_gemm_dU_simt(int n_cells, int nl, int S, int Mg, const float *__restrict__ dZ,
                                                      int ld_z, const int32_t *__restrict__ gather,
                                                      const float *__restrict__ H, int ld, float *__restrict__ dU,
                                                      int accumulate) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int N = 2 * S;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < n_cells; k0 += 16) {
#pragma unroll
    for (int it = 0; it < 4; it++) {
      int idx = tid + it * 256, mm = idx & 63, kk = idx >> 6;
      int c = k0 + kk;
      int m = m0 + mm;
      As[kk][mm] = (c < n_cells && m < Mg) ? dZ[(int64_t)c * ld_z + m] : 0.f;
      int n = n0 + mm;
      float v = 0.f;
      if (c < n_cells && n < N) {
        int half = n >= S;
        int64_t row = gather[2 * ((int64_t)nl + c) + half];
        v = H[row * ld + (n - half * S)];
      }
      Bs[kk][mm] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; kk++) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[i][q] = fmaf(a[i], b[q], acc[i][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int m = m0 + ty * 4 + i;
    if (m >= Mg) continue;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      int n = n0 + tx * 4 + q;
      if (n >= N) continue;
      float *p = dU + (int64_t)m * N + n;
      *p = accumulate ? *p + acc[i][q] : acc[i][q];
    }
  }
}

// ---------------------------------------------------------------- column sums (db)
// partial[s][j] = sum over rows of split s (ascending) ; then db[j] = sum_s partial[s][j].
// VEC consecutive columns per thread (16-byte bf16 / 32-byte fp32 loads per row).
template <typename T, int VEC>
__global__ void k_colsum_partial(int n_rows, int ncols, const T *__restrict__ X, int ldx, int nsplit,
                                 float *__restrict__ partial) {
  using IT = VecIO<T, VEC == 8 ? 4 : 1>;
  int s = blockIdx.y;
  int64_t rows_per = cdiv(n_rows, nsplit);
  int64_t a = s * rows_per, b = a + rows_per < n_rows ? a + rows_per : n_rows;
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) * VEC; j < ncols; j += gridDim.x * blockDim.x * VEC) {
    float acc[VEC];
#pragma unroll
    for (int u = 0; u < VEC; u++) acc[u] = 0.f;
    // (unrolled: several rows' loads in flight per thread; the sum stays in row order)
#pragma unroll 8
    for (int64_t r = a; r < b; r++) {
      const T *x = X + r * ldx + j;
      if constexpr (VEC == 8) {
        float t0[4], t1[4];
        IT::ld(x, t0);
        IT::ld(x + 4, t1);
#pragma unroll
        for (int u = 0; u < 4; u++) { acc[u] += t0[u]; acc[4 + u] += t1[u]; }
      } else {
        acc[0] += to_f(x[0]);
      }
    }
#pragma unroll
    for (int u = 0; u < VEC; u++) partial[(int64_t)s * ncols + j + u] = acc[u];
  }
}

__global__ void k_colsum_final(int ncols, int nsplit, const float *__restrict__ partial, float *__restrict__ out,
                               int accumulate) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ncols; j += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < nsplit; s++) acc += partial[(int64_t)s * ncols + j];
    out[j] = accumulate ? out[j] + acc : acc;
  }
}

// root_off[r] = #graphs whose root row is < r (r = 0..N): the roots seeded at row r are
// root_perm[root_off[r] .. root_off[r+1]).
__global__ void k_root_off(int N, int G, const int32_t *__restrict__ root_row, const int32_t *__restrict__ root_perm,
                           int32_t *__restrict__ root_off) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= N; r += stride) {
    int lo = 0, hi = G;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (root_row[root_perm[mid]] < r) lo = mid + 1; else hi = mid; }
    root_off[r] = lo;
  }
}

// ---------------------------------------------------------------- embedding backward
// For each distinct-token segment of leaf_perm (rows ascending): dE[tok] += sum over its
// rows of dh(row), dh(row) = roots seeded at row + sum_{e in cons(row)} dA[e].
// One 128-thread block per segment, VEC columns per thread; deterministic order.
// dE must be pre-zeroed or hold the accumulation base (absent tokens are untouched).
template <int VEC>
__global__ void __launch_bounds__(128) k_embed_bwd(int S, int n_tok_segs, const int32_t *__restrict__ tok_seg,
                                                   const int32_t *__restrict__ leaf_perm,
                                                   const int32_t *__restrict__ leaf_token,
                                                   const int32_t *__restrict__ cons_off,
                                                   const int32_t *__restrict__ cons_edge,
                                                   const int32_t *__restrict__ root_off,
                                                   const int32_t *__restrict__ root_perm, int G,
                                                   const float *__restrict__ dh_root, const float *__restrict__ dA,
                                                   float *__restrict__ dE) {
  using IF = VecIO<float, VEC>;
  for (int64_t s = blockIdx.x; s < n_tok_segs; s += gridDim.x) {
    const int a = tok_seg[s], b = tok_seg[s + 1];
    const int tok = leaf_token[leaf_perm[a]];
    float *de = dE + (int64_t)tok * S;
    for (int j = threadIdx.x * VEC; j < S; j += blockDim.x * VEC) {
      float acc[VEC], t[VEC];
      IF::ld(de + j, acc);
      for (int q = a; q < b; q++) {
        const int r = leaf_perm[q];
        const int k1 = root_off[r + 1];
        for (int k = root_off[r]; k < k1; k++) {
          IF::ld(dh_root + (int64_t)root_perm[k] * S + j, t);
#pragma unroll
          for (int u = 0; u < VEC; u++) acc[u] += t[u];
        }
        const int e1 = cons_off[r + 1];
        for (int e = cons_off[r]; e < e1; e++) {
          IF::ld(dA + (int64_t)cons_edge[e] * S + j, t);
#pragma unroll
          for (int u = 0; u < VEC; u++) acc[u] += t[u];
        }
      }
      IF::st(de + j, acc);
    }
  }
}

// ---- pieces: segment s has ceil(len/P) pieces; piece k covers sorted leaves
// [a_s + kP, min(b_s, a_s + (k+1)P)). Single-piece segments add straight into dE; the
// pieces of longer segments write partials that k_embed_pieces_final sums in order.
__global__ void k_embed_piece_cnt(int n_tok_segs, const int32_t *__restrict__ tok_seg, int32_t *__restrict__ cnt) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_tok_segs; s += stride)
    cnt[s] = (int)cdiv(tok_seg[s + 1] - tok_seg[s], kEmbedPiece);
}

// Per piece: first the piece's source rows are resolved into shared memory in parallel (one
// thread per leaf: its seeded roots, then its consumer edges, ascending, i.e. the order the
// sums take), so the column loop streams independent row loads (UNR in flight per thread)
// instead of walking a leaf -> row -> cons_off -> cons_edge -> dA chain per leaf.
// Source encoding: >= 0 an edge row of dA (or, with dX, the leaf's own dX row); < 0 the
// seeded root -(g + 1) of dh_root.
constexpr int kPieceSrc = 512;  // sources held per pass (a piece has <= kEmbedPiece leaves)
// piece -> segment map (so a piece finds its segment with one load, not a binary search)
__global__ void k_embed_piece_seg(int n_tok_segs, const int32_t *__restrict__ piece_off, int32_t *__restrict__ seg) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_tok_segs; s += stride)
    for (int k = piece_off[s]; k < piece_off[s + 1]; k++) seg[k] = (int)s;
}

template <int VEC, typename TA>
__global__ void __launch_bounds__(128) k_embed_pieces(int S, int n_tok_segs, int n_pieces,
                                                      const int32_t *__restrict__ tok_seg,
                                                      const int32_t *__restrict__ piece_off,
                                                      const int32_t *__restrict__ piece_seg,
                                                      const int32_t *__restrict__ leaf_perm,
                                                      const int32_t *__restrict__ leaf_token,
                                                      const int32_t *__restrict__ cons_off,
                                                      const int32_t *__restrict__ cons_edge,
                                                      const int32_t *__restrict__ root_off,
                                                      const int32_t *__restrict__ root_perm,
                                                      const float *__restrict__ dh_root, const TA *__restrict__ dA,
                                                      float *__restrict__ dE, float *__restrict__ partial,
                                                      const float *__restrict__ dX) {
  using IF = VecIO<float, VEC>;
  using IA = VecIO<TA, VEC>;
  __shared__ int src[kPieceSrc];
  __shared__ int cnt[kEmbedPiece + 1];
  const int total = piece_off[n_tok_segs];  // n_pieces is only a host-side upper bound
  for (int64_t p = blockIdx.x; p < n_pieces && p < total; p += gridDim.x) {
    const int s = piece_seg[p];  // segment s with piece_off[s] <= p < piece_off[s+1]
    const int k = (int)(p - piece_off[s]);
    const int np = piece_off[s + 1] - piece_off[s];
    const int a = tok_seg[s] + k * kEmbedPiece, b = min(tok_seg[s + 1], a + kEmbedPiece);
    const int tok = leaf_token[leaf_perm[tok_seg[s]]];
    float *dst = np == 1 ? dE + (int64_t)tok * S : partial + p * (int64_t)S;
    // ---- resolve the sources (thread t <-> leaf a + t)
    const int t = threadIdx.x, nleaf = b - a;
    int r = -1, r0 = 0, r1 = 0, e0 = 0, e1 = 0;
    if (t < nleaf) {
      r = leaf_perm[a + t];
      if (!dX) { r0 = root_off[r]; r1 = root_off[r + 1]; e0 = cons_off[r]; e1 = cons_off[r + 1]; }
      cnt[t] = dX ? 1 : (r1 - r0) + (e1 - e0);
    }
    __syncthreads();
    if (t == 0) {  // exclusive prefix over <= 64 counts
      int acc = 0;
      for (int i = 0; i < nleaf; i++) { const int c = cnt[i]; cnt[i] = acc; acc += c; }
      cnt[nleaf] = acc;
    }
    __syncthreads();
    const int nsrc = cnt[nleaf];
    if (nsrc <= kPieceSrc && t < nleaf) {
      int o = cnt[t];
      if (dX) src[o] = r;
      else {
        for (int q = r0; q < r1; q++) src[o++] = -(root_perm[q] + 1);
        for (int e = e0; e < e1; e++) src[o++] = cons_edge[e];
      }
    }
    __syncthreads();
    const float *xsrc = dX;
    if (nsrc <= kPieceSrc) {
      for (int j = threadIdx.x * VEC; j < S; j += blockDim.x * VEC) {
        float acc[VEC];
        if (np == 1) IF::ld(dst + j, acc);
        else {
#pragma unroll
          for (int u = 0; u < VEC; u++) acc[u] = 0.f;
        }
        constexpr int UNR = 4;
        int i = 0;
        for (; i + UNR <= nsrc; i += UNR) {
          float t4[UNR][VEC];
#pragma unroll
          for (int q = 0; q < UNR; q++) {
            const int sv = src[i + q];
            if (xsrc) IF::ld(xsrc + (int64_t)sv * S + j, t4[q]);
            else if (sv >= 0) IA::ld(dA + (int64_t)sv * S + j, t4[q]);
            else IF::ld(dh_root + (int64_t)(-sv - 1) * S + j, t4[q]);
          }
#pragma unroll
          for (int q = 0; q < UNR; q++)
#pragma unroll
            for (int u = 0; u < VEC; u++) acc[u] += t4[q][u];
        }
        for (; i < nsrc; i++) {
          float tv[VEC];
          const int sv = src[i];
          if (xsrc) IF::ld(xsrc + (int64_t)sv * S + j, tv);
          else if (sv >= 0) IA::ld(dA + (int64_t)sv * S + j, tv);
          else IF::ld(dh_root + (int64_t)(-sv - 1) * S + j, tv);
#pragma unroll
          for (int u = 0; u < VEC; u++) acc[u] += tv[u];
        }
        IF::st(dst + j, acc);
      }
      __syncthreads();  // src / cnt reused by the next piece
      continue;
    }
    // (more sources than the shared list holds: wide DAG fan-out) walk the leaves directly
    for (int j = threadIdx.x * VEC; j < S; j += blockDim.x * VEC) {
      float acc[VEC], tv[VEC];
      if (np == 1) IF::ld(dst + j, acc);
      else {
#pragma unroll
        for (int u = 0; u < VEC; u++) acc[u] = 0.f;
      }
      for (int q = a; q < b; q++) {
        const int rr = leaf_perm[q];
        const int k1 = root_off[rr + 1];
        for (int kk = root_off[rr]; kk < k1; kk++) {
          IF::ld(dh_root + (int64_t)root_perm[kk] * S + j, tv);
#pragma unroll
          for (int u = 0; u < VEC; u++) acc[u] += tv[u];
        }
        const int ee = cons_off[rr + 1];
        for (int e = cons_off[rr]; e < ee; e++) {
          IA::ld(dA + (int64_t)cons_edge[e] * S + j, tv);
#pragma unroll
          for (int u = 0; u < VEC; u++) acc[u] += tv[u];
        }
      }
      IF::st(dst + j, acc);
    }
    __syncthreads();
  }
}

template <int VEC>
__global__ void __launch_bounds__(128) k_embed_pieces_final(int S, int n_tok_segs, const int32_t *__restrict__ tok_seg,
                                                            const int32_t *__restrict__ piece_off,
                                                            const int32_t *__restrict__ leaf_perm,
                                                            const int32_t *__restrict__ leaf_token,
                                                            const float *__restrict__ partial,
                                                            float *__restrict__ dE) {
  using IF = VecIO<float, VEC>;
  for (int64_t s = blockIdx.x; s < n_tok_segs; s += gridDim.x) {
    const int p0 = piece_off[s], p1 = piece_off[s + 1];
    if (p1 - p0 <= 1) continue;
    const int tok = leaf_token[leaf_perm[tok_seg[s]]];
    float *de = dE + (int64_t)tok * S;
    for (int j = threadIdx.x * VEC; j < S; j += blockDim.x * VEC) {
      float acc[VEC], t[VEC];
      IF::ld(de + j, acc);
      for (int p = p0; p < p1; p++) {
        IF::ld(partial + (int64_t)p * S + j, t);
#pragma unroll
        for (int u = 0; u < VEC; u++) acc[u] += t[u];
      }
      IF::st(de + j, acc);
    }
  }
}

// ---- sparse embedding-gradient exchange: the batch's distinct tokens
// (the rows of dE a step can touch), row packing and rank-ordered scatter-add
// rows[i] = token of the i-th token segment (ascending tokens: leaf_perm is sorted by token)
__global__ void k_touched_rows(int n_seg, const int32_t *__restrict__ tok_seg, const int32_t *__restrict__ leaf_perm,
                               const int32_t *__restrict__ leaf_token, int32_t *__restrict__ rows) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_seg; i += gridDim.x * blockDim.x)
    rows[i] = leaf_token[leaf_perm[tok_seg[i]]];
}
// dst[i][0..S) = src[rows[i]][0..S) (0 for rows[i] < 0: padding)
__global__ void k_gather_rows(const float *__restrict__ src, int64_t ld, const int32_t *__restrict__ rows, int n,
                              int S, float *__restrict__ dst) {
  const int64_t total = (int64_t)n * S, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int r = rows[i / S];
    dst[i] = r >= 0 ? src[(int64_t)r * ld + i % S] : 0.f;
  }
}
// dst[rows[i]][0..S) += src[i][0..S) (rows of one call distinct: no conflicts, no atomics;
// skipped for rows[i] < 0)
__global__ void k_scatter_add_rows(const float *__restrict__ src, const int32_t *__restrict__ rows, int n, int S,
                                   float *__restrict__ dst, int64_t ld) {
  const int64_t total = (int64_t)n * S, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int r = rows[i / S];
    if (r >= 0) dst[(int64_t)r * ld + i % S] += src[i];
  }
}

__global__ void k_sgd(float *p, const float *g, int64_t n, float lr, int v4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i0 = 0;
  if (v4) {  // 16-byte aligned: float4 body, scalar tail
    const int64_t n4 = n >> 2;
    for (int64_t i = t; i < n4; i += stride) {
      float4 a = reinterpret_cast<float4 *>(p)[i];
      const float4 b = __ldcs(reinterpret_cast<const float4 *>(g) + i);
      a.x -= lr * b.x; a.y -= lr * b.y; a.z -= lr * b.z; a.w -= lr * b.w;
      reinterpret_cast<float4 *>(p)[i] = a;
    }
    i0 = n4 << 2;
  }
  for (int64_t i = i0 + t; i < n; i += stride) p[i] -= lr * g[i];
}

__global__ void k_zero(uint32_t *p, int64_t n) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = 0u;
}

}  // namespace

// ================================================================= launchers
fold_status launch_embed_fwd(bool bf16, int r0, int r1, const int32_t *leaf_token, const float *E, int S, int ld,
                             void *H, float *C, const ScatterA *sc, cudaStream_t st) {
  if (r1 <= r0) return FOLD_OK;
  unsigned g = grid_cap(cdiv((int64_t)(r1 - r0) * 32, 256));
  ScatterA s0{};
  if (bf16)
    k_embed_fwd<__nv_bfloat16><<<g, 256, 0, st>>>(r0, r1, leaf_token, E, S, ld, (__nv_bfloat16 *)H, C,
                                                  sc ? *sc : s0, sc ? 1 : 0);
  else k_embed_fwd<float><<<g, 256, 0, st>>>(r0, r1, leaf_token, E, S, ld, (float *)H, C, s0, 0);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_cell_fwd_simt(int cell, int r0, int r1, const int32_t *gather, int S, int ld, const float *U,
                                 const float *b, float *H, float *C, float *Gact, int ld_g, int nl, cudaStream_t st) {
  if (r1 <= r0) return FOLD_OK;
  dim3 grid((unsigned)cdiv(r1 - r0, 32), (unsigned)cdiv(S, 32));
  if (cell == FOLD_CELL_TREELSTM)
    k_cell_fwd_simt<5><<<grid, 256, 0, st>>>(r0, r1, gather, S, ld, U, b, H, C, Gact, ld_g, nl);
  else
    k_cell_fwd_simt<1><<<grid, 256, 0, st>>>(r0, r1, gather, S, ld, U, b, H, C, Gact, ld_g, nl);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_root_out(bool bf16, int G, int S, int ld, int nl, const int32_t *root_row, const void *H,
                            const float *C, float *h_root, float *c_root, const ScatterA *sc, cudaStream_t st) {
  ScatterA s0{};
  if (G <= 0 || (!h_root && !c_root)) return FOLD_OK;
  unsigned g = grid_cap(cdiv((int64_t)G * S, 256));
  if (bf16) k_root_out<__nv_bfloat16><<<g, 256, 0, st>>>(G, S, ld, nl, root_row, (const __nv_bfloat16 *)H, C, h_root, c_root,
                                                                sc ? *sc : s0, sc ? 1 : 0);
  else k_root_out<float><<<g, 256, 0, st>>>(G, S, ld, nl, root_row, (const float *)H, C, h_root, c_root, s0, 0);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_cell_bwd_pw(bool bf16, int cell, int r0, int r1, int nl, int S, int ld, int ld_g,
                               const int32_t *cons_off, const int32_t *cons_edge, const int32_t *root_off,
                               const int32_t *root_perm, int G, const float *dh_root, const float *dc_root,
                               const int32_t *gather, const void *Gact, const float *C, const float *dA, float *dCe,
                               void *dZ, int ld_z, cudaStream_t st, const int32_t *root_row, const float *dh_node,
                               bool leaf_c) {
  if (r1 <= r0) return FOLD_OK;
  const int vec = (S & 3) == 0 ? 4 : 1;
  unsigned g = grid_cap(cdiv((int64_t)(r1 - r0) * cdiv(S, 32 * vec) * 32, 256));
#define PW_ARGS r0, r1, nl, S, ld, ld_g, cons_off, cons_edge, root_off, root_perm, G, dh_root, dc_root, gather
#define PW_LAUNCH(T, GT, VEC) \
  k_cell_bwd_pw<T, GT, VEC><<<g, 256, 0, st>>>(PW_ARGS, (const T *)Gact, C, dA, dCe, (T *)dZ, ld_z, root_row, \
                                               dh_node, leaf_c ? 0 : nl)
  const bool v4 = (S & 3) == 0;
  const bool lstm = cell == FOLD_CELL_TREELSTM;
  if (bf16) {
    if (lstm) { if (v4) PW_LAUNCH(__nv_bfloat16, 5, 4); else PW_LAUNCH(__nv_bfloat16, 5, 1); }
    else { if (v4) PW_LAUNCH(__nv_bfloat16, 1, 4); else PW_LAUNCH(__nv_bfloat16, 1, 1); }
  } else {
    if (lstm) { if (v4) PW_LAUNCH(float, 5, 4); else PW_LAUNCH(float, 5, 1); }
    else { if (v4) PW_LAUNCH(float, 1, 4); else PW_LAUNCH(float, 1, 1); }
  }
#undef PW_LAUNCH
#undef PW_ARGS
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_gemm_dA_simt(int M, int S, int gates, const float *dZ, int ld_z, const float *U, float *dA,
                                cudaStream_t st) {
  if (M <= 0) return FOLD_OK;
  dim3 grid((unsigned)cdiv(2 * S, 64), (unsigned)cdiv(M, 64));
  k_gemm_dA_simt<<<grid, 256, 0, st>>>(M, 2 * S, gates * S, dZ, ld_z, U, 2 * S, dA, 2 * S);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_gemm_dU_simt(int n_cells, int nl, int S, int gates, const float *dZ, int ld_z,
                                const int32_t *gather, const float *H, int ld, float *dU, int accumulate,
                                cudaStream_t st) {
  dim3 grid((unsigned)cdiv(2 * S, 64), (unsigned)cdiv(gates * S, 64));
  k_gemm_dU_simt<<<grid, 256, 0, st>>>(n_cells, nl, S, gates * S, dZ, ld_z, gather, H, ld, dU, accumulate);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_colsum(bool bf16, int n_rows, int ncols, const void *dZ, int ld_z, float *partial, int nsplit,
                          float *db, int accumulate, cudaStream_t st) {
  const bool v8 = (ncols & 7) == 0 && (ld_z & 7) == 0;
  const int vec = v8 ? 8 : 1;
  dim3 grid((unsigned)cdiv(cdiv(ncols, vec), 256), (unsigned)nsplit);
  if (bf16) {
    if (v8) k_colsum_partial<__nv_bfloat16, 8><<<grid, 256, 0, st>>>(n_rows, ncols, (const __nv_bfloat16 *)dZ, ld_z, nsplit, partial);
    else k_colsum_partial<__nv_bfloat16, 1><<<grid, 256, 0, st>>>(n_rows, ncols, (const __nv_bfloat16 *)dZ, ld_z, nsplit, partial);
  } else {
    if (v8) k_colsum_partial<float, 8><<<grid, 256, 0, st>>>(n_rows, ncols, (const float *)dZ, ld_z, nsplit, partial);
    else k_colsum_partial<float, 1><<<grid, 256, 0, st>>>(n_rows, ncols, (const float *)dZ, ld_z, nsplit, partial);
  }
  FOLD_LAUNCH_CHECK();
  k_colsum_final<<<(unsigned)cdiv(ncols, 256), 256, 0, st>>>(ncols, nsplit, partial, db, accumulate);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_root_off(int N, int G, const int32_t *root_row, const int32_t *root_perm, int32_t *root_off,
                            cudaStream_t st) {
  k_root_off<<<grid_cap(cdiv((int64_t)N + 1, 256)), 256, 0, st>>>(N, G, root_row, root_perm, root_off);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_embed_bwd(int S, int nl, int n_tok_segs, const int32_t *tok_seg, const int32_t *leaf_perm,
                             const int32_t *leaf_token, const int32_t *cons_off,
                             const int32_t *cons_edge, const int32_t *root_off, const int32_t *root_perm, int G,
                             const float *dh_root, const float *dA, float *dE, cudaStream_t st) {
  (void)nl;
  if (n_tok_segs <= 0) return FOLD_OK;
  unsigned g = grid_cap(n_tok_segs);
  if ((S & 3) == 0)
    k_embed_bwd<4><<<g, 128, 0, st>>>(S, n_tok_segs, tok_seg, leaf_perm, leaf_token, cons_off, cons_edge, root_off,
                                      root_perm, G, dh_root, dA, dE);
  else
    k_embed_bwd<1><<<g, 128, 0, st>>>(S, n_tok_segs, tok_seg, leaf_perm, leaf_token, cons_off, cons_edge, root_off,
                                      root_perm, G, dh_root, dA, dE);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_embed_bwd_pieces(int S, int n_leaves, int n_tok_segs, const int32_t *tok_seg,
                                    const int32_t *leaf_perm, const int32_t *leaf_token, const int32_t *cons_off,
                                    const int32_t *cons_edge, const int32_t *root_off, const int32_t *root_perm,
                                    const float *dh_root, const void *dA, bool dA_bf16, float *dE,
                                    const EmbedBwdWs &w, cudaStream_t st, const float *dX) {
  (void)n_leaves;
  if (n_tok_segs <= 0) return FOLD_OK;
  k_embed_piece_cnt<<<grid_cap(cdiv(n_tok_segs, 256)), 256, 0, st>>>(n_tok_segs, tok_seg, w.piece_cnt);
  FOLD_LAUNCH_CHECK();
  // piece_off[0..n_tok_segs] (the total lands in piece_off[n_tok_segs] via a zero tail)
  FOLD_CUDA_TRY(cudaMemsetAsync(w.piece_cnt + n_tok_segs, 0, sizeof(int32_t), st));
  FOLD_TRY(scan_exclusive(w.piece_cnt, w.piece_off, (int64_t)n_tok_segs + 1, w.scan_sums, nullptr, st));
  k_embed_piece_seg<<<grid_cap(cdiv(n_tok_segs, 256)), 256, 0, st>>>(n_tok_segs, w.piece_off, w.piece_seg);
  FOLD_LAUNCH_CHECK();
  // upper bound on pieces (host-side, no sync): sum ceil(len/P) <= n_leaves/P + n_tok_segs
  const int max_pieces = n_leaves / kEmbedPiece + n_tok_segs;
  const unsigned g = grid_cap(max_pieces);
  const bool v4 = (S & 3) == 0;
#define EP_ARGS(T) S, n_tok_segs, max_pieces, tok_seg, w.piece_off, w.piece_seg, leaf_perm, leaf_token, cons_off, cons_edge, \
                root_off, root_perm, dh_root, (const T *)dA, dE, w.partial, dX
  if (dA_bf16) {  // the fused tree backward stores leaf edges' dA in bf16
    if (v4) k_embed_pieces<4, __nv_bfloat16><<<g, 128, 0, st>>>(EP_ARGS(__nv_bfloat16));
    else k_embed_pieces<1, __nv_bfloat16><<<g, 128, 0, st>>>(EP_ARGS(__nv_bfloat16));
  } else {
    if (v4) k_embed_pieces<4, float><<<g, 128, 0, st>>>(EP_ARGS(float));
    else k_embed_pieces<1, float><<<g, 128, 0, st>>>(EP_ARGS(float));
  }
#undef EP_ARGS
  FOLD_LAUNCH_CHECK();
  const unsigned g2 = grid_cap(n_tok_segs);
  if (v4) k_embed_pieces_final<4><<<g2, 128, 0, st>>>(S, n_tok_segs, tok_seg, w.piece_off, leaf_perm, leaf_token,
                                                     w.partial, dE);
  else k_embed_pieces_final<1><<<g2, 128, 0, st>>>(S, n_tok_segs, tok_seg, w.piece_off, leaf_perm, leaf_token,
                                                  w.partial, dE);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_touched_rows(int n_seg, const int32_t *tok_seg, const int32_t *leaf_perm,
                                const int32_t *leaf_token, int32_t *rows, cudaStream_t st) {
  if (n_seg <= 0) return FOLD_OK;
  k_touched_rows<<<grid_cap(cdiv(n_seg, 256)), 256, 0, st>>>(n_seg, tok_seg, leaf_perm, leaf_token, rows);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}
fold_status launch_gather_rows(const float *src, int64_t ld, const int32_t *rows, int n, int S, float *dst,
                               cudaStream_t st) {
  if (n <= 0 || S <= 0) return FOLD_OK;
  k_gather_rows<<<grid_cap(cdiv((int64_t)n * S, 256)), 256, 0, st>>>(src, ld, rows, n, S, dst);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}
fold_status launch_scatter_add_rows(const float *src, const int32_t *rows, int n, int S, float *dst, int64_t ld,
                                    cudaStream_t st) {
  if (n <= 0 || S <= 0) return FOLD_OK;
  k_scatter_add_rows<<<grid_cap(cdiv((int64_t)n * S, 256)), 256, 0, st>>>(src, rows, n, S, dst, ld);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_sgd(float *p, const float *g, int64_t n, float lr, cudaStream_t st) {
  if (n <= 0) return FOLD_OK;
  const int v4 = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g)) & 15) == 0;
  k_sgd<<<grid_cap(cdiv(v4 ? cdiv(n, 4) : n, 256)), 256, 0, st>>>(p, g, n, lr, v4);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_zero(void *p, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return FOLD_OK;
  int64_t n = (int64_t)(bytes / 4);
  k_zero<<<grid_cap(cdiv(n, 256)), 256, 0, st>>>((uint32_t *)p, n);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

}  // namespace fold

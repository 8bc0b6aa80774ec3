// sched.cu — GPU scheduler for dynamic batching (§2, L40-44).
//
// fold_schedule = validate -> consumer lists -> level-synchronous depth frontier
// (one cooperative kernel, grid barrier per depth) -> stable LSD radix sort on
// key = 2*depth + op (ties by node id) -> offsets / rank / gather vectors ->
// consumer CSR (stable sort of cell edges by child row) -> leaves by token ->
// roots. One blocking D2H at the end. All kernels are integer work, HBM/latency bound.
#include <climits>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace fold {

thread_local int64_t g_launches = 0;

namespace {

// flags[] slots (int32) in the workspace header
enum {
  F_ERR0 = 0,  // F_ERR0 + k for the k-th error class (min offending id, INT_MAX = none)
  F_NLEAVES = 8, F_MAXDEPTH = 9, F_NSEG = 10,
  F_QCNT = 12,  // 3 rotating frontier counters 12..14
  F_BAR = 16,   // grid barrier count, generation (16, 17)
  F_NFLAGS = 64
};
enum { E_CHILD = 0, E_OP = 1, E_ARITY = 2, E_TOKEN = 3, E_ROOT = 4, E_CYCLE = 5, E_NCLASS = 6 };
const fold_status kErrStatus[E_NCLASS] = {FOLD_E_CHILD_RANGE, FOLD_E_OP_RANGE, FOLD_E_ARITY,
                                         FOLD_E_TOKEN_RANGE, FOLD_E_ROOT_RANGE, FOLD_E_CYCLE};

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096
constexpr int kScanThreads = 1024;
constexpr int kScanTile = kScanThreads * 4;
constexpr int kPendingInvalid = 0x3fffffff;

inline int bits_for(int64_t maxval) {  // #bits to represent values in [0, maxval]
  int b = 0;
  while (b < 31 && (int64_t(1) << b) <= maxval) b++;
  return b < 1 ? 1 : b;
}

// ---------------------------------------------------------------- workspace layout
struct SchedWs {
  int32_t *flags, *ncons, *pcons_off, *pcons, *pending, *q0, *q1;
  uint32_t *ka, *kb;
  int32_t *va, *vb;
  int32_t *hist, *scan_sums, *seg_flag, *seg_scan;
  int nb;        // radix tiles for the largest sort (2N elements)
  size_t bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

SchedWs sched_ws_layout(void *base, int64_t N, int64_t G) {
  SchedWs w{};
  int64_t M = 2 * N > G ? 2 * N : G;
  if (M < 1) M = 1;
  w.nb = (int)cdiv(M, kSortTile);
  int64_t scan_len_max = (int64_t)256 * w.nb;
  if (scan_len_max < N + 1) scan_len_max = N + 1;
  int64_t nsums = cdiv(scan_len_max, kScanTile) + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
  size_t o_flags = take(F_NFLAGS * 4);
  size_t o_ncons = take((N + 1) * 4), o_pco = take((N + 2) * 4), o_pc = take((2 * N + 1) * 4);
  size_t o_pend = take((N + 1) * 4), o_q0 = take((N + 1) * 4), o_q1 = take((N + 1) * 4);
  size_t o_ka = take((M + 1) * 4), o_kb = take((M + 1) * 4), o_va = take((M + 1) * 4), o_vb = take((M + 1) * 4);
  size_t o_hist = take(scan_len_max * 4 + 4), o_sums = take(nsums * 4 * 2);
  size_t o_sf = take((N + 1) * 4), o_ss = take((N + 2) * 4);
  w.bytes = off;
  if (base) {
    char *b = (char *)base;
    w.flags = (int32_t *)(b + o_flags); w.ncons = (int32_t *)(b + o_ncons);
    w.pcons_off = (int32_t *)(b + o_pco); w.pcons = (int32_t *)(b + o_pc);
    w.pending = (int32_t *)(b + o_pend); w.q0 = (int32_t *)(b + o_q0); w.q1 = (int32_t *)(b + o_q1);
    w.ka = (uint32_t *)(b + o_ka); w.kb = (uint32_t *)(b + o_kb);
    w.va = (int32_t *)(b + o_va); w.vb = (int32_t *)(b + o_vb);
    w.hist = (int32_t *)(b + o_hist); w.scan_sums = (int32_t *)(b + o_sums);
    w.seg_flag = (int32_t *)(b + o_sf); w.seg_scan = (int32_t *)(b + o_ss);
  }
  return w;
}

// ---------------------------------------------------------------- scan (exclusive, int32)
__device__ __forceinline__ int block_excl_scan(int v, int *smem_warp, int *total) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < nw ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) smem_warp[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  int warp_excl = warp > 0 ? smem_warp[warp - 1] : 0;
  if (total) *total = smem_warp[nw - 1];
  int r = warp_excl + x - v;
  __syncthreads();
  return r;
}

// phase 1: per-tile exclusive scan into out, tile totals into sums[tile]
__global__ void k_scan_tiles(const int32_t *in, int32_t *out, int64_t n, int32_t *sums) {
  __shared__ int sw[32];
  int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 4;
  int v[4], s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) { v[i] = (base + i < n) ? in[base + i] : 0; s += v[i]; }
  int tot;
  int ex = block_excl_scan(s, sw, &tot);
#pragma unroll
  for (int i = 0; i < 4; i++) { if (base + i < n) out[base + i] = ex; ex += v[i]; }
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// phase 2: exclusive scan of the tile totals (single block, loops with a carry);
// writes the grand total to *total (if non-null)
__global__ void k_scan_sums(int32_t *sums, int64_t n, int32_t *total) {
  __shared__ int sw[32];
  int carry = 0;
  for (int64_t b = 0; b < n; b += blockDim.x) {
    int64_t i = b + threadIdx.x;
    int v = i < n ? sums[i] : 0;
    int tot;
    int ex = block_excl_scan(v, sw, &tot);
    if (i < n) sums[i] = ex + carry;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_scan_add(int32_t *out, int64_t n, const int32_t *sums) {
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int add = sums[blockIdx.x];
  for (int i = threadIdx.x; i < kScanTile; i += blockDim.x)
    if (base + i < n) out[base + i] += add;
}

// single-block exclusive scan for small arrays (one launch): 1024 threads x 16 items
constexpr int kSmallScan = kScanThreads * 16;
__global__ void k_scan_small(const int32_t *in, int32_t *out, int n, int32_t *total) {
  __shared__ int sw[32];
  int v[16], sum = 0;
  const int base = threadIdx.x * 16;
#pragma unroll
  for (int i = 0; i < 16; i++) { v[i] = base + i < n ? in[base + i] : 0; sum += v[i]; }
  int tot;
  int ex = block_excl_scan(sum, sw, &tot);
#pragma unroll
  for (int i = 0; i < 16; i++) { if (base + i < n) out[base + i] = ex; ex += v[i]; }
  if (threadIdx.x == 0 && total) *total = tot;
}

fold_status excl_scan(const int32_t *in, int32_t *out, int64_t n, int32_t *sums, int32_t *total,
                      cudaStream_t st) {
  if (n <= 0) return FOLD_OK;
  if (n <= kSmallScan) {
    k_scan_small<<<1, kScanThreads, 0, st>>>(in, out, (int)n, total);
    FOLD_LAUNCH_CHECK();
    return FOLD_OK;
  }
  int64_t nt = cdiv(n, kScanTile);
  k_scan_tiles<<<(unsigned)nt, kScanThreads, 0, st>>>(in, out, n, sums);
  FOLD_LAUNCH_CHECK();
  k_scan_sums<<<1, kScanThreads, 0, st>>>(sums, nt, total);
  FOLD_LAUNCH_CHECK();
  k_scan_add<<<(unsigned)nt, 256, 0, st>>>(out, n, sums);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

// ---------------------------------------------------------------- stable LSD radix sort
// Sorts (key, val) pairs by key, stable, count read on device (*d_n <= n_max).
__global__ void k_rs_hist(const uint32_t *keys, const int32_t *d_n, int shift, int32_t *hist, int nb) {
  __shared__ int h[256];
  int n = *d_n;
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += kSortThreads) {
    int64_t idx = base + i;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

__global__ void k_rs_scatter(const uint32_t *kin, const int32_t *vin, const int32_t *d_n, int shift,
                             const int32_t *hist_scan, int nb, uint32_t *kout, int32_t *vout) {
  __shared__ int run[256];
  __shared__ int wcnt[kSortThreads / 32][257];
  __shared__ int base[256];
  int n = *d_n;
  int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  base[tid] = hist_scan[(int64_t)tid * nb + blockIdx.x];
  run[tid] = 0;
  for (int w = 0; w < kSortThreads / 32; w++) wcnt[w][tid] = 0;
  __syncthreads();
  int64_t tile0 = (int64_t)blockIdx.x * kSortTile;
  if (tile0 >= n) return;
  for (int round = 0; round < kSortItems; round++) {
    int64_t idx = tile0 + (int64_t)round * kSortThreads + tid;
    bool valid = idx < n;
    uint32_t k = valid ? kin[idx] : 0u;
    int v = valid ? vin[idx] : 0;
    int d = valid ? (int)((k >> shift) & 255u) : 256;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int lrank = __popc(peers & lanemask_lt());
    if (lrank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      int pre = 0;
      for (int w = 0; w < warp; w++) pre += wcnt[w][d];
      int pos = base[d] + run[d] + pre + lrank;
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    {
      int s = 0;
#pragma unroll
      for (int w = 0; w < kSortThreads / 32; w++) { s += wcnt[w][tid]; wcnt[w][tid] = 0; }
      run[tid] += s;
      if (tid == 0) for (int w = 0; w < kSortThreads / 32; w++) wcnt[w][256] = 0;
    }
    __syncthreads();
    if (tile0 + (int64_t)(round + 1) * kSortThreads >= n) break;
  }
}

// Sorts (ws.ka, ws.va) with *d_n valid entries by the low `nbits` bits of the keys.
// Result pointers returned in *kres / *vres (either the a or b buffers).
fold_status radix_sort(SchedWs &w, const int32_t *d_n, int64_t n_max, int nbits, uint32_t **kres,
                       int32_t **vres, cudaStream_t st) {
  uint32_t *ki = w.ka, *ko = w.kb;
  int32_t *vi = w.va, *vo = w.vb;
  int nb = (int)cdiv(n_max < 1 ? 1 : n_max, kSortTile);
  for (int shift = 0; shift < nbits; shift += 8) {
    k_rs_hist<<<nb, kSortThreads, 0, st>>>(ki, d_n, shift, w.hist, nb);
    FOLD_LAUNCH_CHECK();
    FOLD_TRY(excl_scan(w.hist, w.hist, (int64_t)256 * nb, w.scan_sums, nullptr, st));
    k_rs_scatter<<<nb, kSortThreads, 0, st>>>(ki, vi, d_n, shift, w.hist, nb, ko, vo);
    FOLD_LAUNCH_CHECK();
    uint32_t *tk = ki; ki = ko; ko = tk;
    int32_t *tv = vi; vi = vo; vo = tv;
  }
  *kres = ki;
  *vres = vi;
  return FOLD_OK;
}

// ---------------------------------------------------------------- validation / lists
__global__ void k_validate(int N, int G, int V, const int32_t *op, const int32_t *child,
                           const int32_t *token, const int32_t *root, int32_t *flags,
                           int32_t *ncons, int32_t *pending) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    int n = (int)i;
    int o = op[n], c0 = child[2 * n], c1 = child[2 * n + 1];
    bool crange = (c0 < -1 || c0 >= N || c1 < -1 || c1 >= N);
    if (crange) atomicMin(&flags[F_ERR0 + E_CHILD], n);
    bool orange = (o != FOLD_OP_EMBED && o != FOLD_OP_CELL);
    if (orange) atomicMin(&flags[F_ERR0 + E_OP], n);
    bool ar_ok = (o == FOLD_OP_EMBED) ? (c0 == -1 && c1 == -1) : (c0 >= 0 && c1 >= 0);
    if (!ar_ok) atomicMin(&flags[F_ERR0 + E_ARITY], n);
    if (o == FOLD_OP_EMBED && (token[n] < 0 || token[n] >= V)) atomicMin(&flags[F_ERR0 + E_TOKEN], n);
    bool good_cell = (o == FOLD_OP_CELL) && !crange && c0 >= 0 && c1 >= 0;
    if (good_cell) { atomicAdd(&ncons[c0], 1); atomicAdd(&ncons[c1], 1); }
    pending[n] = (o == FOLD_OP_CELL) ? (good_cell ? 2 : kPendingInvalid) : 0;
  }
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += stride)
    if (root[g] < 0 || root[g] >= N) atomicMin(&flags[F_ERR0 + E_ROOT], (int)g);
}

// parents list (unordered within a node) + initial frontier (EMBED nodes, depth 1)
__global__ void k_fill_parents(int N, const int32_t *op, const int32_t *child, const int32_t *pcons_off,
                               int32_t *fillc, int32_t *pcons, int32_t *depth, int32_t *q0,
                               int32_t *flags) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t nloop = cdiv(N, stride) * stride;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloop; i += stride) {
    bool in = i < N;
    int n = (int)i;
    bool leaf = false;
    if (in) {
      int o = op[n], c0 = child[2 * n], c1 = child[2 * n + 1];
      bool good_cell = (o == FOLD_OP_CELL) && c0 >= 0 && c0 < N && c1 >= 0 && c1 < N;
      if (good_cell) {
        pcons[pcons_off[c0] + atomicAdd(&fillc[c0], 1)] = n;
        pcons[pcons_off[c1] + atomicAdd(&fillc[c1], 1)] = n;
      }
      leaf = (o == FOLD_OP_EMBED);
      depth[n] = leaf ? 1 : -1;
    }
    int slot = warp_push(&flags[F_QCNT + 1], leaf);
    if (leaf) q0[slot] = n;
    int nl = __popc(__ballot_sync(0xffffffffu, leaf));
    if ((threadIdx.x & 31) == 0 && nl) atomicAdd(&flags[F_NLEAVES], nl);
  }
}

__device__ __forceinline__ int ld_volatile(const int32_t *p) { return *(volatile const int32_t *)p; }

__device__ void grid_barrier(int32_t *flags) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile int32_t *gen = &flags[F_BAR + 1];
    int g = *gen;
    __threadfence();
    if (atomicAdd(&flags[F_BAR], 1) == (int)gridDim.x - 1) {
      atomicExch(&flags[F_BAR], 0);
      __threadfence();
      atomicAdd((int32_t *)gen, 1);
    } else {
      while (*gen == g) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

// Level-synchronous depth propagation. Frontier_1 = EMBED nodes; a
// parent whose last pending child finishes at level L gets depth L+1. One grid
// barrier per level; must be launched cooperatively (all blocks co-resident).
__global__ void k_depth_frontier(const int32_t *pcons_off, const int32_t *pcons, int32_t *pending,
                                 int32_t *depth, int32_t *q0, int32_t *q1, int32_t *flags) {
  int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int L = 1;
  for (;; L++) {
    int ncur = ld_volatile(&flags[F_QCNT + (L % 3)]);
    if (ncur == 0) break;
    const int32_t *cur = (L & 1) ? q0 : q1;
    int32_t *nxt = (L & 1) ? q1 : q0;
    if (gtid == 0) flags[F_QCNT + ((L + 2) % 3)] = 0;
    int64_t nloop = cdiv(ncur, stride) * stride;
    for (int64_t i = gtid; i < nloop; i += stride) {
      bool in = i < ncur;
      int x = in ? ld_volatile(&cur[i]) : 0;
      int e0 = in ? pcons_off[x] : 0, e1 = in ? pcons_off[x + 1] : 0;
      for (int j = 0; __any_sync(0xffffffffu, e0 + j < e1); j++) {
        bool act = false;
        int p = 0;
        if (e0 + j < e1) {
          p = pcons[e0 + j];
          act = (atomicSub(&pending[p], 1) == 1);
          if (act) depth[p] = L + 1;
        }
        int slot = warp_push(&flags[F_QCNT + ((L + 1) % 3)], act);
        if (act) nxt[slot] = p;
      }
    }
    grid_barrier(flags);
  }
  if (gtid == 0) flags[F_MAXDEPTH] = L - 1;
}

__global__ void k_post_depth(int N, const int32_t *op, const int32_t *depth, int32_t *flags,
                             uint32_t *keys, int32_t *vals) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    int n = (int)i, d = depth[n];
    if (d < 0) atomicMin(&flags[F_ERR0 + E_CYCLE], n);
    keys[n] = (uint32_t)(2 * (d < 0 ? 0 : d) + (op[n] & 1));
    vals[n] = n;
  }
}

// perm/rank + group_off/level_off by binary search over the sorted keys
__global__ void k_perm_offsets(int N, const uint32_t *skeys, const int32_t *svals, const int32_t *flags,
                               int32_t *perm, int32_t *rank, int32_t *group_off, int32_t *level_off) {
  int D = flags[F_MAXDEPTH];
  int nk = 2 * (D + 1);
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    int n = svals[i];
    perm[i] = n;
    rank[n] = (int)i;
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nk; k += stride) {
    int lo = 0, hi = N;
    while (lo < hi) { int mid = (lo + hi) >> 1; if ((int)skeys[mid] < (int)k) lo = mid + 1; else hi = mid; }
    group_off[k] = lo;
    if ((k & 1) == 0) level_off[k >> 1] = lo;
  }
}

__global__ void k_gather(int N, const int32_t *op, const int32_t *child, const int32_t *perm,
                         const int32_t *rank, int32_t *gather) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
    int n = perm[r];
    int c0 = child[2 * n], c1 = child[2 * n + 1];
    bool cell = op[n] == FOLD_OP_CELL;
    // out-of-range children are reported by k_validate; never index with them
    gather[2 * r] = (cell && c0 >= 0 && c0 < N) ? rank[c0] : -1;
    gather[2 * r + 1] = (cell && c1 >= 0 && c1 < N) ? rank[c1] : -1;
  }
}

// cell edges e in [0, 2 n_cells): key = child row, val = e; count = 2 (N - n_leaves)
__global__ void k_cons_keys(int N, const int32_t *gather, int32_t *flags, int32_t *d_count,
                            uint32_t *keys, int32_t *vals) {
  int nl = flags[F_NLEAVES];
  int cnt = 2 * (N - nl);
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_count = cnt;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += stride) {
    keys[e] = (uint32_t)gather[2 * (int64_t)nl + e];
    vals[e] = (int)e;
  }
}

__global__ void k_cons_finish(int N, const uint32_t *skeys, const int32_t *svals, const int32_t *d_count,
                              int32_t *cons_off, int32_t *cons_edge) {
  int cnt = *d_count;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride)
    cons_edge[i] = svals[i];
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= N; r += stride) {
    int lo = 0, hi = cnt;
    while (lo < hi) { int mid = (lo + hi) >> 1; if ((int)skeys[mid] < (int)r) lo = mid + 1; else hi = mid; }
    cons_off[r] = lo;
  }
}

// leaves (rows [0, n_leaves)) keyed by token
__global__ void k_leaf_keys(const int32_t *token, const int32_t *perm, const int32_t *flags,
                            int32_t *d_count, uint32_t *keys, int32_t *vals, int32_t *leaf_token) {
  int nl = flags[F_NLEAVES];
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_count = nl;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += stride) {
    int t = token[perm[r]];
    keys[r] = (uint32_t)t;
    vals[r] = (int)r;
    leaf_token[r] = t;
  }
}

__global__ void k_seg_flags(int N, const uint32_t *skeys, const int32_t *svals, const int32_t *d_count,
                            int32_t *leaf_perm, int32_t *seg_flag) {
  int cnt = *d_count;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    bool in = i < cnt;
    if (in) leaf_perm[i] = svals[i];
    seg_flag[i] = (in && (i == 0 || skeys[i] != skeys[i - 1])) ? 1 : 0;
  }
}

__global__ void k_seg_write(int N, const int32_t *seg_flag, const int32_t *seg_scan, const int32_t *d_count,
                            const int32_t *flags, int32_t *tok_seg) {
  int cnt = *d_count;
  int nseg = flags[F_NSEG];
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride)
    if (seg_flag[i]) tok_seg[seg_scan[i]] = (int)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) tok_seg[nseg] = cnt;
}

__global__ void k_root_keys(int N, int G, const int32_t *root, const int32_t *rank, int32_t *root_row,
                            uint32_t *keys, int32_t *vals) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += stride) {
    int ro = root[g];
    int rr = (ro >= 0 && ro < N) ? rank[ro] : 0;  // invalid roots are reported by k_validate
    root_row[g] = rr;
    keys[g] = (uint32_t)rr;
    vals[g] = (int)g;
  }
}

// Stable sort of graph ids by root row for G <= 4096 in one block: bitonic sort of the
// unique composite keys (root_row << 32 | g), so ties keep ascending g.
constexpr int kSmallRoots = 4096;
__global__ void k_roots_small(int N, int G, const int32_t *root, const int32_t *rank, int32_t *root_row,
                              int32_t *root_perm) {
  __shared__ unsigned long long key[kSmallRoots];
  int n2 = 1;
  while (n2 < G) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    if (i < G) {
      int ro = root[i];
      int rr = (ro >= 0 && ro < N) ? rank[ro] : 0;  // invalid roots are reported by k_validate
      root_row[i] = rr;
      key[i] = ((unsigned long long)(unsigned)rr << 32) | (unsigned)i;
    } else {
      key[i] = ~0ull;
    }
  }
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          unsigned long long a = key[i], b = key[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) { key[i] = b; key[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < G; i += blockDim.x) root_perm[i] = (int32_t)(key[i] & 0xffffffffu);
}

__global__ void k_copy_i32(const int32_t *src, int32_t *dst, int64_t n) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

__global__ void k_init_flags(int32_t *flags, int N, int G) {
  int t = threadIdx.x;
  if (t < F_NFLAGS) flags[t] = (t < E_NCLASS) ? INT_MAX : (t == 20 ? N : (t == 23 ? G : 0));
}

inline unsigned grid_for(int64_t n, int threads = 256) {
  int64_t b = cdiv(n < 1 ? 1 : n, threads);
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)b;
}

}  // namespace

thread_local int32_t g_last_detail = -1;

// device-wide exclusive int32 scan for other translation units; `sums` needs
// scan_sums_count(n) entries
fold_status scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *sums, int32_t *total,
                           cudaStream_t st) {
  return excl_scan(in, out, n, sums, total, st);
}
int64_t scan_sums_count(int64_t n) { return cdiv(n < 1 ? 1 : n, kScanTile) + 2; }

size_t schedule_workspace(int64_t N, int64_t G) { return sched_ws_layout(nullptr, N, G).bytes; }

fold_status run_schedule(const fold_graphs *gr, fold_schedule_t *s, void *ws_ptr, size_t ws_bytes,
                         cudaStream_t st) {
  g_last_detail = -1;
  if (!gr || !s) return FOLD_E_INVALID;
  const int N = gr->n_nodes, G = gr->n_graphs, V = gr->vocab;
  if (N < 0 || G < 0 || V < 0) return FOLD_E_INVALID;
  s->n_nodes = N; s->n_graphs = G;
  s->n_levels = s->n_leaves = s->n_cells = s->n_tok_segs = 0;
  if (N == 0) {
    if (G > 0) { g_last_detail = 0; return FOLD_E_ROOT_RANGE; }
    if (s->level_off_host) { s->level_off_host[0] = 0; s->level_off_host[1] = 0; }
    if (s->level_off) FOLD_CUDA_TRY(cudaMemsetAsync(s->level_off, 0, 2 * sizeof(int32_t), st));
    if (s->group_off) FOLD_CUDA_TRY(cudaMemsetAsync(s->group_off, 0, 3 * sizeof(int32_t), st));
    if (s->cons_off) FOLD_CUDA_TRY(cudaMemsetAsync(s->cons_off, 0, sizeof(int32_t), st));
    if (s->tok_seg) FOLD_CUDA_TRY(cudaMemsetAsync(s->tok_seg, 0, sizeof(int32_t), st));
    return FOLD_OK;
  }
  if (!gr->op || !gr->child || !gr->token || (G > 0 && !gr->root)) return FOLD_E_INVALID;
  if (!s->depth || !s->perm || !s->rank || !s->gather || !s->level_off || !s->group_off ||
      !s->cons_off || !s->cons_edge || !s->leaf_perm || !s->tok_seg || !s->leaf_token || (G > 0 && (!s->root_row || !s->root_perm)) ||
      !s->level_off_host)
    return FOLD_E_INVALID;
  SchedWs w = sched_ws_layout(ws_ptr, N, G);
  if (!ws_ptr || ws_bytes < w.bytes) return FOLD_E_WORKSPACE;

  // ---- validate, consumer counts, pending counts
  k_init_flags<<<1, F_NFLAGS, 0, st>>>(w.flags, N, G);
  FOLD_LAUNCH_CHECK();
  FOLD_CUDA_TRY(cudaMemsetAsync(w.ncons, 0, (size_t)(N + 1) * 4, st));
  k_validate<<<grid_for(N > G ? N : G), 256, 0, st>>>(N, G, V, gr->op, gr->child, gr->token, gr->root,
                                                       w.flags, w.ncons, w.pending);
  FOLD_LAUNCH_CHECK();
  FOLD_TRY(excl_scan(w.ncons, w.pcons_off, N + 1, w.scan_sums, nullptr, st));
  FOLD_CUDA_TRY(cudaMemsetAsync(w.ncons, 0, (size_t)(N + 1) * 4, st));  // reuse as fill counters
  k_fill_parents<<<grid_for(N), 256, 0, st>>>(N, gr->op, gr->child, w.pcons_off, w.ncons, w.pcons,
                                               s->depth, w.q0, w.flags);
  FOLD_LAUNCH_CHECK();

  // ---- depth frontier (cooperative: all blocks resident for the grid barrier)
  {
    static thread_local int occ = 0, nsm = 0;
    if (!occ) {
      int dev;
      FOLD_CUDA_TRY(cudaGetDevice(&dev));
      FOLD_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      FOLD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_depth_frontier, 256, 0));
      if (occ < 1) occ = 1;
    }
    int64_t want = cdiv(N, 256);
    int64_t cap = (int64_t)nsm * (occ < 2 ? occ : 2);
    int blocks = (int)(want < cap ? want : cap);
    if (blocks < 1) blocks = 1;
    const int32_t *a0 = w.pcons_off, *a1 = w.pcons;
    int32_t *a2 = w.pending, *a3 = s->depth, *a4 = w.q0, *a5 = w.q1, *a6 = w.flags;
    void *args[] = {(void *)&a0, (void *)&a1, (void *)&a2, (void *)&a3, (void *)&a4, (void *)&a5, (void *)&a6};
    FOLD_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_depth_frontier, dim3(blocks), dim3(256), args, 0, st));
    g_launches++;
  }
  k_post_depth<<<grid_for(N), 256, 0, st>>>(N, gr->op, s->depth, w.flags, w.ka, w.va);
  FOLD_LAUNCH_CHECK();

  // ---- stable sort by key = 2*depth + op (ties by node id: input order is id order)
  // count pointer: a constant N lives in the flags scratch slot 20
  int32_t *d_N = w.flags + 20, *d_cnt = w.flags + 21;  // flags[20] = N (k_init_flags)
  uint32_t *sk;
  int32_t *sv;
  FOLD_TRY(radix_sort(w, d_N, N, bits_for(2 * (int64_t)N + 1), &sk, &sv, st));
  k_perm_offsets<<<grid_for(2 * (int64_t)N + 3), 256, 0, st>>>(N, sk, sv, w.flags, s->perm, s->rank,
                                                                s->group_off, s->level_off);
  FOLD_LAUNCH_CHECK();
  k_gather<<<grid_for(N), 256, 0, st>>>(N, gr->op, gr->child, s->perm, s->rank, s->gather);
  FOLD_LAUNCH_CHECK();

  // ---- consumer CSR: cell edges sorted (stably) by child row
  k_cons_keys<<<grid_for(2 * (int64_t)N), 256, 0, st>>>(N, s->gather, w.flags, d_cnt, w.ka, w.va);
  FOLD_LAUNCH_CHECK();
  FOLD_TRY(radix_sort(w, d_cnt, 2 * (int64_t)N, bits_for(N), &sk, &sv, st));
  k_cons_finish<<<grid_for(2 * (int64_t)N + 1), 256, 0, st>>>(N, sk, sv, d_cnt, s->cons_off, s->cons_edge);
  FOLD_LAUNCH_CHECK();

  // ---- leaves by (token, row) and token segments
  int32_t *d_cnt2 = w.flags + 22;
  k_leaf_keys<<<grid_for(N), 256, 0, st>>>(gr->token, s->perm, w.flags, d_cnt2, w.ka, w.va, s->leaf_token);
  FOLD_LAUNCH_CHECK();
  FOLD_TRY(radix_sort(w, d_cnt2, N, bits_for(V > 0 ? V - 1 : 0), &sk, &sv, st));
  k_seg_flags<<<grid_for(N), 256, 0, st>>>(N, sk, sv, d_cnt2, s->leaf_perm, w.seg_flag);
  FOLD_LAUNCH_CHECK();
  FOLD_TRY(excl_scan(w.seg_flag, w.seg_scan, N, w.scan_sums, w.flags + F_NSEG, st));
  k_seg_write<<<grid_for(N), 256, 0, st>>>(N, w.seg_flag, w.seg_scan, d_cnt2, w.flags, s->tok_seg);
  FOLD_LAUNCH_CHECK();

  // ---- roots
  if (G > 0 && G <= kSmallRoots) {
    k_roots_small<<<1, 1024, 0, st>>>(N, G, gr->root, s->rank, s->root_row, s->root_perm);
    FOLD_LAUNCH_CHECK();
  } else if (G > 0) {
    int32_t *d_G = w.flags + 23;  // flags[23] = G (k_init_flags)
    k_root_keys<<<grid_for(G), 256, 0, st>>>(N, G, gr->root, s->rank, s->root_row, w.ka, w.va);
    FOLD_LAUNCH_CHECK();
    FOLD_TRY(radix_sort(w, d_G, G, bits_for(N), &sk, &sv, st));
    k_copy_i32<<<grid_for(G), 256, 0, st>>>(sv, s->root_perm, G);
    FOLD_LAUNCH_CHECK();
  }

  // ---- the one host sync: flags + level_off prefix
  int32_t hflags[F_NFLAGS];
  const int kPrefix = 4096;
  int npre = (N + 2) < kPrefix ? (N + 2) : kPrefix;
  FOLD_CUDA_TRY(cudaMemcpyAsync(hflags, w.flags, sizeof(hflags), cudaMemcpyDeviceToHost, st));
  FOLD_CUDA_TRY(cudaMemcpyAsync(s->level_off_host, s->level_off, (size_t)npre * 4, cudaMemcpyDeviceToHost, st));
  FOLD_CUDA_TRY(cudaStreamSynchronize(st));
  for (int e = 0; e < E_NCLASS; e++) {
    if (hflags[F_ERR0 + e] != INT_MAX) {
      g_last_detail = hflags[F_ERR0 + e];
      return kErrStatus[e];
    }
  }
  int D = hflags[F_MAXDEPTH];
  if (D + 2 > npre) {
    FOLD_CUDA_TRY(cudaMemcpyAsync(s->level_off_host, s->level_off, (size_t)(D + 2) * 4, cudaMemcpyDeviceToHost, st));
    FOLD_CUDA_TRY(cudaStreamSynchronize(st));
  }
  s->n_levels = D;
  s->n_leaves = hflags[F_NLEAVES];
  s->n_cells = N - s->n_leaves;
  s->n_tok_segs = hflags[F_NSEG];
  return FOLD_OK;
}

}  // namespace fold

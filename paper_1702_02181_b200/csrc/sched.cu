// sched.cu — GPU scheduler for dynamic batching (§2, L40-44).
//
// fold_schedule is ONE cooperative persistent kernel (k_schedule) whose phases are
// separated by grid barriers: validate -> consumer counts and lists -> level-synchronous
// depth frontier (one barrier per depth) -> stable counting/radix sort on
// key = 2*depth + op, ties by node id (L42-43) -> perm / rank / offsets / gather vectors
// (L44) -> consumer CSR (stable sort of cell edges by child row) -> leaves by token ->
// roots. Radix pass counts depend on the batch's depth, node count and vocabulary, which
// only the device knows: it chooses them itself, so the host sees one launch and one
// blocking D2H (the executor's launch shapes need level_off). Small batches run as a
// single block, where a "grid barrier" is a __syncthreads. All phases are integer work,
// HBM / latency bound.
#include <climits>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "../../include/fold_mo.h"

namespace fold {

thread_local int64_t g_launches = 0;

namespace {

// flags[] slots (int32) in the workspace header
enum {
  F_ERR0 = 0,  // F_ERR0 + k for the k-th error class (min offending id, INT_MAX = none)
  F_NLEAVES = 8, F_MAXDEPTH = 9, F_NSEG = 10,
  F_QCNT = 12,  // 3 rotating frontier counters 12..14
  F_MULTI = 24,     // 1: some row has >= 2 consumer edges, or a root row is consumed
  F_NDISTROOT = 25, // number of distinct root rows
  F_SHARED = 26,    // 1: some node has >= 2 consumer edges (set in P1)
  F_BAR = 16,   // grid barrier count, generation (16, 17)
  F_NFLAGS = 64
};
enum { E_CHILD = 0, E_OP = 1, E_ARITY = 2, E_TOKEN = 3, E_ROOT = 4, E_LEVEL = 5, E_CYCLE = 6, E_NCLASS = 7 };
const fold_status kErrStatus[E_NCLASS] = {FOLD_E_CHILD_RANGE, FOLD_E_OP_RANGE, FOLD_E_ARITY,
                                         FOLD_E_TOKEN_RANGE, FOLD_E_ROOT_RANGE, FOLD_E_LEVEL,
                                         FOLD_E_CYCLE};

constexpr int kScanThreads = 1024;
constexpr int kScanTile = kScanThreads * 4;
constexpr int kPendingInvalid = 0x3fffffff;

inline int bits_for(int64_t maxval) {  // #bits to represent values in [0, maxval]
  int b = 0;
  while (b < 31 && (int64_t(1) << b) <= maxval) b++;
  return b < 1 ? 1 : b;
}

// ---------------------------------------------------------------- workspace layout
constexpr int kSchedThreads = 512;
constexpr int kSchedWarps = kSchedThreads / 32;
constexpr int kMaxBins = 1024;      // radix digit <= 10 bits
constexpr int kMaxSchedBlocks = 512;
constexpr int kLoMirror = 4096;     // level_off entries mirrored after the flags (one D2H copy)
constexpr int kSmallN = 16384;      // cap of the one-block path (shared-memory depth frontier)
constexpr int kOneBlockN = 4096;    // default: up to this many nodes run as one block (measured)
constexpr int kRootRankMax = 8192;  // P11 ranks the roots in shared memory up to this many graphs
static_assert(kSchedWarps * (kMaxBins + 1) + 2 * kMaxBins + 64 >= kRootRankMax, "P11 root rows fit dsm");

struct SchedWs {
  int32_t *flags, *ncons, *fillc, *pcons_off, *pcons, *pending, *q0, *q1;
  uint32_t *ka, *kb;
  int32_t *va, *vb;
  int32_t *hist, *tot, *bsums, *seg_flag, *seg_scan;
  size_t bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

SchedWs sched_ws_layout(void *base, int64_t N, int64_t G) {
  SchedWs w{};
  int64_t M = 2 * N > G ? 2 * N : G;
  if (M < 1) M = 1;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
  size_t o_flags = take((F_NFLAGS + kLoMirror) * 4);  // flags, then a level_off prefix mirror
  size_t o_ncons = take((N + 1) * 4), o_fill = take((N + 1) * 4), o_pco = take((N + 2) * 4);
  size_t o_pc = take((2 * N + 1) * 4);
  size_t o_pend = take((N + 1) * 4), o_q0 = take((N + 1) * 4), o_q1 = take((N + 1) * 4);
  size_t o_ka = take((M + 1) * 4), o_kb = take((M + 1) * 4), o_va = take((M + 1) * 4), o_vb = take((M + 1) * 4);
  size_t o_hist = take((size_t)kMaxBins * kMaxSchedBlocks * 4), o_tot = take((kMaxBins + 1) * 4);
  size_t o_bs = take((kMaxSchedBlocks + 1) * 4);
  size_t o_sf = take((N + 1) * 4), o_ss = take((N + 2) * 4);
  w.bytes = off;
  if (base) {
    char *b = (char *)base;
    w.flags = (int32_t *)(b + o_flags); w.ncons = (int32_t *)(b + o_ncons); w.fillc = (int32_t *)(b + o_fill);
    w.pcons_off = (int32_t *)(b + o_pco); w.pcons = (int32_t *)(b + o_pc);
    w.pending = (int32_t *)(b + o_pend); w.q0 = (int32_t *)(b + o_q0); w.q1 = (int32_t *)(b + o_q1);
    w.ka = (uint32_t *)(b + o_ka); w.kb = (uint32_t *)(b + o_kb);
    w.va = (int32_t *)(b + o_va); w.vb = (int32_t *)(b + o_vb);
    w.hist = (int32_t *)(b + o_hist); w.tot = (int32_t *)(b + o_tot); w.bsums = (int32_t *)(b + o_bs);
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

// ---------------------------------------------------------------- the persistent kernel
struct SchedArgs {
  int N, G, V;
  const int32_t *op, *child, *token, *root;
  const int32_t *level;  // caller-fixed levels (manual batching) or nullptr
  fold_schedule_t s;  // output arrays (device pointers)
  SchedWs w;
  int dbg;            // FOLD_DBG_SCHED: phase timeline
};

__device__ __forceinline__ int ld_volatile(const int32_t *p) { return *(volatile const int32_t *)p; }
__device__ __forceinline__ int ld_acq(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int dev_bits_for(int maxval) {  // #bits for values in [0, maxval], >= 1
  int b = 32 - __clz(maxval > 0 ? maxval : 1);
  return b < 1 ? 1 : b;
}

// Grid-wide barrier (all blocks co-resident: cooperative launch). Release: every thread's
// prior writes are fenced before the block arrives; acquire: the waiting thread's
// ld.acquire also invalidates this SM's L1, so later plain loads see other blocks' writes.
// Debug phase timeline (FOLD_DBG_SCHED=1): block 0 stamps %globaltimer at each phase start
// (read back with fold_debug_sched_trace; instrumentation only).
__device__ unsigned long long g_sched_trace[16];
__device__ __forceinline__ void sched_stamp(int dbg, int ph) {
  if (dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_sched_trace[ph] = t;
  }
}

__device__ void gsync(int32_t *flags) {
  __syncthreads();
  // one block: __syncthreads orders the block's global writes; data updated by atomics is
  // never read through L1 before its phase's barrier (flags are read volatile)
  if (gridDim.x == 1) return;
  if (threadIdx.x == 0) {
    int32_t *cnt = &flags[F_BAR], *gen = &flags[F_BAR + 1];
    const int g = ld_acq(gen);
    __threadfence();
    if (atomicAdd(cnt, 1) == (int)gridDim.x - 1) {
      atomicExch(cnt, 0);
      __threadfence();
      atomicAdd(gen, 1);
    } else {
      while (ld_acq(gen) == g) __nanosleep(32);
    }
  }
  __syncthreads();
}

// block-wide sum (any blockDim multiple of 32)
__device__ int block_sum(int v, int *sw) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sw[warp] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < nw; i++) t += sw[i];
  __syncthreads();
  return t;
}

// Device-wide exclusive scan of in[0, n) into out (in place allowed), each block a
// contiguous chunk; *total (nullable) receives the sum. Ends with a grid barrier.
__device__ void grid_excl_scan(const int32_t *in, int32_t *out, int n, int32_t *total, SchedWs &w, int *sw) {
  const int nb = gridDim.x, b = blockIdx.x, T = blockDim.x;
  const int chunk = (int)round_up(cdiv(n, nb), (int64_t)T * 4);
  const int lo = min(n, b * chunk), hi = min(n, lo + chunk);
  int s = 0;
  for (int i = lo + threadIdx.x; i < hi; i += T) s += in[i];
  s = block_sum(s, sw);
  if (threadIdx.x == 0) w.bsums[b] = s;
  gsync(w.flags);
  int p = 0;
  for (int i = threadIdx.x; i < b; i += T) p += w.bsums[i];
  int carry = block_sum(p, sw);
  for (int t0 = lo; t0 < hi; t0 += T * 4) {
    const int base = t0 + threadIdx.x * 4;
    int v[4], sum = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) { v[i] = base + i < hi ? in[base + i] : 0; sum += v[i]; }
    int tot;
    int ex = block_excl_scan(sum, sw, &tot) + carry;
#pragma unroll
    for (int i = 0; i < 4; i++) { if (base + i < hi) out[base + i] = ex; ex += v[i]; }
    carry += tot;
  }
  if (b == nb - 1 && threadIdx.x == 0 && total) *total = carry;
  gsync(w.flags);
}

// One stable counting pass: (kin, vin)[0, n) -> (kout, vout) ordered by the digit
// (key >> shift) & (nbins - 1), ties in input order. nbins <= kMaxBins.
// Shared memory: wcnt[kSchedWarps][nbins + 1], run[nbins], base[nbins].
__device__ void sort_pass(const uint32_t *kin, const int32_t *vin, int n, int shift, int nbins, uint32_t *kout,
                          int32_t *vout, SchedWs &w, int *dsm) {
  const int nb = gridDim.x, b = blockIdx.x, T = blockDim.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  int *wcnt = dsm;                                   // [kSchedWarps][nbins + 1]
  int *run = dsm + kSchedWarps * (nbins + 1);        // [nbins]
  int *base = run + nbins;                           // [nbins]
  const uint32_t mask = (uint32_t)nbins - 1u;
  const int chunk = (int)round_up(cdiv(n, nb), T);
  const int lo = min(n, b * chunk), hi = min(n, lo + chunk);
  // 1. block histogram
  for (int d = tid; d < nbins; d += T) run[d] = 0;
  for (int i = tid; i < kSchedWarps * (nbins + 1); i += T) wcnt[i] = 0;
  __syncthreads();
  for (int i = lo + tid; i < hi; i += T) atomicAdd(&run[(kin[i] >> shift) & mask], 1);
  __syncthreads();
  if (nb == 1) {
    // one block: the digit offsets are the exclusive scan of its own histogram (no
    // cross-block prefix through global memory)
    int carry = 0;
    for (int d0 = 0; d0 < nbins; d0 += T) {
      const int d = d0 + tid;
      const int v = d < nbins ? run[d] : 0;
      int tot;
      const int ex = block_excl_scan(v, (int *)(base + nbins), &tot);
      if (d < nbins) base[d] = carry + ex;
      carry += tot;
    }
    __syncthreads();
    for (int d = tid; d < nbins; d += T) run[d] = 0;
  } else {
  for (int d = tid; d < nbins; d += T) w.hist[d * nb + b] = run[d];
  gsync(w.flags);
  // 2. per digit (one warp each): exclusive prefix over blocks, digit totals
  for (int d = (b * T + tid) >> 5; d < nbins; d += (nb * T) >> 5) {
    int carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int bb = b0 + lane;
      const int t = bb < nb ? w.hist[d * nb + bb] : 0;
      int x = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (bb < nb) w.hist[d * nb + bb] = carry + x - t;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) w.tot[d] = carry;
  }
  gsync(w.flags);
  // 3. digit offsets (every block scans the totals), then the stable in-order scatter
  {
    int carry = 0;
    for (int d0 = 0; d0 < nbins; d0 += T) {
      const int d = d0 + tid;
      const int v = d < nbins ? w.tot[d] : 0;
      int tot;
      const int ex = block_excl_scan(v, (int *)(base + nbins), &tot);  // scratch after base
      if (d < nbins) base[d] = carry + ex + w.hist[d * nb + b];
      carry += tot;
    }
    for (int d = tid; d < nbins; d += T) run[d] = 0;
  }
  }
  __syncthreads();
  for (int t0 = lo; t0 < hi; t0 += T) {
    const int i = t0 + tid;
    const bool valid = i < hi;
    const uint32_t k = valid ? kin[i] : 0u;
    const int v = valid ? vin[i] : 0;
    const int d = valid ? (int)((k >> shift) & mask) : nbins;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int lrank = __popc(peers & lanemask_lt());
    const int cnt = __popc(peers);
    if (lrank == 0) wcnt[warp * (nbins + 1) + d] = cnt;
    __syncthreads();
    if (valid) {
      int pre = 0;
      for (int ww = 0; ww < warp; ww++) pre += wcnt[ww * (nbins + 1) + d];
      const int pos = base[d] + run[d] + pre + lrank;
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    if (lrank == 0) {
      if (valid) atomicAdd(&run[d], cnt);
      wcnt[warp * (nbins + 1) + d] = 0;
    }
    __syncthreads();
  }
  gsync(w.flags);
}

// Stable sort of (ka, va)[0, n) by the low nbits of the keys; result pointers in k / v.
__device__ void sort_pairs(SchedWs &w, int n, int nbits, const uint32_t *&k, const int32_t *&v, int *dsm) {
  uint32_t *ki = w.ka, *ko = w.kb;
  int32_t *vi = w.va, *vo = w.vb;
  const int passes = (nbits + 9) / 10;
  const int db = (nbits + passes - 1) / passes;
  for (int p = 0; p < passes; p++) {
    sort_pass(ki, vi, n, p * db, 1 << db, ko, vo, w, dsm);
    uint32_t *tk = ki; ki = ko; ko = tk;
    int32_t *tv = vi; vi = vo; vo = tv;
  }
  k = ki;
  v = vi;
}

__device__ __forceinline__ bool any_input_error(const int32_t *flags) {
  for (int e = 0; e < E_CYCLE; e++)
    if (ld_volatile(&flags[F_ERR0 + e]) != INT_MAX) return true;
  return false;
}

__global__ void __launch_bounds__(kSchedThreads) k_schedule(SchedArgs a) {
  extern __shared__ int dsm[];
  __shared__ int sw[32];
  SchedWs &w = a.w;
  fold_schedule_t &s = a.s;
  int32_t *flags = w.flags;
  const int N = a.N, G = a.G, V = a.V;
  const int tid = threadIdx.x, T = blockDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * T + tid, gstride = (int64_t)gridDim.x * T;

  sched_stamp(a.dbg, 0);
  // ---- P0: flags (barrier slots were zeroed by the host), counters
  if (blockIdx.x == 0 && tid < F_NFLAGS && (tid < F_BAR || tid > F_BAR + 1))
    flags[tid] = tid < E_NCLASS ? INT_MAX : 0;
  for (int64_t i = gtid; i <= N; i += gstride) { w.ncons[i] = 0; w.fillc[i] = 0; }
  gsync(flags);

  sched_stamp(a.dbg, 1);
  // ---- P1: validate (classes in order CHILD_RANGE, OP_RANGE, ARITY, TOKEN_RANGE,
  // ROOT_RANGE; smallest offending id), consumer counts, pending child counts
  for (int64_t i = gtid; i < N; i += gstride) {
    const int n = (int)i;
    const int o = a.op[n], c0 = a.child[2 * n], c1 = a.child[2 * n + 1];
    const bool crange = (c0 < -1 || c0 >= N || c1 < -1 || c1 >= N);
    if (crange) atomicMin(&flags[F_ERR0 + E_CHILD], n);
    if (o != FOLD_OP_EMBED && o != FOLD_OP_CELL) atomicMin(&flags[F_ERR0 + E_OP], n);
    const bool ar_ok = (o == FOLD_OP_EMBED) ? (c0 == -1 && c1 == -1) : (c0 >= 0 && c1 >= 0);
    if (!ar_ok) atomicMin(&flags[F_ERR0 + E_ARITY], n);
    if (o == FOLD_OP_EMBED && (a.token[n] < 0 || a.token[n] >= V)) atomicMin(&flags[F_ERR0 + E_TOKEN], n);
    const bool good_cell = (o == FOLD_OP_CELL) && !crange && c0 >= 0 && c1 >= 0;
    if (good_cell) {
      // a node read by two edges (incl. cell(x, x)) needs the general consumer-CSR sort
      const int o0 = atomicAdd(&w.ncons[c0], 1), o1 = atomicAdd(&w.ncons[c1], 1);
      if (o0 > 0 || o1 > 0) flags[F_SHARED] = 1;
    }
    if (a.level) {  // manual batching: level[EMBED] == 1, level[CELL] > level[children], <= N
      const int lv = a.level[n];
      bool bad = lv < 1 || lv > N;
      if (o == FOLD_OP_EMBED) bad = bad || lv != 1;
      if (good_cell) bad = bad || lv <= a.level[c0] || lv <= a.level[c1];
      if (bad && (o == FOLD_OP_EMBED || good_cell)) atomicMin(&flags[F_ERR0 + E_LEVEL], n);
      if (o == FOLD_OP_EMBED || good_cell) atomicMax(&flags[F_MAXDEPTH], lv < 1 ? 1 : lv);
    }
    w.pending[n] = (o == FOLD_OP_CELL) ? (good_cell ? 2 : kPendingInvalid) : 0;
    // tree-like depth walk (P4): no parent yet, empty arrival slot (sort scratch, free until P5)
    reinterpret_cast<int32_t *>(w.kb)[n] = -1;
    w.va[n] = -1;
  }
  for (int64_t g = gtid; g < G; g += gstride)
    if (a.root[g] < 0 || a.root[g] >= N) atomicMin(&flags[F_ERR0 + E_ROOT], (int)g);
  gsync(flags);
  if (any_input_error(flags)) return;  // uniform: every block reads the same flags

  sched_stamp(a.dbg, 2);
  // ---- P2: parent-list offsets
  grid_excl_scan(w.ncons, w.pcons_off, N + 1, nullptr, w, sw);

  sched_stamp(a.dbg, 3);
  // ---- P3: parent lists (unordered within a node), initial frontier = EMBED nodes (depth 1)
  {
    const int64_t nloop = cdiv(N, gstride) * gstride;
    for (int64_t i = gtid; i < nloop; i += gstride) {
      const bool in = i < N;
      const int n = (int)i;
      bool leaf = false;
      if (in) {
        const int o = a.op[n], c0 = a.child[2 * n], c1 = a.child[2 * n + 1];
        if (o == FOLD_OP_CELL) {
          w.pcons[w.pcons_off[c0] + atomicAdd(&w.fillc[c0], 1)] = n;
          w.pcons[w.pcons_off[c1] + atomicAdd(&w.fillc[c1], 1)] = n;
          // the parent of each child (meaningful when every node has <= 1 consumer edge)
          reinterpret_cast<int32_t *>(w.kb)[c0] = n;
          reinterpret_cast<int32_t *>(w.kb)[c1] = n;
        }
        leaf = (o == FOLD_OP_EMBED);
        s.depth[n] = a.level ? a.level[n] : (leaf ? 1 : -1);
      }
      const int slot = warp_push(&flags[F_QCNT + 1], leaf);
      if (leaf) w.q0[slot] = n;
      const int nl = __popc(__ballot_sync(0xffffffffu, leaf));
      if ((tid & 31) == 0 && nl) atomicAdd(&flags[F_NLEAVES], nl);
    }
  }
  gsync(flags);

  sched_stamp(a.dbg, 4);
  // ---- P4: level-synchronous depth propagation: a parent whose last
  // pending child finishes at level L gets depth L + 1; one barrier per level.
  // One block (small batches; deep chains are the latency-bound case): the pending counts
  // and both frontiers live in shared memory (the sort's scratch, sized 3N for this
  // launch), so a level is a __syncthreads plus shared-memory atomics.
  int L = 1;
  if (gridDim.x == 1 && !a.level) {
    int *pend = dsm, *qa = dsm + N, *qb = dsm + 2 * N;
    __shared__ int qn[2];
    const int n0 = ld_volatile(&flags[F_QCNT + 1]);
    for (int i = tid; i < N; i += T) pend[i] = w.pending[i];
    for (int i = tid; i < n0; i += T) qa[i] = w.q0[i];
    if (tid == 0) { qn[0] = n0; qn[1] = 0; }
    __syncthreads();
    for (;; L++) {
      const int cb = (L & 1) ? 0 : 1;  // current queue: qa on odd levels
      const int ncur = qn[cb];
      if (ncur == 0) break;
      const int *cur = cb ? qb : qa;
      int *nxt = cb ? qa : qb;
      for (int i = tid; i < ncur; i += T) {
        const int x = cur[i];
        for (int e = w.pcons_off[x]; e < w.pcons_off[x + 1]; e++) {
          const int p = w.pcons[e];
          if (atomicSub(&pend[p], 1) == 1) {
            s.depth[p] = L + 1;
            nxt[atomicAdd(&qn[cb ^ 1], 1)] = p;
          }
        }
      }
      __syncthreads();
      if (tid == 0) qn[cb] = 0;  // becomes the next-next frontier
      __syncthreads();
    }
  }
#ifdef FOLD_SCHED_LEVELSYNC  // the level-synchronous frontier (one grid barrier per level)
  for (; !a.level && gridDim.x > 1; L++) {
    const int ncur = ld_volatile(&flags[F_QCNT + (L % 3)]);
    if (ncur == 0) break;
    const int32_t *cur = (L & 1) ? w.q0 : w.q1;
    int32_t *nxt = (L & 1) ? w.q1 : w.q0;
    if (gtid == 0) flags[F_QCNT + ((L + 2) % 3)] = 0;
    const int64_t nloop = cdiv(ncur, gstride) * gstride;
    for (int64_t i = gtid; i < nloop; i += gstride) {
      const bool in = i < ncur;
      const int x = in ? cur[i] : 0;
      const int e0 = in ? w.pcons_off[x] : 0, e1 = in ? w.pcons_off[x + 1] : 0;
      for (int j = 0; __any_sync(0xffffffffu, e0 + j < e1); j++) {
        bool act = false;
        int p = 0;
        if (e0 + j < e1) {
          p = w.pcons[e0 + j];
          act = (atomicSub(&w.pending[p], 1) == 1);
          if (act) s.depth[p] = L + 1;
        }
        const int slot = warp_push(&flags[F_QCNT + ((L + 1) % 3)], act);
        if (act) nxt[slot] = p;
      }
    }
    gsync(flags);
  }
#else
  // Many blocks: asynchronous propagation by last arrival, no barrier per level. A thread
  // takes a node whose depth is final and decrements each parent's pending count (release:
  // fence, then the atomic); the thread that brings a parent to 0 (acquire: the atomic, then a
  // fence) reads its children's depths and sets depth = 1 + max (L40: the same value the
  // level-synchronous frontier gives, whose last finishing child has the largest depth), then
  // walks on from that parent. Trees: every walk ends at a parent another walk completes, so
  // the whole depth pass is ONE barrier; the chain of a depth-256 caterpillar is walked by one
  // thread (C4 B=1024 P4 1203 us with a barrier per level). DAGs: a node completing several
  // parents walks one and queues the rest for the next round (a barrier per round).
  if (!a.level && gridDim.x > 1 && ld_volatile(&flags[F_SHARED]) == 0) {
    // tree-like batches (every node read by <= 1 edge): a node's parent is unique (kb), and its
    // two children meet in an exchange slot (va, -1 = empty): the first arriver leaves its depth
    // there, the second gets it back from the same atomic and continues with
    // 1 + max(both). The depth travels inside the atomic, so no fence or depth load is on the
    // walk; the parent's parent is loaded while the exchange is in flight (one L2 round trip
    // per tree level).
    const int32_t *par = reinterpret_cast<const int32_t *>(w.kb);
    const int n0 = ld_volatile(&flags[F_QCNT + 1]);
    int dmax = n0 > 0 ? 1 : 0;
    for (int64_t i = gtid; i < n0; i += gstride) {
      int dx = 1;
      int p = __ldcg(&par[w.q0[i]]);
      while (p >= 0) {
        const int pp = __ldcg(&par[p]);
        const int other = atomicExch(&w.va[p], dx);
        if (other < 0) break;  // the sibling is not done: it continues from p
        dx = 1 + (other > dx ? other : dx);
        s.depth[p] = dx;
        if (dx > dmax) dmax = dx;
        p = pp;
      }
    }
    if (dmax > 0) atomicMax(&flags[F_MAXDEPTH], dmax);
    gsync(flags);
  } else if (!a.level && gridDim.x > 1) {
    int dmax = 0;
    for (int r = 1;; r++) {
      const int ncur = ld_volatile(&flags[F_QCNT + (r % 3)]);
      if (ncur == 0) break;
      const int32_t *src = (r & 1) ? w.q0 : w.q1;
      int32_t *ovf = (r & 1) ? w.q1 : w.q0;
      if (gtid == 0) flags[F_QCNT + ((r + 2) % 3)] = 0;
      for (int64_t i = gtid; i < ncur; i += gstride) {
        int x = src[i];
        int dx = r == 1 ? 1 : __ldcg(&s.depth[x]);  // round 1: the leaves (depth 1)
        if (dx > dmax) dmax = dx;
        for (;;) {
          int next = -1, dnext = 0;
          const int e0 = __ldcg(&w.pcons_off[x]), e1 = __ldcg(&w.pcons_off[x + 1]);
          for (int e = e0; e < e1; e++) {
            const int p = __ldcg(&w.pcons[e]);
            const int c0 = __ldg(&a.child[2 * p]), c1 = __ldg(&a.child[2 * p + 1]);
            __threadfence();
            if (atomicSub(&w.pending[p], 1) != 1) continue;
            __threadfence();
            const int d0 = c0 == x ? dx : __ldcg(&s.depth[c0]);
            const int d1 = c1 == x ? dx : __ldcg(&s.depth[c1]);
            const int dp = 1 + (d0 > d1 ? d0 : d1);
            s.depth[p] = dp;
            if (next < 0) {
              next = p;
              dnext = dp;
            } else {  // a second completed parent (shared node): the next round walks it
              __threadfence();
              ovf[atomicAdd(&flags[F_QCNT + ((r + 1) % 3)], 1)] = p;
            }
          }
          if (next < 0) break;
          x = next;
          dx = dnext;
          if (dx > dmax) dmax = dx;
        }
      }
      gsync(flags);
    }
    if (dmax > 0) atomicMax(&flags[F_MAXDEPTH], dmax);
    gsync(flags);
  }
#endif
#ifdef FOLD_SCHED_LEVELSYNC
  const int D = a.level ? ld_volatile(&flags[F_MAXDEPTH]) : L - 1;
#else
  const int D = (a.level || gridDim.x > 1) ? ld_volatile(&flags[F_MAXDEPTH]) : L - 1;
#endif
  if (gtid == 0 && !a.level) flags[F_MAXDEPTH] = D;

  sched_stamp(a.dbg, 5);
  // ---- P5: sort keys (cycle: a node never reached keeps depth -1)
  for (int64_t i = gtid; i < N; i += gstride) {
    const int n = (int)i, d = s.depth[n];
    if (d < 0) atomicMin(&flags[F_ERR0 + E_CYCLE], n);
    w.ka[n] = (uint32_t)(2 * (d < 0 ? 0 : d) + (a.op[n] & 1));
    w.va[n] = n;
  }
  gsync(flags);
  if (ld_volatile(&flags[F_ERR0 + E_CYCLE]) != INT_MAX) return;

  sched_stamp(a.dbg, 6);
  // ---- P6: stable sort by key = 2 depth + op (L42-43); ties keep ascending node id
  const int nk = 2 * (D + 1);
  const uint32_t *sk;
  const int32_t *sv;
  sort_pairs(w, N, dev_bits_for(nk - 1), sk, sv, dsm);

  sched_stamp(a.dbg, 7);
  // ---- P7: perm / rank, group and level offsets (binary search over the sorted keys)
  for (int64_t i = gtid; i < N; i += gstride) {
    const int n = sv[i];
    s.perm[i] = n;
    s.rank[n] = (int)i;
  }
  for (int64_t k = gtid; k <= nk; k += gstride) {
    int lo = 0, hi = N;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if ((int)sk[mid] < (int)k) lo = mid + 1; else hi = mid; }
    s.group_off[k] = lo;
    if ((k & 1) == 0) {
      s.level_off[k >> 1] = lo;
      if ((k >> 1) < kLoMirror) flags[F_NFLAGS + (k >> 1)] = lo;  // fetched with the flags
    }
  }
  gsync(flags);

  sched_stamp(a.dbg, 8);
  // ---- P8: gather vectors (L44: the indices encode the topology)
  for (int64_t r = gtid; r < N; r += gstride) {
    const int n = s.perm[r];
    const bool cell = a.op[n] == FOLD_OP_CELL;
    s.gather[2 * r] = cell ? s.rank[a.child[2 * n]] : -1;
    s.gather[2 * r + 1] = cell ? s.rank[a.child[2 * n + 1]] : -1;
  }
  gsync(flags);

  sched_stamp(a.dbg, 9);
  // ---- P9: consumer CSR: cell edges e in [0, 2 n_cells), key = child row, stable
  const int nl = ld_volatile(&flags[F_NLEAVES]);
  const int ne = 2 * (N - nl);
  if (ld_volatile(&flags[F_SHARED]) == 0) {
    // every node is read by at most one edge (trees): cons_off is the exclusive scan of
    // "row is consumed" and each edge lands at its child row's offset -- the same CSR the
    // stable sort yields, without the sort passes
    for (int64_t r = gtid; r <= N; r += gstride) w.seg_flag[r] = r < N ? w.ncons[s.perm[r]] : 0;
    gsync(flags);
    grid_excl_scan(w.seg_flag, s.cons_off, N + 1, nullptr, w, sw);
    for (int64_t e = gtid; e < ne; e += gstride) s.cons_edge[s.cons_off[s.gather[2 * (int64_t)nl + e]]] = (int)e;
    gsync(flags);
  } else {
  for (int64_t e = gtid; e < ne; e += gstride) {
    w.ka[e] = (uint32_t)s.gather[2 * (int64_t)nl + e];
    w.va[e] = (int)e;
  }
  gsync(flags);
  sort_pairs(w, ne, dev_bits_for(N - 1), sk, sv, dsm);
  for (int64_t i = gtid; i < ne; i += gstride) {
    s.cons_edge[i] = sv[i];
    if (i > 0 && sk[i] == sk[i - 1]) flags[F_MULTI] = 1;  // a row read by two edges
  }
  for (int64_t r = gtid; r <= N; r += gstride) {
    int lo = 0, hi = ne;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if ((int)sk[mid] < (int)r) lo = mid + 1; else hi = mid; }
    s.cons_off[r] = lo;
  }
  gsync(flags);
  }

  sched_stamp(a.dbg, 10);
  // ---- P10: leaves by (token, row) and token segments
  for (int64_t r = gtid; r < nl; r += gstride) {
    const int t = a.token[s.perm[r]];
    w.ka[r] = (uint32_t)t;
    w.va[r] = (int)r;
    s.leaf_token[r] = t;
  }
  gsync(flags);
  sort_pairs(w, nl, dev_bits_for(V - 1), sk, sv, dsm);
  for (int64_t i = gtid; i < nl; i += gstride) {
    s.leaf_perm[i] = sv[i];
    w.seg_flag[i] = (i == 0 || sk[i] != sk[i - 1]) ? 1 : 0;
  }
  gsync(flags);
  grid_excl_scan(w.seg_flag, w.seg_scan, nl, &flags[F_NSEG], w, sw);
  for (int64_t i = gtid; i < nl; i += gstride)
    if (w.seg_flag[i]) s.tok_seg[w.seg_scan[i]] = (int)i;
  if (gtid == 0) s.tok_seg[ld_volatile(&flags[F_NSEG])] = nl;

  sched_stamp(a.dbg, 11);
  // ---- P11: roots, and graph ids ordered by (root row, g)
  if (G > 0 && G <= kRootRankMax) {
    // up to a few thousand graphs: every block stages all root rows in shared memory and each
    // graph's position is its stable rank, #{g' : (row', g') < (row, g)} -- one pass and no
    // barrier instead of the radix passes' (C3 B=1024: 25 us)
    __syncthreads();
    for (int g = tid; g < G; g += T) dsm[g] = s.rank[a.root[g]];
    __syncthreads();
    // one warp per graph, the lanes split the other graphs and the counts are warp-reduced
    const int lane = tid & 31;
    const int64_t gw = gtid >> 5, nw = gstride >> 5;
    for (int64_t g = gw; g < G; g += nw) {
      const int rr = dsm[g];
      int pos = 0, dup = 0;
      for (int j = lane; j < G; j += 32) {
        const int k = dsm[j];
        pos += (k < rr || (k == rr && j < (int)g)) ? 1 : 0;
        dup += (k == rr && j < (int)g) ? 1 : 0;
      }
      pos = __reduce_add_sync(0xffffffffu, pos);
      dup = __reduce_add_sync(0xffffffffu, dup);
      if (lane == 0) {
        s.root_row[g] = rr;
        s.root_perm[pos] = (int)g;
        if (dup == 0) {
          atomicAdd(&flags[F_NDISTROOT], 1);
          if (s.cons_off[rr + 1] > s.cons_off[rr]) flags[F_MULTI] = 1;  // a consumed root
        }
      }
    }
  } else if (G > 0) {
    for (int64_t g = gtid; g < G; g += gstride) {
      const int rr = s.rank[a.root[g]];
      s.root_row[g] = rr;
      w.ka[g] = (uint32_t)rr;
      w.va[g] = (int)g;
    }
    gsync(flags);
    sort_pairs(w, G, dev_bits_for(N - 1), sk, sv, dsm);
    for (int64_t q = gtid; q < G; q += gstride) {
      s.root_perm[q] = sv[q];
      const int rr = (int)sk[q];
      if (q == 0 || sk[q] != sk[q - 1]) {
        atomicAdd(&flags[F_NDISTROOT], 1);
        if (s.cons_off[rr + 1] > s.cons_off[rr]) flags[F_MULTI] = 1;  // a consumed root
      }
    }
  }
  sched_stamp(a.dbg, 12);
}


// ================================================================ multi-op schedule (NEXT-3)
// fold_mo.h: several operations and tensor types per depth. One
// cooperative kernel, phases separated by grid barriers: validate (op table arities and
// types, L33) -> depth by relaxation rounds (a node whose children all have depths takes
// 1 + their max, L40; one barrier per round, D + 1 rounds; nodes never assigned depend on a
// cycle) -> stable sort by key = depth*K + op (L42: the batched instances, ties by id) ->
// stable partition of that order by output type (L43: per-type concatenation in depth and
// enumeration order) -> per-(type, depth) offsets and (d, t, i) edge labels (L44) -> the
// executor's consumer CSR, root lists and (op, token) leaf segments.
enum { MOE_CHILD = 0, MOE_OP = 1, MOE_ARITY = 2, MOE_TYPE = 3, MOE_TOKEN = 4, MOE_ROOT = 5, MOE_CYCLE = 6,
       MOE_NCLASS = 7 };
const fold_status kMoErrStatus[MOE_NCLASS] = {FOLD_E_CHILD_RANGE, FOLD_E_OP_RANGE, FOLD_E_ARITY,
                                             (fold_status)FOLD_E_TYPE, FOLD_E_TOKEN_RANGE, FOLD_E_ROOT_RANGE,
                                             FOLD_E_CYCLE};

struct MoSchedArgs {
  int N, G, K, T;
  int kind[FOLD_MO_MAX_OPS], arity[FOLD_MO_MAX_OPS], in_type[FOLD_MO_MAX_OPS], out_type[FOLD_MO_MAX_OPS],
      vocab[FOLD_MO_MAX_OPS];
  const int32_t *op, *child, *token, *root;
  fold_mo_schedule_t s;
  SchedWs w;
  int32_t *opos, *gcnt, *tcnt, *tscan;
};

__global__ void __launch_bounds__(kSchedThreads) k_mo_schedule(MoSchedArgs a) {
  extern __shared__ int dsm[];
  __shared__ int sw[32];
  SchedWs &w = a.w;
  fold_mo_schedule_t &s = a.s;
  int32_t *flags = w.flags;
  const int N = a.N, G = a.G, K = a.K, T = a.T;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid, gstride = (int64_t)gridDim.x * blockDim.x;

  // ---- P0: flags, depths unassigned (0)
  if (blockIdx.x == 0 && tid < F_NFLAGS && (tid < F_BAR || tid > F_BAR + 1))
    flags[tid] = tid < MOE_NCLASS ? INT_MAX : 0;
  for (int64_t i = gtid; i < N; i += gstride) s.depth[i] = 0;
  gsync(flags);

  // ---- P1: validate (CHILD_RANGE, OP_RANGE, ARITY, TYPE, TOKEN_RANGE, ROOT_RANGE)
  for (int64_t i = gtid; i < N; i += gstride) {
    const int n = (int)i, o = a.op[n], c0 = a.child[2 * n], c1 = a.child[2 * n + 1];
    const bool crange = c0 < -1 || c0 >= N || c1 < -1 || c1 >= N;
    if (crange) atomicMin(&flags[F_ERR0 + MOE_CHILD], n);
    if (o < 0 || o >= K) { atomicMin(&flags[F_ERR0 + MOE_OP], n); continue; }
    const int ar = a.arity[o];
    const bool ar_ok = (ar > 0 ? c0 >= 0 : c0 == -1) && (ar > 1 ? c1 >= 0 : c1 == -1);
    if (!ar_ok) atomicMin(&flags[F_ERR0 + MOE_ARITY], n);
    if (!crange && ar_ok)
      for (int k = 0; k < ar; k++) {
        const int oc = a.op[a.child[2 * n + k]];
        if (oc >= 0 && oc < K && a.out_type[oc] != a.in_type[o]) atomicMin(&flags[F_ERR0 + MOE_TYPE], n);
      }
    if (a.kind[o] == FOLD_MO_EMBED && (a.token[n] < 0 || a.token[n] >= a.vocab[o]))
      atomicMin(&flags[F_ERR0 + MOE_TOKEN], n);
  }
  for (int64_t g = gtid; g < G; g += gstride)
    if (a.root[g] < 0 || a.root[g] >= N) atomicMin(&flags[F_ERR0 + MOE_ROOT], (int)g);
  gsync(flags);
  for (int e = 0; e < MOE_CYCLE; e++)
    if (ld_volatile(&flags[F_ERR0 + e]) != INT_MAX) return;  // uniform across blocks

  // ---- P2: depths by relaxation rounds (L40); round r's "changed" flag in F_QCNT + r % 3
  for (int r = 0;; r++) {
    const int slot = F_QCNT + r % 3;
    if (gtid == 0) flags[F_QCNT + (r + 1) % 3] = 0;
    bool changed = false;
    const int64_t nloop = cdiv(N, gstride) * gstride;
    for (int64_t i = gtid; i < nloop; i += gstride) {
      bool ch = false;
      if (i < N && ld_volatile(&s.depth[i]) == 0) {
        const int n = (int)i, ar = a.arity[a.op[n]];
        int dm = 0;
        bool ready = true;
        for (int k = 0; k < ar; k++) {
          const int dc = ld_volatile(&s.depth[a.child[2 * n + k]]);
          ready = ready && dc > 0;
          dm = dc > dm ? dc : dm;
        }
        if (ready) {
          s.depth[n] = 1 + dm;
          atomicMax(&flags[F_MAXDEPTH], 1 + dm);
          ch = true;
        }
      }
      changed = changed || ch;
    }
    if (__any_sync(0xffffffffu, changed) && lane == 0) flags[slot] = 1;
    gsync(flags);
    if (ld_volatile(&flags[slot]) == 0) break;
  }
  for (int64_t i = gtid; i < N; i += gstride)
    if (ld_volatile(&s.depth[i]) == 0) atomicMin(&flags[F_ERR0 + MOE_CYCLE], (int)i);
  gsync(flags);
  if (ld_volatile(&flags[F_ERR0 + MOE_CYCLE]) != INT_MAX) return;
  const int D = ld_volatile(&flags[F_MAXDEPTH]);

  // ---- P3: (depth, op) groups (L42) and the stable order by key = depth*K + op
  const int nk = (D + 1) * K;
  for (int64_t k = gtid; k <= nk; k += gstride) a.gcnt[k] = 0;
  gsync(flags);
  for (int64_t i = gtid; i < N; i += gstride) {
    const int key = s.depth[i] * K + a.op[i];
    w.ka[i] = (uint32_t)key;
    w.va[i] = (int)i;
    atomicAdd(&a.gcnt[key], 1);
  }
  gsync(flags);
  grid_excl_scan(a.gcnt, s.group_off, nk + 1, nullptr, w, sw);
  for (int64_t k = gtid; k <= nk && k < kLoMirror; k += gstride) flags[F_NFLAGS + k] = s.group_off[k];
  const uint32_t *sk;
  const int32_t *sv;
  sort_pairs(w, N, dev_bits_for(nk - 1), sk, sv, dsm);
  for (int64_t i = gtid; i < N; i += gstride) {
    s.order[i] = sv[i];
    a.opos[sv[i]] = (int)i;
  }
  gsync(flags);

  // ---- P4: per-type pools (L43): the order, stably partitioned by output type
  for (int64_t i = gtid; i < N; i += gstride) {
    const int n = s.order[i];
    w.ka[i] = (uint32_t)a.out_type[a.op[n]];
    w.va[i] = n;
  }
  gsync(flags);
  sort_pairs(w, N, dev_bits_for(T - 1), sk, sv, dsm);
  for (int64_t t = gtid; t <= T; t += gstride) {
    int lo = 0, hi = N;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if ((int)sk[mid] < (int)t) lo = mid + 1; else hi = mid; }
    s.type_off[t] = lo;
  }
  const int tl = T * (D + 2);
  for (int64_t k = gtid; k <= tl; k += gstride) a.tcnt[k] = 0;
  gsync(flags);
  for (int64_t i = gtid; i < N; i += gstride) {
    const int n = sv[i], t = (int)sk[i];
    s.pool[i] = n;
    s.pool_row[n] = (int)i - s.type_off[t];
    atomicAdd(&a.tcnt[t * (D + 2) + s.depth[n]], 1);
  }
  gsync(flags);
  grid_excl_scan(a.tcnt, a.tscan, tl + 1, nullptr, w, sw);
  for (int64_t k = gtid; k < tl; k += gstride) s.tlevel_off[k] = a.tscan[k] - a.tscan[(k / (D + 2)) * (D + 2)];
  gsync(flags);

  // ---- P5: edge labels (d, t, i) (L44)
  for (int64_t e = gtid; e < 2 * (int64_t)N; e += gstride) {
    const int c = a.child[e];
    int32_t *lab = s.label + 3 * e;
    if (c < 0) { lab[0] = lab[1] = lab[2] = -1; continue; }
    const int d = s.depth[c], t = a.out_type[a.op[c]];
    lab[0] = d; lab[1] = t; lab[2] = s.pool_row[c] - s.tlevel_off[t * (D + 2) + d];
  }

  // ---- P6: consumers by global pool index: edges e = 2 * order position + k, stable
  for (int64_t e = gtid; e < 2 * (int64_t)N; e += gstride) {
    const int m = s.order[e >> 1], c = a.child[2 * m + (int)(e & 1)];
    w.ka[e] = (uint32_t)(c >= 0 ? s.type_off[a.out_type[a.op[c]]] + s.pool_row[c] : N);
    w.va[e] = (int)e;
  }
  gsync(flags);
  sort_pairs(w, 2 * N, dev_bits_for(N), sk, sv, dsm);
  for (int64_t i = gtid; i < 2 * (int64_t)N; i += gstride) s.cons_edge[i] = sv[i];
  for (int64_t r = gtid; r <= N; r += gstride) {
    int lo = 0, hi = 2 * N;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if ((int)sk[mid] < (int)r) lo = mid + 1; else hi = mid; }
    s.cons_off[r] = lo;
  }
  gsync(flags);

  // ---- P7: graphs rooted at each node (by global pool index), ascending g
  if (G > 0) {
    for (int64_t g = gtid; g < G; g += gstride) {
      const int n = a.root[g];
      w.ka[g] = (uint32_t)(s.type_off[a.out_type[a.op[n]]] + s.pool_row[n]);
      w.va[g] = (int)g;
    }
    gsync(flags);
    sort_pairs(w, G, dev_bits_for(N - 1), sk, sv, dsm);
    for (int64_t i = gtid; i < G; i += gstride) s.root_graph[i] = sv[i];
    for (int64_t r = gtid; r <= N; r += gstride) {
      int lo = 0, hi = G;
      while (lo < hi) { const int mid = (lo + hi) >> 1; if ((int)sk[mid] < (int)r) lo = mid + 1; else hi = mid; }
      s.root_off[r] = lo;
    }
  } else {
    for (int64_t r = gtid; r <= N; r += gstride) s.root_off[r] = 0;
  }
  gsync(flags);

  // ---- P8: leaves (the depth-1 groups, all EMBED) by (op, token, order position)
  const int l0 = s.group_off[K], nl = s.group_off[2 * K] - l0;
  int vmax = 1;
  for (int o = 0; o < K; o++) vmax = a.vocab[o] > vmax ? a.vocab[o] : vmax;
  const int vbits = dev_bits_for(vmax - 1);
  for (int64_t i = gtid; i < nl; i += gstride) {
    const int p = l0 + (int)i, n = s.order[p];
    w.ka[i] = ((uint32_t)a.op[n] << vbits) | (uint32_t)a.token[n];
    w.va[i] = p;
  }
  if (gtid == 0) flags[F_NLEAVES] = nl;
  gsync(flags);
  sort_pairs(w, nl, vbits + dev_bits_for(K - 1), sk, sv, dsm);
  for (int64_t i = gtid; i < nl; i += gstride) {
    s.leaf_order[i] = sv[i];
    w.seg_flag[i] = (i == 0 || sk[i] != sk[i - 1]) ? 1 : 0;
  }
  gsync(flags);
  grid_excl_scan(w.seg_flag, w.seg_scan, nl, &flags[F_NSEG], w, sw);
  for (int64_t i = gtid; i < nl; i += gstride)
    if (w.seg_flag[i]) s.leaf_seg[w.seg_scan[i]] = (int)i;
  if (gtid == 0) s.leaf_seg[ld_volatile(&flags[F_NSEG])] = nl;
}

}  // namespace

thread_local int32_t g_last_detail = -1;
// (node, depth, op) context of the last data-dependent error (errors carry
// (depth, operation)); see fold.h fold_last_error_context
thread_local int32_t g_last_ctx[3] = {-1, -1, -1};

// device-wide exclusive int32 scan for other translation units; `sums` needs
// scan_sums_count(n) entries
fold_status scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *sums, int32_t *total,
                           cudaStream_t st) {
  return excl_scan(in, out, n, sums, total, st);
}
int64_t scan_sums_count(int64_t n) { return cdiv(n < 1 ? 1 : n, kScanTile) + 2; }

int debug_sched_trace(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, g_sched_trace, 13 * 8) == cudaSuccess ? 13 : -1;
}

size_t schedule_workspace(int64_t N, int64_t G) { return sched_ws_layout(nullptr, N, G).bytes; }

fold_status run_schedule(const fold_graphs *gr, fold_schedule_t *s, void *ws_ptr, size_t ws_bytes, int max_blocks_hint,
                         cudaStream_t st) {
  g_last_detail = -1;
  g_last_ctx[0] = g_last_ctx[1] = g_last_ctx[2] = -1;
  if (!gr || !s) return FOLD_E_INVALID;
  const int N = gr->n_nodes, G = gr->n_graphs, V = gr->vocab;
  if (N < 0 || G < 0 || V < 0) return FOLD_E_INVALID;
  s->n_nodes = N; s->n_graphs = G;
  s->n_levels = s->n_leaves = s->n_cells = s->n_tok_segs = 0;
  s->tree_like = 0;
  if (N == 0) {
    if (G > 0) { g_last_detail = 0; g_last_ctx[0] = 0; return FOLD_E_ROOT_RANGE; }
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

  // grid: one block for small batches, else enough blocks for ~2K nodes each, all
  // co-resident (cooperative launch)
  const size_t dsmem = (size_t)(kSchedWarps * (kMaxBins + 1) + 2 * kMaxBins + 64) * sizeof(int);
  static thread_local int max_blocks_dev[kMaxDevices] = {};
  static thread_local size_t smem_set_dev[kMaxDevices] = {};
  const int dev = cur_dev();
  int &max_blocks = max_blocks_dev[dev];
  size_t &smem_set = smem_set_dev[dev];
  if (!max_blocks) {
    int nsm, occ = 0;
    FOLD_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    FOLD_CUDA_TRY(cudaFuncSetAttribute(k_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
    FOLD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_schedule, kSchedThreads, dsmem));
    if (occ < 1) occ = 1;
    max_blocks = nsm * (occ < 2 ? occ : 2);
    if (max_blocks > kMaxSchedBlocks) max_blocks = kMaxSchedBlocks;
  }
  // one block up to small_n nodes, else ~per_block nodes per block (FOLD_SCHED_SMALLN /
  // FOLD_SCHED_PER_BLOCK override the defaults for tuning experiments)
  static const int small_n = [] {
    const char *e = getenv("FOLD_SCHED_SMALLN");
    const int v = e ? atoi(e) : kOneBlockN;
    return v < 0 ? 0 : (v > kSmallN ? kSmallN : v);
  }();
  static const int per_block = [] {
    const char *e = getenv("FOLD_SCHED_PER_BLOCK");
    const int v = e ? atoi(e) : 2048;
    return v < 256 ? 256 : v;
  }();
  int blocks = N <= small_n ? 1 : (int)cdiv(N, per_block);
  if (blocks > max_blocks) blocks = max_blocks;
  // caller cap (fold_schedule_ex): a schedule that runs BESIDE other kernels (the next batch's,
  // overlapping this batch's weight-gradient GEMM) takes few SMs; the cap never selects the
  // one-block path, whose shared-memory frontier holds only small batches
  if (max_blocks_hint > 0 && blocks > max_blocks_hint) blocks = max_blocks_hint < 2 ? 2 : max_blocks_hint;
  // one block: its depth propagation keeps pending counts and both frontiers in shared
  // memory (3N ints, at most 192 KB for kSmallN nodes)
  size_t launch_smem = dsmem;
  if (blocks == 1 && (size_t)3 * N * sizeof(int) > launch_smem) launch_smem = (size_t)3 * N * sizeof(int);
  if (launch_smem > smem_set) {
    FOLD_CUDA_TRY(cudaFuncSetAttribute(k_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)launch_smem));
    smem_set = launch_smem;
  }
  static const int dbg = [] { const char *e = getenv("FOLD_DBG_SCHED"); return e ? atoi(e) : 0; }();
  SchedArgs args{N, G, V, gr->op, gr->child, gr->token, gr->root, gr->level, *s, w, dbg};
  if (blocks == 1) {  // no grid barrier: a plain launch (cheaper than a cooperative one)
    k_schedule<<<1, kSchedThreads, launch_smem, st>>>(args);
  } else {
    FOLD_CUDA_TRY(cudaMemsetAsync(w.flags + F_BAR, 0, 2 * sizeof(int32_t), st));
    void *kargs[] = {(void *)&args};
    FOLD_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_schedule, dim3(blocks), dim3(kSchedThreads), kargs,
                                              launch_smem, st));
  }
  FOLD_LAUNCH_CHECK();

  // ---- the one host sync: flags + the level_off prefix mirrored after them, one copy into
  // a pinned staging buffer
  static thread_local int32_t *hbuf = nullptr;
  if (!hbuf) FOLD_CUDA_TRY(cudaMallocHost((void **)&hbuf, (F_NFLAGS + kLoMirror) * sizeof(int32_t)));
  const int npre = (N + 2) < kLoMirror ? (N + 2) : kLoMirror;
  FOLD_CUDA_TRY(cudaMemcpyAsync(hbuf, w.flags, (size_t)(F_NFLAGS + npre) * 4, cudaMemcpyDeviceToHost, st));
  FOLD_CUDA_TRY(cudaStreamSynchronize(st));
  const int32_t *hflags = hbuf;
  memcpy(s->level_off_host, hbuf + F_NFLAGS, (size_t)npre * 4);
  for (int e = 0; e < E_NCLASS; e++) {
    if (hflags[F_ERR0 + e] != INT_MAX) {
      g_last_detail = hflags[F_ERR0 + e];
      // error path only: the offending node's op id (and its caller-fixed level) from the
      // caller's arrays; depth stays -1 for errors found before depths exist (validation,
      // cycles) and is the caller's level for FOLD_E_LEVEL
      const int32_t id = g_last_detail;
      g_last_ctx[0] = id;
      if (e != E_ROOT && id >= 0 && id < N) {
        int32_t v[2] = {-1, -1};
        FOLD_CUDA_TRY(cudaMemcpyAsync(&v[0], gr->op + id, 4, cudaMemcpyDeviceToHost, st));
        if (e == E_LEVEL && gr->level) FOLD_CUDA_TRY(cudaMemcpyAsync(&v[1], gr->level + id, 4, cudaMemcpyDeviceToHost, st));
        FOLD_CUDA_TRY(cudaStreamSynchronize(st));
        g_last_ctx[2] = v[0];
        g_last_ctx[1] = v[1];
      }
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
  // tree-like: every row is read by at most one edge and the rows nobody reads are exactly
  // the (unconsumed) roots -- the backward can then form each child's gradient in the
  // epilogue of its single consumer's dA tile
  s->tree_like = (hflags[F_MULTI] == 0 && N - 2 * s->n_cells == hflags[F_NDISTROOT]) ? 1 : 0;
  return FOLD_OK;
}

// ---------------------------------------------------------------- multi-op host side
namespace {
struct MoWsLayout {
  SchedWs w;
  int32_t *opos, *gcnt, *tcnt, *tscan;
  size_t bytes;
};
MoWsLayout mo_ws_layout(void *base, int64_t N, int64_t G, int K, int T) {
  MoWsLayout L{};
  L.w = sched_ws_layout(base, N, G);
  size_t off = L.w.bytes;
  auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
  const size_t o_opos = take((N + 1) * 4), o_g = take(((N + 1) * K + 2) * 4);
  const size_t o_t = take(((size_t)T * (N + 2) + 2) * 4), o_ts = take(((size_t)T * (N + 2) + 2) * 4);
  L.bytes = off;
  if (base) {
    char *b = (char *)base;
    L.opos = (int32_t *)(b + o_opos); L.gcnt = (int32_t *)(b + o_g);
    L.tcnt = (int32_t *)(b + o_t); L.tscan = (int32_t *)(b + o_ts);
  }
  return L;
}
}  // namespace

bool mo_table_ok(const fold_mo_table *t) {
  if (!t || t->n_ops < 1 || t->n_ops > FOLD_MO_MAX_OPS || t->n_types < 1 || t->n_types > FOLD_MO_MAX_TYPES) return false;
  for (int i = 0; i < t->n_types; i++) if (t->S[i] < 1 || t->S[i] > 4096) return false;
  for (int o = 0; o < t->n_ops; o++) {
    const int k = t->kind[o], a = t->arity[o];
    if (t->out_type[o] < 0 || t->out_type[o] >= t->n_types) return false;
    if (k == FOLD_MO_EMBED) { if (a != 0 || t->vocab[o] < 1 || t->vocab[o] > (1 << 24)) return false; continue; }
    if (k != FOLD_MO_LSTM && k != FOLD_MO_RNN) return false;
    if (a < 1 || a > 2 || t->in_type[o] < 0 || t->in_type[o] >= t->n_types) return false;
    if (k == FOLD_MO_LSTM && t->in_type[o] != t->out_type[o]) return false;
  }
  return true;
}

size_t mo_schedule_workspace(const fold_mo_table *t, int64_t N, int64_t G) {
  if (!mo_table_ok(t)) return 0;
  return mo_ws_layout(nullptr, N < 0 ? 0 : N, G < 0 ? 0 : G, t->n_ops, t->n_types).bytes;
}

fold_status run_mo_schedule(const fold_mo_table *t, const fold_mo_graphs *gr, fold_mo_schedule_t *s, void *ws_ptr,
                            size_t ws_bytes, cudaStream_t st) {
  g_last_detail = -1;
  g_last_ctx[0] = g_last_ctx[1] = g_last_ctx[2] = -1;
  if (!mo_table_ok(t) || !gr || !s) return FOLD_E_INVALID;
  const int N = gr->n_nodes, G = gr->n_graphs, K = t->n_ops, T = t->n_types;
  if (N < 0 || G < 0) return FOLD_E_INVALID;
  s->n_nodes = N; s->n_graphs = G; s->n_levels = 0; s->n_leaf_segs = 0;
  s->op = gr->op; s->child = gr->child; s->token = gr->token; s->root = gr->root;
  if (N == 0) {
    if (G > 0) { g_last_detail = 0; g_last_ctx[0] = 0; return FOLD_E_ROOT_RANGE; }
    if (s->group_off_host) s->group_off_host[0] = 0;
    return FOLD_OK;
  }
  if (!gr->op || !gr->child || !gr->token || (G > 0 && !gr->root)) return FOLD_E_INVALID;
  if (!s->depth || !s->group_off || !s->type_off || !s->pool || !s->pool_row || !s->tlevel_off || !s->label ||
      !s->order || !s->cons_off || !s->cons_edge || !s->root_off || (G > 0 && !s->root_graph) || !s->leaf_seg ||
      !s->leaf_order || !s->group_off_host)
    return FOLD_E_INVALID;
  MoWsLayout L = mo_ws_layout(ws_ptr, N, G, K, T);
  if (!ws_ptr || ws_bytes < L.bytes) return FOLD_E_WORKSPACE;
  const size_t dsmem = (size_t)(kSchedWarps * (kMaxBins + 1) + 2 * kMaxBins + 64) * sizeof(int);
  static thread_local int max_blocks_dev[kMaxDevices] = {};
  const int dev = cur_dev();
  int &max_blocks = max_blocks_dev[dev];
  if (!max_blocks) {
    int nsm, occ = 0;
    FOLD_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    FOLD_CUDA_TRY(cudaFuncSetAttribute(k_mo_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
    FOLD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mo_schedule, kSchedThreads, dsmem));
    if (occ < 1) occ = 1;
    max_blocks = nsm * (occ < 2 ? occ : 2);
    if (max_blocks > kMaxSchedBlocks) max_blocks = kMaxSchedBlocks;
  }
  // nodes per block (FOLD_MO_SCHED_PER_BLOCK; measured on C6 B=1024, 87k nodes: 2048 -> 0.75 ms,
  // 512 -> 1.00, 8192 -> 1.21: the depth rounds' grid barriers cost more with more blocks)
  static const int mo_per_block = [] {
    const char *e = getenv("FOLD_MO_SCHED_PER_BLOCK");
    const int v = e ? atoi(e) : 2048;
    return v < 128 ? 128 : v;
  }();
  int blocks = N <= kOneBlockN ? 1 : (int)cdiv(N, mo_per_block);
  if (blocks > max_blocks) blocks = max_blocks;
  MoSchedArgs args{};
  args.N = N; args.G = G; args.K = K; args.T = T;
  for (int o = 0; o < K; o++) {
    args.kind[o] = t->kind[o]; args.arity[o] = t->arity[o]; args.in_type[o] = t->in_type[o];
    args.out_type[o] = t->out_type[o]; args.vocab[o] = t->vocab[o];
  }
  args.op = gr->op; args.child = gr->child; args.token = gr->token; args.root = gr->root;
  args.s = *s; args.w = L.w;
  args.opos = L.opos; args.gcnt = L.gcnt; args.tcnt = L.tcnt; args.tscan = L.tscan;
  if (blocks == 1) {
    k_mo_schedule<<<1, kSchedThreads, dsmem, st>>>(args);
  } else {
    FOLD_CUDA_TRY(cudaMemsetAsync(L.w.flags + F_BAR, 0, 2 * sizeof(int32_t), st));
    void *kargs[] = {(void *)&args};
    FOLD_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_mo_schedule, dim3(blocks), dim3(kSchedThreads), kargs,
                                              dsmem, st));
  }
  FOLD_LAUNCH_CHECK();
  // the one host sync: flags + the group_off prefix mirrored after them
  static thread_local int32_t *hbuf = nullptr;
  if (!hbuf) FOLD_CUDA_TRY(cudaMallocHost((void **)&hbuf, (F_NFLAGS + kLoMirror) * sizeof(int32_t)));
  const int64_t cap = (int64_t)(N + 1) * K + 1;
  const int npre = (int)(cap < kLoMirror ? cap : kLoMirror);
  FOLD_CUDA_TRY(cudaMemcpyAsync(hbuf, L.w.flags, (size_t)(F_NFLAGS + npre) * 4, cudaMemcpyDeviceToHost, st));
  FOLD_CUDA_TRY(cudaStreamSynchronize(st));
  for (int e = 0; e < MOE_NCLASS; e++) {
    if (hbuf[F_ERR0 + e] != INT_MAX) {
      g_last_detail = hbuf[F_ERR0 + e];
      g_last_ctx[0] = g_last_detail;
      if (e != MOE_ROOT && g_last_detail >= 0 && g_last_detail < N) {
        int32_t v = -1;
        FOLD_CUDA_TRY(cudaMemcpyAsync(&v, gr->op + g_last_detail, 4, cudaMemcpyDeviceToHost, st));
        FOLD_CUDA_TRY(cudaStreamSynchronize(st));
        g_last_ctx[2] = v;
      }
      return kMoErrStatus[e];
    }
  }
  const int D = hbuf[F_MAXDEPTH];
  const int ng = (D + 1) * K + 1;
  if (ng <= npre) {
    memcpy(s->group_off_host, hbuf + F_NFLAGS, (size_t)ng * 4);
  } else {
    FOLD_CUDA_TRY(cudaMemcpyAsync(s->group_off_host, s->group_off, (size_t)ng * 4, cudaMemcpyDeviceToHost, st));
    FOLD_CUDA_TRY(cudaStreamSynchronize(st));
  }
  s->n_levels = D;
  s->n_leaf_segs = hbuf[F_NSEG];
  return FOLD_OK;
}

}  // namespace fold

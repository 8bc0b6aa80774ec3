// exec_tc.cu — tcgen05 (5th-gen tensor core) kernels for the BF16 path.
//
//  k_fwd_levels    every cell level of the forward (gather -> operation ->
//                  concat, once per depth) in ONE persistent launch. The gather is moved
//                  to production time: whoever produces a pool row (embedding kernel, or
//                  this kernel's epilogue for an earlier level) also writes it into the
//                  A-operand row of each consumer edge (planes A_L / A_R, row = consumer
//                  cell). So a level's A rows are contiguous and TMA streams them as dense
//                  128B-swizzled boxes; tcgen05.mma multiplies them with a gate-interleaved
//                  slab of U into a TMEM accumulator; the epilogue warps apply the gates,
//                  append (h, c) to the level's pool rows (the concat becomes an append)
//                  and push h to its consumers' A rows. Depth order is kept by device-side
//                  level counters instead of one launch per level.
//  k_gemm_dA_tc    backward edge gradients of one level: dA = dZ_level * U.
//  k_gemm_dU_tc    weight gradient over all cells at once: dU = dZ^T * [A_L | A_R], both
//                  operands MN-major dense TMA boxes; split-K over cells with a
//                  fixed-order reduction (deterministic).
// All three run on CTA PAIRS (cluster of 2, tcgen05.mma.cta_group::2, M = 256): each CTA
// stages its 128 A rows and half of the B tile, so the operand bytes each SM pulls from L2
// per FLOP drop by a third against single-CTA 128-row tiles (measured: single-CTA tiles
// were bound by L2->SM ingress at ~56 B/clk/SM, not by the tensor pipe).
// Warp roles: warp 0 TMA producer (both CTAs), warp 1 MMA issuer (leader CTA, one lane),
// warp 2 TMEM allocator, warp 3 idle, warps 4.. epilogue (warp w reads TMEM lanes
// 32 (w % 4) .. +31 of its own CTA).
#include <atomic>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <unordered_map>

#include "exec.cuh"
#include "ptx.cuh"

namespace fold {

namespace {

// Debug timeline (FOLD_DBG_FWD=1): per tile, globaltimer stamps at five points of the
// forward pipeline (read back with fold_debug_fwd_trace; instrumentation only).
constexpr int kTraceTiles = 65536;
__device__ unsigned long long g_fwd_trace[9][kTraceTiles];
__device__ __forceinline__ void trace(int dbg, int pt, int T) {
  if (dbg && T < kTraceTiles) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fwd_trace[pt][T] = t;
  }
}
// FOLD_DBG_BWD=1: the same for k_bwd_levels at ten points (see fold_debug_bwd_trace)
__device__ unsigned long long g_bwd_trace[10][kTraceTiles];
__device__ unsigned long long g_bwd_clk[2][kTraceTiles];  // SM clock64 at points 8 and 3
__device__ __forceinline__ void btrace(int dbg, int pt, int T) {
  if (dbg && T < kTraceTiles) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_bwd_trace[pt][T] = t;
    if (pt == 8 || pt == 3) g_bwd_clk[pt == 3][T] = clock64();
  }
}

constexpr int BM = 128;     // rows per CTA (the pair's MMA has M = 256)
constexpr int PM = 2 * BM;  // rows per CTA pair
constexpr int BK = 64;      // K elements per stage (128 B of bf16 = one swizzle row)
#ifndef FOLD_DU_ST
#define FOLD_DU_ST 6
#endif
constexpr int ST = FOLD_DU_ST;  // pipeline stages (dA / dU GEMMs)
constexpr int kThreads = 256;

// (offset from the __shared__ base rather than integer casts of the pointer, so the compiler
// keeps the shared address space and emits LDS/STS instead of generic LD/ST)
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
  return p + ((1024u - (ptx::smem_u32(p) & 1023u)) & 1023u);
}

constexpr int tmem_cols_for(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}

// =================================================================== forward: all cell levels
// One persistent launch runs every cell level d = 2..D (the while-loop over
// depths, each iteration gather -> cell -> concat). Tiles are enumerated level by level
// (level d's tiles before level d+1's) and dealt round-robin to the CTAs; a tile of level
// d waits on a device counter until all tiles of level d-1 are published, so the depth
// ordering of the paper's loop is kept with no host round trip and no launch per level.
// Narrow levels use narrower state-column tiles (W_narrow) so they still spread over the
// SMs (the U slab each CTA streams shrinks with W).
struct FwdLevels {
  const int32_t *lo;     // schedule level_off (device)
  int D, S, Ww, Wn;      // deepest level, state size, wide / narrow tile widths
  int narrow_below;      // a level whose wide tiling has fewer tiles than this uses Wn
  int Wm, G, npairs;     // mid tile width, gates, CTA pairs of the launch
  int pf;                // L2 prefetch distance of the A-plane boxes in k-blocks (0: off)
};

__host__ __device__ inline int fwd_level_W(const FwdLevels &L, int M) {
  const int64_t mt = cdiv(M, PM);
  if (mt * cdiv(L.S, L.Ww) < L.narrow_below) return L.Wn;
  // wide levels: Ww unless the mid width fills the waves of CTA pairs better (a 1024-row
  // level at S = 1024 is 88 W=48 tiles = two waves on 74 pairs, or 128 W=32 tiles in the
  // same two waves of cheaper MMAs); per-MMA cost of an M=256 pair tile of N columns in
  // 1/64 cycles: max(32 N, 4096 + 16 N) (tensor issue vs shared-memory operand bytes)
  auto cost = [&](int W) {
    const int64_t N = (int64_t)L.G * W, t = mt * cdiv(L.S, W);
    const int64_t c = 32 * N > 4096 + 16 * N ? 32 * N : 4096 + 16 * N;
    return cdiv(t, (int64_t)L.npairs) * c;
  };
  return cost(L.Wm) < cost(L.Ww) ? L.Wm : L.Ww;
}

// Walks the level table in tile order (each warp role keeps its own copy).
struct LevelCursor {
  int d, t0, nt, prev_nt, r0, r1, W, NT;
  __device__ void load(const FwdLevels &L) {
    r0 = __ldg(L.lo + d); r1 = __ldg(L.lo + d + 1);
    W = fwd_level_W(L, r1 - r0);
    NT = (int)cdiv(L.S, W);
    nt = (int)cdiv(r1 - r0, PM) * NT;  // pair tiles
  }
  __device__ void init(const FwdLevels &L) { d = 2; t0 = 0; prev_nt = 0; load(L); }
  __device__ void seek(const FwdLevels &L, int T) {
    while (T >= t0 + nt) { t0 += nt; prev_nt = nt; d++; load(L); }
  }
};

template <int GATES>
struct FwdCfg {
  static constexpr int WMAX = GATES == 5 ? 48 : 128;   // wide tile: N = GATES * W <= 256
  static constexpr int WNAR = GATES == 5 ? 16 : 32;    // narrow tile (N/2 a multiple of 8 rows)
  static constexpr int WMID = GATES == 5 ? 32 : 64;    // mid tile (wave filling on 1-2-wave levels)
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = GATES * WMAX * 64;    // this CTA's half of the B rows
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static_assert(STAGE % 1024 == 0, "stages stay 1024 B aligned (128B swizzle atoms)");
  static constexpr int ACC_STRIDE = 256;  // TMEM columns per accumulator buffer (2 buffers)
  static constexpr int TMEM_COLS = 512;
  // epilogue staging: the tile's saved gates [GATES][128][W] bf16 leave through TMA bulk
  // stores (row-scattered per-thread stores of 5 gate blocks were LSU-bound); the cell
  // states (one fp32 block) are stored directly, which leaves room for a 5th stage
  static constexpr int G_STAGE = GATES * BM * WMAX * 2;
  static constexpr int C_STAGE = 0;
  // pipeline stages: as many as the rest of shared memory holds (at most 8)
  // (220 KB of dynamic shared memory: the kernel's static arrays take ~4.3 KB of the 227)
  static constexpr int NST_FIT = (220 * 1024 - G_STAGE - C_STAGE - 1024) / STAGE;
  static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
  static constexpr int SMEM = NST * STAGE + G_STAGE + C_STAGE + 1024;
  static constexpr int EPI_WARPS = 8;     // 2 per SM sub-partition: each owns half the columns
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static_assert(GATES * WMAX <= 256 && (GATES * WNAR) % 16 == 0 && (GATES * WNAR / 2) % 8 == 0, "UMMA N, M=256");
  static_assert((GATES * WMID) % 16 == 0 && (GATES * WMID / 2) % 8 == 0, "UMMA N, M=256");
  static_assert(SMEM <= 227 * 1024, "smem");
};

// k-blocks per pipeline stage of a tile: wide tiles 1; narrow tiles pack as many
// (A box of bx0 rows + U box of GATES * W / 2 rows) pairs as one stage holds, so a tile's
// K loop needs fewer round trips through the ring (narrow levels are latency bound).
template <int GATES>
__host__ __device__ inline int fwd_kps(int W, int bx0) {
  using Cfg = FwdCfg<GATES>;
  if (W == Cfg::WMAX) return 1;
  const int k = Cfg::STAGE / (bx0 * 128 + GATES * W * 64);
  return k < 1 ? 1 : k > 8 ? 8 : k;
}

// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4..11 epilogue
// (warp w reads TMEM lanes 32 (w % 4) .. +31, column chunks (w - 4) / 4, +2, +4, ...).
// B operand per stage: one box of GATES*W rows of the gate-interleaved bf16 U (Uil8: row
// (j/8)*8*GATES + g*8 + j%8 holds U row g*S + j; K halves padded to Sp = round_up(S, 64) so
// every box starts 128 B aligned): tile column jc*8*GATES + g*8 + u is gate g of state
// column j0 + 8*jc + u, for any tile width W that is a multiple of 8.
template <int GATES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(FwdCfg<GATES>::THREADS, 1)
    k_fwd_levels(const __grid_constant__ CUtensorMap tmAL, const __grid_constant__ CUtensorMap tmAR,
                 const __grid_constant__ CUtensorMap tmAL16, const __grid_constant__ CUtensorMap tmAR16,
                 const __grid_constant__ CUtensorMap tmAL64, const __grid_constant__ CUtensorMap tmAR64,
                 const __grid_constant__ CUtensorMap tmUw, const __grid_constant__ CUtensorMap tmUn,
                 const __grid_constant__ CUtensorMap tmGw, const __grid_constant__ CUtensorMap tmGn,
                 const __grid_constant__ CUtensorMap tmUm, const __grid_constant__ CUtensorMap tmGm, FwdLevels L,
                 int total_tiles, int nl, int ld, const int32_t *__restrict__ gather, const float *__restrict__ bias,
                 __nv_bfloat16 *__restrict__ H, float *C, __nv_bfloat16 *__restrict__ Gact, int ld_g, ScatterA sc,
                 int *rt_cnt, const int32_t *__restrict__ tstart, int dbg) {
  using Cfg = FwdCfg<GATES>;
  constexpr int ST = Cfg::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  uint8_t *gsm = smem + ST * Cfg::STAGE;
  __shared__ __align__(8) uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  // epilogue -> store warp hand-off: epi_done (8 epilogue warps arrive per tile), stg_free
  // (the store warp: the tile's bulk stores finished reading the staging)
  __shared__ __align__(8) uint64_t epi_done, stg_free;
  __shared__ int2 credit_list[2][8][32];  // per tile parity, per epilogue warp: (tile, credit)
  __shared__ int credit_n[2][8];          // entries, or -1: overflow (the store warp walks the rows)
  // per epilogue warp: the bias of its column chunks of the current tile (GATES x 8 floats per
  // chunk, fetched before the accumulator wait so the loads hide behind the tile's MMAs)
  __shared__ __align__(16) float bias_sm[Cfg::EPI_WARPS][GATES * Cfg::WMAX / 2];
  __shared__ uint32_t tmem_base_sh;
  const int S = L.S;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    // tempty (leader's copy used): drained by the epilogue warps of both CTAs
    for (int a = 0; a < 2; a++) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], 2 * Cfg::EPI_WARPS); }
    ptx::mbar_init(&epi_done, Cfg::EPI_WARPS);
    ptx::mbar_init(&stg_free, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmAL);
    ptx::prefetch_tmap(&tmAR);
    ptx::prefetch_tmap(&tmAL16);
    ptx::prefetch_tmap(&tmAR16);
    ptx::prefetch_tmap(&tmAL64);
    ptx::prefetch_tmap(&tmAR64);
    ptx::prefetch_tmap(&tmUw);
    ptx::prefetch_tmap(&tmUn);
    ptx::prefetch_tmap(&tmGw);
    ptx::prefetch_tmap(&tmUm);
  }
  if (warp == 2) {
    ptx::tmem_alloc2(&tmem_base_sh, Cfg::TMEM_COLS);
    ptx::tmem_relinquish2();
  }
  const float *bsrc = bias;  // 5 x 8 floats per chunk, warp-uniform (broadcast) loads
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits and the pair's TMEM allocation visible to both CTAs
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  const int KBh = (int)cdiv(S, BK), KB = 2 * KBh, Sp = KBh * BK;

  if (warp == 0) {
    // TMA producer: per stage one dense box of A rows (the level's contiguous cell rows of
    // the left / right operand plane) + one box of GATES * W / 2 rows of U. Narrow tiles
    // load only the rows they hold (16- or 64-row boxes; the MMA's other rows see stale
    // shared memory and their accumulator rows are never read). The first stages' U boxes
    // do not depend on the previous levels, so they are issued before the dependency wait.
    if (lane == 0) {
      LevelCursor cur;
      cur.init(L);
      int it = 0;
      // A-operand box rows for a CTA holding m rows (narrow tiles load only their rows)
      auto box_of = [](int m) { return m <= 0 ? 0 : m <= 16 ? 16 : m <= 64 ? 64 : BM; };
      const int pf = L.pf;
      for (int T = pair; T < total_tiles; T += npairs) {
        cur.seek(L, T);
        const int lt = T - cur.t0, W = cur.W;
        const int ct = (cur.r0 - nl) + (lt / cur.NT) * PM;  // first cell of the pair tile
        const int rows = min(PM, cur.r1 - nl - ct);
        const int bx0 = box_of(min(rows, BM)), bx1 = box_of(rows - BM), bx = rank ? bx1 : bx0;
        const CUtensorMap *mL = bx == 16 ? &tmAL16 : bx == 64 ? &tmAL64 : &tmAL;
        const CUtensorMap *mR = bx == 16 ? &tmAR16 : bx == 64 ? &tmAR64 : &tmAR;
        const int c0 = ct + (int)rank * BM, j0 = (lt % cur.NT) * W;
        // L2 prefetch of the A-plane boxes pf k-blocks ahead (the planes were pushed one level
        // earlier and mostly left L2; the column tiles of a row tile request each k-block at
        // about the same time), and of the next tile's head during this tile's last k-blocks
        const CUtensorMap *nL = nullptr, *nR = nullptr;
        int c0n = 0, bxn = 0;
        if (pf > 0 && T + npairs < total_tiles) {
          LevelCursor nx = cur;
          nx.seek(L, T + npairs);
          const int ctn = (nx.r0 - nl) + ((T + npairs - nx.t0) / nx.NT) * PM;
          const int rwn = min(PM, nx.r1 - nl - ctn);
          bxn = rank ? box_of(rwn - BM) : box_of(min(rwn, BM));
          nL = bxn == 16 ? &tmAL16 : bxn == 64 ? &tmAL64 : &tmAL;
          nR = bxn == 16 ? &tmAR16 : bxn == 64 ? &tmAR64 : &tmAR;
          c0n = ctn + (int)rank * BM;
        }
        const CUtensorMap *tmU = W == Cfg::WMAX ? &tmUw : W == Cfg::WMID ? &tmUm : &tmUn;
        if (rank == 0) trace(dbg, 0, T);
        // the leader's full barrier counts both CTAs' bytes: A rows of both + the B rows
        const uint32_t bytes = (uint32_t)(bx0 + bx1) * 128 + GATES * W * 128;
        const int urow = GATES * j0 + (int)rank * (GATES * W / 2);
        // narrow tiles pack kps k-blocks per stage (fewer pipeline round trips per tile)
        const int kps = fwd_kps<GATES>(W, bx0), abox = bx0 * 128, ubox = GATES * W * 64;
        const int nst = (KB + kps - 1) / kps;
        // inputs already published (the common case on wide levels): A and U per stage in
        // order; otherwise the first stages' U boxes go out before the wait
#ifndef FOLD_FWD_EARLY_U
        // wait for the inputs before any box of the tile (as in k_bwd_levels; FOLD_FWD_EARLY_U
        // restores the early U boxes: C4 forward 4.80 -> 5.05 ms)
        ptx::wait_counter_relaxed(rt_cnt + ct, rows * 2 * S);
#endif
        const bool ready = ptx::ld_relaxed_gpu(rt_cnt + ct) >= rows * 2 * S;
        if (ready) ptx::fence_proxy_async_global();
        const int pre = ready ? 0 : (nst < ST ? nst : ST);
        if (ready && rank == 0) trace(dbg, 1, T);
        if (ready && kps == 1) {  // wide tiles, inputs published: one (A, U) box pair per stage
          for (int kb = 0; kb < KB; kb++, it++) {
            if (pf > 0) {
              const int kp = kb + pf;
              if (kp < KB) {
                const int hp = kp >= KBh;
                if (bx) ptx::tma_prefetch_2d(hp ? mR : mL, (kp - hp * KBh) * BK, c0);
              } else if (bxn && kp - KB < KB) {
                const int kq = kp - KB, hq = kq >= KBh;
                ptx::tma_prefetch_2d(hq ? nR : nL, (kq - hq * KBh) * BK, c0n);
              }
            }
            const int s = it % ST;
            const uint32_t ph = (it / ST) & 1;
            ptx::mbar_wait(&empty[s], ph ^ 1);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], bytes);
            const int half = kb >= KBh, kc = (kb - half * KBh) * BK;
            uint8_t *A = smem + s * Cfg::STAGE;
            if (bx) ptx::tma_load_2d_pair(half ? mR : mL, &full[s], A, kc, c0);
            ptx::tma_load_2d_pair(tmU, &full[s], A + Cfg::A_BYTES, half * Sp + kc, urow);
          }
          continue;
        }
        const int uoff = kps == 1 ? Cfg::A_BYTES : kps * abox;
        for (int q = 0; q < nst; q++) {
          const int s = (it + q) % ST;
          const uint32_t ph = ((it + q) / ST) & 1;
          const int kb0 = q * kps, nk = min(kps, KB - kb0);
          uint8_t *stg = smem + s * Cfg::STAGE;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)nk * bytes);
          for (int j = 0; j < nk; j++) {
            const int kb = kb0 + j, half = kb >= KBh, kc = (kb - half * KBh) * BK;
            ptx::tma_load_2d_pair(tmU, &full[s], stg + uoff + j * ubox, half * Sp + kc, urow);
          }
          if (q < pre - 1) continue;
          if (q == pre - 1) {
            // both children's h (all S columns) pushed into every A row of this pair tile
            // (and their C rows written); the rows are read only by TMA and, after this
            // tile's MMA, through L2 by the epilogue
            ptx::wait_counter_relaxed(rt_cnt + ct, rows * 2 * S);
            ptx::fence_proxy_async_global();
            if (rank == 0) trace(dbg, 1, T);
            if (bx)
              for (int q2 = 0; q2 < pre; q2++) {
                const int s2 = (it + q2) % ST;
                for (int j = 0; j < kps && q2 * kps + j < KB; j++) {
                  const int kb = q2 * kps + j, h2 = kb >= KBh;
                  ptx::tma_load_2d_pair(h2 ? mR : mL, &full[s2], smem + s2 * Cfg::STAGE + j * abox,
                                        (kb - h2 * KBh) * BK, c0);
                }
              }
            continue;
          }
          if (bx)
            for (int j = 0; j < nk; j++) {
              const int kb = kb0 + j, half = kb >= KBh, kc = (kb - half * KBh) * BK;
              ptx::tma_load_2d_pair(half ? mR : mL, &full[s], stg + j * abox, kc, c0);
            }
        }
        it += nst;
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // converged warp, elected lane issues (ptx::elect_one)
      LevelCursor cur;
      cur.init(L);
      int it = 0, tc = 0;
      for (int T = pair; T < total_tiles; T += npairs, tc++) {
        cur.seek(L, T);
        const uint32_t idesc = ptx::idesc_bf16(PM, GATES * cur.W, 0, 0);
        const int acc = tc & 1;
        const uint32_t aph = (tc >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], aph ^ 1);
        __syncwarp();
        ptx::tc_fence_after();
        const uint32_t dst = tbase + acc * Cfg::ACC_STRIDE;
        const int ct = (cur.r0 - nl) + ((T - cur.t0) / cur.NT) * PM;
        const int rows0 = min(BM, cur.r1 - nl - ct);
        const int bx0 = rows0 <= 16 ? 16 : rows0 <= 64 ? 64 : BM;
        const int kps = fwd_kps<GATES>(cur.W, bx0), abox = bx0 * 128, ubox = GATES * cur.W * 64;
        const int nst = (KB + kps - 1) / kps;
        if (kps == 1) {  // one k-block per stage, U at the fixed offset A_BYTES
          for (int kb = 0; kb < KB; kb++, it++) {
            int s = it % ST;
            uint32_t ph = (it / ST) & 1;
            ptx::mbar_wait(&full[s], ph);
            __syncwarp();
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(smem + s * Cfg::STAGE), b0 = a0 + Cfg::A_BYTES;
            const uint64_t da = ptx::sdesc_sw128(a0, 16, 1024), db = ptx::sdesc_sw128(b0, 16, 1024);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / 16; k++)
                ptx::umma_bf16_2cta(dst, ptx::desc_add(da, 32 * k), ptx::desc_add(db, 32 * k), idesc, (kb | k) != 0);
              ptx::umma_commit_2cta(&empty[s]);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) {
            ptx::umma_commit_2cta(&tfull[acc]);
            trace(dbg, 2, T);
          }
          __syncwarp();
          continue;
        }
        for (int q = 0; q < nst; q++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&full[s], ph);
          __syncwarp();
          ptx::tc_fence_after();
          const uint32_t st0 = ptx::smem_u32(smem + s * Cfg::STAGE);
          const int nk = min(kps, KB - q * kps);
          for (int j = 0; j < nk; j++) {
            const uint64_t da = ptx::sdesc_sw128(st0 + j * abox, 16, 1024);
            const uint64_t db = ptx::sdesc_sw128(st0 + kps * abox + j * ubox, 16, 1024);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / 16; k++)
                ptx::umma_bf16_2cta(dst, ptx::desc_add(da, 32 * k), ptx::desc_add(db, 32 * k), idesc, (q | j | k) != 0);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::umma_commit_2cta(&empty[s]);
          __syncwarp();
        }
        if (ptx::elect_one()) {
          ptx::umma_commit_2cta(&tfull[acc]);
          trace(dbg, 2, T);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // Epilogue: TMEM lane = tile row; gates -> (h, c); append to the level's pool rows and
    // push h to the A-operand row of every consumer edge (the next levels' "gather").
    const int q = warp & 3;            // TMEM lane quarter
    const int grp = (warp - 4) >> 2;   // column-chunk group (0 or 1)
    const int row = q * 32 + lane;
    // per-row metadata (child rows, consumer edges) of the next tile is fetched while the
    // current tile's epilogue runs
    struct Meta { int gl, gr, ce0, ce1, e0; };
    auto fetch_meta = [&](const LevelCursor &cu, int T, Meta &m) {
      m.gl = m.gr = m.ce0 = m.ce1 = 0; m.e0 = 0;
      if (T >= total_tiles) return;
      const int64_t rr = cu.r0 + (int64_t)((T - cu.t0) / cu.NT) * PM + rank * BM + row;
      if (rr < cu.r1) {
        m.gl = __ldg(gather + 2 * rr); m.gr = __ldg(gather + 2 * rr + 1);
        m.ce0 = __ldg(sc.cons_off + rr); m.ce1 = __ldg(sc.cons_off + rr + 1);
        if (m.ce1 > m.ce0) m.e0 = __ldg(sc.cons_edge + m.ce0);
      }
    };
    LevelCursor cur, nxc;
    cur.init(L);
    nxc.init(L);
    Meta nxt;
    nxc.seek(L, pair);
    fetch_meta(nxc, pair, nxt);

    // Publication goes through the store warp (warp 3): per tile each epilogue warp fences
    // its pushes / staging writes, sums its rows' credits (h columns pushed) per consumer
    // tile into credit_list and arrives on epi_done; the store warp issues the bulk stores,
    // waits for them, fences (cumulative over the mbarrier hand-off) and adds the credits.
    // Latency-bound levels (at most 2 tiles per CTA pair): each epilogue warp publishes its
    // own rows right after its stores (fence + one atomic per distinct consumer tile), so
    // the dependency does not wait for the store warp's G bulk store; consumers need only h
    // (pushed) and c (stored directly). Wide levels keep the hand-off below (one fence per
    // tile in the store warp, the epilogue warps never block on a fence).
    auto publish = [&](int ce0, int ce1, int e0, int cols) {
      __syncwarp();
      __threadfence();
      for (int k = 0;; k++) {
        const int e = ce0 + k;
        const bool act = e < ce1 && cols > 0;
        if (!__any_sync(0xffffffffu, act)) break;
        const int ts = act ? __ldg(tstart + ((k == 0 ? e0 : __ldg(sc.cons_edge + e)) >> 1)) : -1;
        unsigned todo = __ballot_sync(0xffffffffu, act);
        while (todo) {
          const int src = __ffs(todo) - 1;
          const int key = __shfl_sync(0xffffffffu, ts, src);
          const bool mine = act && ts == key;
          const int sum = (int)__reduce_add_sync(0xffffffffu, mine ? (unsigned)cols : 0u);
          todo &= ~__ballot_sync(0xffffffffu, mine);
          if (lane == src) atomicAdd(rt_cnt + key, sum);
        }
      }
    };
    auto warp_credits = [&](int par, int ce0, int ce1, int e0, int cols) {
      const int ew = warp - 4;
      int n = 0;
      bool over = false;
      for (int k = 0; !over; k++) {
        const int e = ce0 + k;
        const bool act = e < ce1 && cols > 0;
        if (!__any_sync(0xffffffffu, act)) break;
        const int ts = act ? __ldg(tstart + ((k == 0 ? e0 : __ldg(sc.cons_edge + e)) >> 1)) : -1;
        unsigned todo = __ballot_sync(0xffffffffu, act);
        while (todo) {
          if (n == 32) { over = true; break; }
          const int src = __ffs(todo) - 1;
          const int key = __shfl_sync(0xffffffffu, ts, src);
          const bool mine = act && ts == key;
          const int sum = (int)__reduce_add_sync(0xffffffffu, mine ? (unsigned)cols : 0u);
          todo &= ~__ballot_sync(0xffffffffu, mine);
          if (lane == src) credit_list[par][ew][n] = make_int2(key, sum);
          n++;
        }
      }
      if (lane == 0) credit_n[par][ew] = over ? -1 : n;
    };
    int tc = 0;
    for (int T = pair; T < total_tiles; T += npairs, tc++) {
      cur.seek(L, T);
      const int acc = tc & 1;
      const uint32_t aph = (tc >> 1) & 1;
      const int lt = T - cur.t0, W = cur.W, chunks = W / 8;
      const int j0 = (lt % cur.NT) * W;
      const int64_t r = cur.r0 + (int64_t)(lt / cur.NT) * PM + rank * BM + row;
      const bool valid = r < cur.r1;
      const Meta m = nxt;
      if (T + npairs < total_tiles) nxc.seek(L, T + npairs);
      fetch_meta(nxc, T + npairs, nxt);
      const int64_t gl = m.gl, gr = m.gr;
      const int ce0 = m.ce0, ce1 = m.ce1;
      const int64_t c = r - nl;
      // child cell states: loaded only after the accumulator is ready (this tile's MMA ran
      // after its producer saw the children published), then one chunk ahead of the math
      float cl[8], cr[8];
      auto load_c = [&](int jb) {
        if (GATES != 5) return;
        // leaf children have c = 0 (their C rows are not materialised in BF16 mode)
        const bool lok = valid && gl >= nl, rok = valid && gr >= nl;
        if (jb + 8 <= S) {  // C rows have stride ld (a multiple of 8): 16-byte aligned
#pragma unroll
          for (int u = 0; u < 8; u++) { cl[u] = 0.f; cr[u] = 0.f; }
          if (lok) {
            float4 a = __ldcg(reinterpret_cast<const float4 *>(C + gl * ld + jb));
            float4 b = __ldcg(reinterpret_cast<const float4 *>(C + gl * ld + jb + 4));
            cl[0] = a.x; cl[1] = a.y; cl[2] = a.z; cl[3] = a.w; cl[4] = b.x; cl[5] = b.y; cl[6] = b.z; cl[7] = b.w;
          }
          if (rok) {
            float4 a = __ldcg(reinterpret_cast<const float4 *>(C + gr * ld + jb));
            float4 b = __ldcg(reinterpret_cast<const float4 *>(C + gr * ld + jb + 4));
            cr[0] = a.x; cr[1] = a.y; cr[2] = a.z; cr[3] = a.w; cr[4] = b.x; cr[5] = b.y; cr[6] = b.z; cr[7] = b.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; u++) {
            cl[u] = (lok && jb + u < S) ? __ldcg(C + gl * ld + jb + u) : 0.f;
            cr[u] = (rok && jb + u < S) ? __ldcg(C + gr * ld + jb + u) : 0.f;
          }
        }
      };
      // full-width tiles stage G and C in shared memory and leave by TMA (partial tiles at
      // the S edge store directly)
      const int64_t c_tile = (int64_t)(cur.r0 - nl) + (int64_t)(lt / cur.NT) * PM + rank * BM;
      // (the bulk stores never write past the level's last row: a later level's tile may
      // already own those rows)
      const bool staged = j0 + W <= S && c_tile + BM <= cur.r1 - nl;
      float *bw = bias_sm[warp - 4];
      {
        const int nchw = (chunks - grp + 1) / 2;  // this warp's chunks jc = grp, grp + 2, ...
        for (int i = lane; i < nchw * GATES * 8; i += 32) {
          const int cl = i / (GATES * 8), rem = i - cl * (GATES * 8), g = rem >> 3, u = rem & 7;
          const int jj = j0 + (grp + 2 * cl) * 8 + u;
          bw[i] = jj < S ? __ldg(bsrc + g * S + jj) : 0.f;
        }
        __syncwarp();
      }
      // the children's cell states of the first chunk are loaded while the tile's MMAs run:
      // once this warp itself has observed the tile's inputs published (acquire), not only
      // after the accumulator is ready (on latency-bound levels the L2 round trip was on every
      // level's critical path)
      {
        const int ct = (cur.r0 - nl) + (lt / cur.NT) * PM;
        if (lane == 0) ptx::wait_counter(rt_cnt + ct, min(PM, cur.r1 - nl - ct) * 2 * S);
        __syncwarp();
      }
      load_c(j0 + grp * 8);
      ptx::mbar_wait(&tfull[acc], aph);
      ptx::tc_fence_after();
      if (warp == 4 && lane == 0 && rank == 0) trace(dbg, 3, T);
      if (tc > 0) ptx::mbar_wait(&stg_free, (tc - 1) & 1);  // previous tile's staging consumed
      if (warp == 4 && lane == 0 && rank == 0) trace(dbg, 5, T);
      const uint32_t tl = tbase + acc * Cfg::ACC_STRIDE + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int jc = grp; jc < chunks; jc += 2) {
        float z[GATES][8];
#pragma unroll
        for (int g = 0; g < GATES; g++) ptx::tmem_ld8(tl + jc * 8 * GATES + g * 8, z[g]);
        ptx::tmem_ld_wait();
        const int jb = j0 + jc * 8;
        float ccl[8], ccr[8];
#pragma unroll
        for (int u = 0; u < 8; u++) { ccl[u] = cl[u]; ccr[u] = cr[u]; }
        if (jc + 2 < chunks) load_c(jb + 16);  // next chunk of this warp, in flight during math
        if (!valid || jb >= S) continue;
        // full 8-column chunk: H / C / A rows (stride ld) and G gate blocks (stride ld) are
        // 16-byte aligned for any S; the bias gate blocks (stride S) only when S % 4 == 0
        const bool fullc = jb + 8 <= S;
        float hh[8];
        if constexpr (GATES == 1) {
#pragma unroll
          for (int u = 0; u < 8; u++) hh[u] = tanh_fast(z[0][u] + bw[((jc - grp) >> 1) * 8 + u]);
          if (staged) {
            uint4 pk = make_uint4(pack_bf16x2(hh[0], hh[1]), pack_bf16x2(hh[2], hh[3]), pack_bf16x2(hh[4], hh[5]),
                                  pack_bf16x2(hh[6], hh[7]));
            *reinterpret_cast<uint4 *>(gsm + row * W * 2 + jc * 16) = pk;
            *reinterpret_cast<float4 *>(C + r * ld + jb) = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4 *>(C + r * ld + jb + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
          } else if (fullc) {
            uint4 pk = make_uint4(pack_bf16x2(hh[0], hh[1]), pack_bf16x2(hh[2], hh[3]), pack_bf16x2(hh[4], hh[5]),
                                  pack_bf16x2(hh[6], hh[7]));
            *reinterpret_cast<uint4 *>(Gact + c * ld_g + jb) = pk;
            *reinterpret_cast<float4 *>(C + r * ld + jb) = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4 *>(C + r * ld + jb + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            for (int u = 0; u < 8 && jb + u < S; u++) {
              Gact[c * ld_g + jb + u] = __float2bfloat16_rn(hh[u]);
              C[r * ld + jb + u] = 0.f;
            }
          }
        } else {
          float gs[5][8], cc[8];
          const float *bc = bw + ((jc - grp) >> 1) * (GATES * 8);
#pragma unroll
          for (int g = 0; g < 5; g++) {
            float bz[8];
            const float4 x = *reinterpret_cast<const float4 *>(bc + g * 8);
            const float4 y = *reinterpret_cast<const float4 *>(bc + g * 8 + 4);
            bz[0] = x.x; bz[1] = x.y; bz[2] = x.z; bz[3] = x.w; bz[4] = y.x; bz[5] = y.y; bz[6] = y.z; bz[7] = y.w;
#pragma unroll
            for (int u = 0; u < 8; u++) gs[g][u] = g == 4 ? tanh_fast(z[g][u] + bz[u]) : sigmoid_fast(z[g][u] + bz[u]);
          }
#pragma unroll
          for (int u = 0; u < 8; u++) {
            cc[u] = gs[0][u] * gs[4][u] + gs[1][u] * ccl[u] + gs[2][u] * ccr[u];
            hh[u] = gs[3][u] * tanh_fast(cc[u]);
          }
          __nv_bfloat16 *ga = Gact + c * ld_g;
          if (staged) {
            *reinterpret_cast<float4 *>(C + r * ld + jb) = make_float4(cc[0], cc[1], cc[2], cc[3]);
            *reinterpret_cast<float4 *>(C + r * ld + jb + 4) = make_float4(cc[4], cc[5], cc[6], cc[7]);
#pragma unroll
            for (int g = 0; g < 5; g++)
              *reinterpret_cast<uint4 *>(gsm + (g * BM + row) * W * 2 + jc * 16) =
                  make_uint4(pack_bf16x2(gs[g][0], gs[g][1]), pack_bf16x2(gs[g][2], gs[g][3]),
                             pack_bf16x2(gs[g][4], gs[g][5]), pack_bf16x2(gs[g][6], gs[g][7]));
          } else if (fullc) {
            *reinterpret_cast<float4 *>(C + r * ld + jb) = make_float4(cc[0], cc[1], cc[2], cc[3]);
            *reinterpret_cast<float4 *>(C + r * ld + jb + 4) = make_float4(cc[4], cc[5], cc[6], cc[7]);
#pragma unroll
            for (int g = 0; g < 5; g++)
              *reinterpret_cast<uint4 *>(ga + g * ld + jb) =
                  make_uint4(pack_bf16x2(gs[g][0], gs[g][1]), pack_bf16x2(gs[g][2], gs[g][3]),
                             pack_bf16x2(gs[g][4], gs[g][5]), pack_bf16x2(gs[g][6], gs[g][7]));
          } else {
            for (int u = 0; u < 8 && jb + u < S; u++) {
              int j = jb + u;
              C[r * ld + j] = cc[u];
#pragma unroll
              for (int g = 0; g < 5; g++) ga[g * ld + j] = __float2bfloat16_rn(gs[g][u]);
            }
          }
        }
        // h: every consumer's A-operand row (push-gather); rows without consumers (roots,
        // dead nodes) are appended to the H pool instead
        if (fullc) {
          uint4 pk = make_uint4(pack_bf16x2(hh[0], hh[1]), pack_bf16x2(hh[2], hh[3]), pack_bf16x2(hh[4], hh[5]),
                                pack_bf16x2(hh[6], hh[7]));
          if (ce1 == ce0) *reinterpret_cast<uint4 *>(H + r * ld + jb) = pk;
          for (int e = ce0; e < ce1; e++) {
            int ed = e == ce0 ? m.e0 : __ldg(sc.cons_edge + e);
            *reinterpret_cast<uint4 *>(((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld + jb) = pk;
          }
        } else {
          for (int u = 0; u < 8 && jb + u < S; u++) {
            __nv_bfloat16 hv = __float2bfloat16_rn(hh[u]);
            if (ce1 == ce0) H[r * ld + jb + u] = hv;
            for (int e = ce0; e < ce1; e++) {
              int ed = __ldg(sc.cons_edge + e);
              (((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld)[jb + u] = hv;
            }
          }
        }
      }
      // this accumulator buffer may be overwritten by the MMA of tile i+2 (the leader's
      // barrier collects both CTAs' epilogue warps)
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_leader(&tempty[acc]);
      // hand the tile to the store warp
      ptx::fence_proxy_async_smem();
      ptx::fence_proxy_async_global();
      int cols = 0;
      if (valid)
        for (int jc = grp; jc < chunks; jc += 2) cols += max(0, min(8, S - (j0 + jc * 8)));
      if (cur.nt <= 2 * npairs) {  // latency-bound level: publish here
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&epi_done);
        publish(ce0, ce1, m.e0, cols);
      } else {
        warp_credits(tc & 1, ce0, ce1, m.e0, cols);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&epi_done);
      }
      if (warp == 4 && lane == 0 && rank == 0) trace(dbg, 6, T);
    }
  } else if (warp == 3) {
    // Store warp: bulk stores of the staged G / C tiles, then the tile's publication.
    if (lane == 0) {
      LevelCursor cur;
      cur.init(L);
      int tc = 0;
      for (int T = pair; T < total_tiles; T += npairs, tc++) {
        cur.seek(L, T);
        const int lt = T - cur.t0, W = cur.W, chunks = W / 8;
        const int j0 = (lt % cur.NT) * W;
        const int64_t c_tile = (int64_t)(cur.r0 - nl) + (int64_t)(lt / cur.NT) * PM + rank * BM;
        const bool staged = j0 + W <= S && c_tile + BM <= cur.r1 - nl;
        ptx::mbar_wait(&epi_done, tc & 1);
        if (staged) {
          const CUtensorMap *tG = W == Cfg::WMAX ? &tmGw : W == Cfg::WMID ? &tmGm : &tmGn;
#pragma unroll
          for (int g = 0; g < GATES; g++) ptx::tma_store_2d(tG, gsm + g * BM * W * 2, g * ld + j0, (int)c_tile);
          ptx::bulk_commit();
          ptx::bulk_wait_read0();
        }
        if (rank == 0) trace(dbg, 7, T);
        ptx::mbar_arrive(&stg_free);
        // (the staged G rows are read only by the backward, after this kernel; the C rows
        // the consumers read were stored by the epilogue threads, ordered by the fence below
        // or by the epilogue warps' own fences on latency-bound levels)
        if (rank == 0) trace(dbg, 8, T);
        if (cur.nt <= 2 * npairs) {  // the epilogue warps published this tile themselves
          if (rank == 0) trace(dbg, 4, T);
          continue;
        }
        __threadfence();
        const int par = tc & 1;
        for (int w = 0; w < Cfg::EPI_WARPS; w++) {
          const int n = credit_n[par][w];
          if (n >= 0) {
            for (int i = 0; i < n; i++) atomicAdd(rt_cnt + credit_list[par][w][i].x, credit_list[par][w][i].y);
          } else {  // overflow (wide DAG fan-out): walk warp w's 32 rows edge by edge
            const int grp = w >> 2;
            int cols = 0;
            for (int jc = grp; jc < chunks; jc += 2) cols += max(0, min(8, S - (j0 + jc * 8)));
            for (int i = 0; i < 32 && cols > 0; i++) {
              const int64_t r = cur.r0 + (int64_t)(lt / cur.NT) * PM + rank * BM + (w & 3) * 32 + i;
              if (r >= cur.r1) break;
              for (int e = __ldg(sc.cons_off + r); e < __ldg(sc.cons_off + r + 1); e++)
                atomicAdd(rt_cnt + __ldg(tstart + (__ldg(sc.cons_edge + e) >> 1)), cols);
            }
          }
        }
        if (rank == 0) trace(dbg, 4, T);
      }
      ptx::bulk_wait0();  // the last G bulk stores are complete before the CTA exits
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // neither CTA leaves while the pair's MMAs / arrivals may touch it
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tbase, Cfg::TMEM_COLS);
  }
}

// =================================================================== forward: narrow tail levels
// Levels with at most a few rows (the tops of trees, chains, single trees) are latency
// bound: in k_fwd_levels every such level still streams its U slab through shared memory
// and runs M = 256 MMAs for a handful of rows. k_fwd_narrow keeps U STATIONARY instead and
// swaps the operands: CTA x owns state columns [8x, 8x + 8) and holds their GATES * 8
// gate-interleaved U rows (all 2S inputs) in shared memory for the whole kernel; per chunk
// of <= 8 rows of a level it loads only the chunk's A rows (8 x 2S bf16) and computes
// Z^T = U_x * A^T with one CTA (cta_group::1). An SS-mode MMA costs about its operand bytes
// read from shared memory, dominated by the M = 128 U operand, so the two K halves (h_L and
// h_R inputs) are stacked in M: slot q holds U_x[:, K-block q of h_L] in rows 0..UROWS-1 and
// U_x[:, K-block q of h_R] in rows UROWS..2 UROWS-1 (rows past that alias the next slot and
// are never read back), the B operand holds the chunk's h_L K-block q in rows 0..7 and its
// h_R K-block q in rows 8..15 (SBO = the distance between the halves), so one M = 128,
// N = 16 MMA per 16 K advances both halves: Z = D[0:UROWS, 0:8] + D[UROWS:2 UROWS, 8:16],
// S/16 MMAs per chunk instead of 2S/16. The epilogue (three warps = TMEM lanes 0..95)
// regroups the gates of each (state column, row) through shared memory, applies the cell,
// appends c / G, pushes h to the consumers' A rows and publishes h-column credits exactly
// like k_fwd_levels, so the two kernels share the dependency counters (this one runs after
// it, on the remaining levels d0..D).
constexpr int NW_ROWS = 8;          // rows per chunk
constexpr int NW_THREADS = 224;     // warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4-6 epilogue
constexpr int NW_MAX_S = 1024;      // U slice (GATES*8 rows x 2S) + A chunk fit in shared memory

template <int GATES>
struct NwCfg {
  static constexpr int UROWS = GATES * 8;               // U rows per CTA (per K half)
  static constexpr int USLOT = 2 * UROWS * 128;         // bytes per K-block slot (both halves)
  static constexpr int SLACK = (16 - 2 * UROWS / 8) * 1024; // the M = 128 operand reads 16 8-row groups
  static constexpr int BKB = NW_ROWS * 128;             // bytes per K-block of the A chunk
  static int smem(int KBh) { return 2 * KBh * BKB + KBh * USLOT + SLACK + 1024; }
  static_assert(2 * UROWS <= 96, "both halves' U rows are read by TMEM lane quarters 0..2");
};

template <int GATES>
__global__ void __launch_bounds__(NW_THREADS, 1)
    k_fwd_narrow(const __grid_constant__ CUtensorMap tmUs, const __grid_constant__ CUtensorMap tmAL8,
                 const __grid_constant__ CUtensorMap tmAR8, const __grid_constant__ CUtensorMap tmA4, int use3d,
                 const int32_t *__restrict__ lo, int d0, int D, int S,
                 int nl, int ld, const int32_t *__restrict__ gather, const float *__restrict__ bias,
                 __nv_bfloat16 *__restrict__ H, float *C, __nv_bfloat16 *__restrict__ Gact, int ld_g, ScatterA sc,
                 int *rt_cnt, const int32_t *__restrict__ tstart, int dbg) {
  using Cfg = NwCfg<GATES>;
  dbg = dbg && blockIdx.x == 0;  // timeline of CTA 0 only
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  const int KBh = (int)cdiv(S, BK), KB = 2 * KBh, Sp = KBh * BK;
  uint8_t *Bsm = smem, *Usm = smem + KB * Cfg::BKB;  // B: [slot][half][8 rows]; U: [slot][half][UROWS]
  __shared__ __align__(8) uint64_t u_full, b_full, b_empty, acc_full[2], acc_empty[2];
  __shared__ float zs[2][GATES * 8][NW_ROWS + 1];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j0 = blockIdx.x * 8;
  const int ncols = min(8, S - j0);
  if (tid == 0) {
    ptx::mbar_init(&u_full, 1);
    ptx::mbar_init(&b_full, 1);
    ptx::mbar_init(&b_empty, 1);
    for (int a = 0; a < 2; a++) { ptx::mbar_init(&acc_full[a], 1); ptx::mbar_init(&acc_empty[a], 3); }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmUs);
    ptx::prefetch_tmap(&tmAL8);
    ptx::prefetch_tmap(&tmAR8);
    ptx::prefetch_tmap(&tmA4);
  }
  if (warp == 2) { ptx::tmem_alloc(&tmem_base_sh, 32); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;

  // chunk walk (every role keeps its own cursor): level d, rows [r, r + rows)
  struct Cur {
    int d, r, r1;
    __device__ void init(const int32_t *lo, int d0) { d = d0; r = __ldg(lo + d); r1 = __ldg(lo + d + 1); }
    __device__ bool next(const int32_t *lo, int D) {  // advance to the next chunk
      r += NW_ROWS;
      while (r >= r1) {
        if (++d > D) return false;
        r = __ldg(lo + d); r1 = __ldg(lo + d + 1);
      }
      return true;
    }
    __device__ bool valid(const int32_t *lo, int D) {  // skip empty leading levels
      while (r >= r1) {
        if (++d > D) return false;
        r = __ldg(lo + d); r1 = __ldg(lo + d + 1);
      }
      return true;
    }
  };
  // a chunk's inputs are complete once its 256-row tile has all 2S h columns of its rows
  auto tile_target = [&](const Cur &cu, int &key) {
    const int c = cu.r - nl;
    key = __ldg(tstart + c);
    const int tend = min(key + PM, cu.r1 - nl);
    return (tend - key) * 2 * S;
  };

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(&u_full, (uint32_t)(KBh * Cfg::USLOT));
      for (int kb = 0; kb < KB; kb++) {
        const int half = kb >= KBh, q = kb - half * KBh;
        ptx::tma_load_2d(&tmUs, &u_full, Usm + q * Cfg::USLOT + half * (Cfg::USLOT / 2), half * Sp + q * BK,
                         blockIdx.x * Cfg::UROWS);
      }
      Cur cu;
      cu.init(lo, d0);
      int i = 0;
      for (bool ok = cu.valid(lo, D); ok; ok = cu.next(lo, D), i++) {
        if (i > 0) ptx::mbar_wait(&b_empty, (i - 1) & 1);
        trace(dbg, 0, i);
        int key;
        const int target = tile_target(cu, key);
        ptx::wait_counter_relaxed(rt_cnt + key, target);
        ptx::fence_proxy_async_global();
        trace(dbg, 1, i);
        ptx::mbar_arrive_expect_tx(&b_full, (uint32_t)(KB * Cfg::BKB));
        const int c0 = cu.r - nl;
        if (use3d) {  // one 4D box: the chunk's 8 rows x both halves x all K-blocks
          ptx::tma_load_4d(&tmA4, &b_full, Bsm, 0, c0, 0, 0);
        } else {
          for (int kb = 0; kb < KB; kb++) {
            const int half = kb >= KBh, q = kb - half * KBh;
            ptx::tma_load_2d(half ? &tmAR8 : &tmAL8, &b_full, Bsm + (2 * q + half) * Cfg::BKB, q * BK, c0);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // converged warp, elected lane issues (ptx::elect_one)
      constexpr uint32_t idesc = ptx::idesc_bf16(128, 2 * NW_ROWS, 0, 0);
      ptx::mbar_wait(&u_full, 0);
      Cur cu;
      cu.init(lo, d0);
      int i = 0;
      const uint64_t du = ptx::sdesc_sw128(ptx::smem_u32(Usm), 16, 1024);
      const uint64_t dbb = ptx::sdesc_sw128(ptx::smem_u32(Bsm), 16, 1024);
      for (bool ok = cu.valid(lo, D); ok; ok = cu.next(lo, D), i++) {
        const int acc = i & 1;
        ptx::mbar_wait(&acc_empty[acc], ((i >> 1) & 1) ^ 1);
        ptx::mbar_wait(&b_full, i & 1);
        __syncwarp();
        ptx::tc_fence_after();
        if (lane == 0) trace(dbg, 7, i);
        const uint32_t dst = tbase + acc * 2 * NW_ROWS;
        for (int q = 0; q < KBh; q++) {  // B rows 0..7: h_L K-block q, rows 8..15: h_R K-block q
          const uint64_t dq = ptx::desc_add(du, q * Cfg::USLOT), bq = ptx::desc_add(dbb, 2 * q * Cfg::BKB);
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; k++)
              ptx::umma_bf16(dst, ptx::desc_add(dq, 32 * k), ptx::desc_add(bq, 32 * k), idesc, (q | k) != 0);
          }
          __syncwarp();
        }
        if (ptx::elect_one()) {
          ptx::umma_commit(&b_empty);
          ptx::umma_commit(&acc_full[acc]);
          trace(dbg, 2, i);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int t = tid - 128;          // 0..95 (the math uses 0..63)
    const int q = warp & 3;           // TMEM lane quarter 0 / 1 / 2
    const int n = t >> 3, u = t & 7;  // this thread's (row in chunk, state column) in the math
    const int j = j0 + u;
    Cur cu;
    cu.init(lo, d0);
    int i = 0;
    for (bool ok = cu.valid(lo, D); ok; ok = cu.next(lo, D), i++) {
      const int acc = i & 1;
      const int rows = min(NW_ROWS, cu.r1 - cu.r);
      const int64_t r = cu.r + n;
      const bool act = n < rows && u < ncols;
      // children's c (published with their h): fetched while the MMA runs
      int64_t gl = 0, gr = 0;
      float cl = 0.f, cr = 0.f;
      if (act) {
        gl = __ldg(gather + 2 * r);
        gr = __ldg(gather + 2 * r + 1);
        if (GATES == 5 && (gl >= nl || gr >= nl)) {
          int key;
          const int target = tile_target(cu, key);
          ptx::wait_counter(rt_cnt + key, target);
          if (gl >= nl) cl = __ldcg(C + gl * ld + j);
          if (gr >= nl) cr = __ldcg(C + gr * ld + j);
        }
      }
      if (t == 0) trace(dbg, 5, i);
      ptx::mbar_wait(&acc_full[acc], (i >> 1) & 1);
      ptx::tc_fence_after();
      if (t == 0) trace(dbg, 3, i);
      float z0[8], z1[8];
      const int m = q * 32 + lane;  // D row = stacked U row
      const int hf = m >= Cfg::UROWS;   // which K half this row accumulated
      // its half's 8 columns: rows < UROWS pair with B rows 0..7, the next UROWS with 8..15
      // (tcgen05.ld addresses are warp-uniform: read both and select per lane)
      const uint32_t ta = tbase + acc * 2 * NW_ROWS + ((uint32_t)(q * 32) << 16);
      ptx::tmem_ld8(ta, z0);
      ptx::tmem_ld8(ta + NW_ROWS, z1);
      ptx::tmem_ld_wait();
      if (m < 2 * Cfg::UROWS)
#pragma unroll
        for (int k = 0; k < NW_ROWS; k++) zs[hf][m - hf * Cfg::UROWS][k] = hf ? z1[k] : z0[k];
      ptx::tc_fence_before();
      ptx::named_bar_sync(1, 96);
      if (lane == 0) ptx::mbar_arrive(&acc_empty[acc]);
      if (act) {
        const int64_t c = r - nl;
        float hh;
        if constexpr (GATES == 1) {
          hh = tanh_fast(zs[0][u][n] + zs[1][u][n] + __ldg(bias + j));
          C[r * ld + j] = 0.f;
          Gact[c * ld_g + j] = __float2bfloat16_rn(hh);
        } else {
          float gs[5];
#pragma unroll
          for (int g = 0; g < 5; g++) {
            const float x = zs[0][g * 8 + u][n] + zs[1][g * 8 + u][n] + __ldg(bias + g * S + j);
            gs[g] = g == 4 ? tanh_fast(x) : sigmoid_fast(x);
          }
          const float cc = gs[0] * gs[4] + gs[1] * cl + gs[2] * cr;
          hh = gs[3] * tanh_fast(cc);
          C[r * ld + j] = cc;
#pragma unroll
          for (int g = 0; g < 5; g++) Gact[c * ld_g + g * ld + j] = __float2bfloat16_rn(gs[g]);
        }
        const __nv_bfloat16 hv = __float2bfloat16_rn(hh);
        const int e0 = __ldg(sc.cons_off + r), e1 = __ldg(sc.cons_off + r + 1);
        if (e0 == e1) H[r * ld + j] = hv;
        for (int e = e0; e < e1; e++) {
          const int ed = __ldg(sc.cons_edge + e);
          (((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld)[j] = hv;
        }
      }
      ptx::fence_proxy_async_global();
      ptx::named_bar_sync(1, 96);
      if (t == 0) trace(dbg, 6, i);
      // publish: h columns [j0, j0 + ncols) of every row of the chunk, per consumer edge
      if (t < rows) {
        const int64_t rr = cu.r + t;
        const int e0 = __ldg(sc.cons_off + rr), e1 = __ldg(sc.cons_off + rr + 1);
        if (e1 > e0) __threadfence();
        for (int e = e0; e < e1; e++) atomicAdd(rt_cnt + __ldg(tstart + (__ldg(sc.cons_edge + e) >> 1)), ncols);
      }
      if (t == 0) trace(dbg, 4, i);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 32); }
}

// =================================================================== dA = dZ * U (one level)
// B operand = the bf16 U in its natural row order [gates*S][2*Sp] read MN-major (N = the
// padded input columns contiguous, K = the gates*S rows): no transposed copy is needed.
// CTA pairs, persistent (grid = 2 * min(#pair tiles, #pairs)); pair tile t -> (N tile
// t % NTn, 256-row tile t / NTn); each CTA stages its 128 dZ rows and 128 of the 256 B
// columns; two TMEM accumulators so the fp32 store epilogue of tile i overlaps the main
// loop of tile i+1.
constexpr int DA_N = 256;
constexpr int MN_CHUNK = 64 * 128;       // bytes per 64-element MN chunk of 64 K rows
constexpr int DA_A_BYTES = BM * 128, DA_B_BYTES = (DA_N / 2) * 128, DA_STAGE = DA_A_BYTES + DA_B_BYTES;
constexpr int DA_SMEM = ST * DA_STAGE + 1024;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_dA_tc(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmU, int c0, int M,
                 int KB, int S, int NTn, int ntiles, float *__restrict__ dA) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], 2 * 4); }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmZ);
    ptx::prefetch_tmap(&tmU);
  }
  if (warp == 2) { ptx::tmem_alloc2(&tmem_base_sh, 512); ptx::tmem_relinquish2(); }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        const int mt = c0 + (t / NTn) * PM + (int)rank * BM, nb = (t % NTn) * DA_N + (int)rank * (DA_N / 2);
        for (int kb = 0; kb < KB; kb++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * DA_STAGE);
          uint8_t *A = smem + s * DA_STAGE;
          ptx::tma_load_2d_pair(&tmZ, &full[s], A, kb * BK, mt);
#pragma unroll
          for (int ch = 0; ch < DA_N / 128; ch++)
            ptx::tma_load_2d_pair(&tmU, &full[s], A + DA_A_BYTES + ch * MN_CHUNK, nb + ch * 64, kb * BK);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // converged warp, elected lane issues (ptx::elect_one)
      constexpr uint32_t idesc = ptx::idesc_bf16(PM, DA_N, 0, 1);
      int it = 0, tc = 0;
      for (int t = pair; t < ntiles; t += npairs, tc++) {
        const int acc = tc & 1;
        ptx::mbar_wait(&tempty[acc], ((tc >> 1) & 1) ^ 1);
        __syncwarp();
        ptx::tc_fence_after();
        const uint32_t dst = tbase + acc * 256;
        for (int kb = 0; kb < KB; kb++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&full[s], ph);
          __syncwarp();
          ptx::tc_fence_after();
          const uint32_t a0 = ptx::smem_u32(smem + s * DA_STAGE), b0 = a0 + DA_A_BYTES;
          const uint64_t da = ptx::sdesc_sw128(a0, 16, 1024), db = ptx::sdesc_sw128(b0, MN_CHUNK, 1024);
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; k++)
              ptx::umma_bf16_2cta(dst, ptx::desc_add(da, 32 * k), ptx::desc_add(db, 2048 * k), idesc, (kb | k) != 0);
            ptx::umma_commit_2cta(&empty[s]);
          }
          __syncwarp();
        }
        if (ptx::elect_one()) ptx::umma_commit_2cta(&tfull[acc]);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int N2 = 2 * S, Sp = (int)round_up(S, BK);
    int tc = 0;
    for (int t = pair; t < ntiles; t += npairs, tc++) {
      const int acc = tc & 1;
      const int mt = c0 + (t / NTn) * PM + (int)rank * BM, n0 = (t % NTn) * DA_N;
      const int row = q * 32 + lane;
      const int64_t c = mt + row;
      const bool valid = (c - c0) < M;
      float *out = dA + c * N2;
      ptx::mbar_wait(&tfull[acc], (tc >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tl = tbase + acc * 256 + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int nc = 0; nc < DA_N / 8; nc++) {
        float v[8];
        ptx::tmem_ld8(tl + nc * 8, v);
        ptx::tmem_ld_wait();
        // padded B column n' = half * Sp + col  ->  dA column half * S + col (col < S)
        const int np = n0 + nc * 8, half = np >= Sp, col = np - half * Sp;
        if (!valid || col >= S) continue;
        const int n = half * S + col;
        if (col + 8 <= S && (S & 3) == 0) {
          *reinterpret_cast<float4 *>(out + n) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4 *>(out + n + 4) = make_float4(v[4], v[5], v[6], v[7]);
        } else {
          for (int u = 0; u < 8 && col + u < S; u++) out[n + u] = v[u];
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_leader(&tempty[acc]);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, 512); }
}

// =================================================================== backward: all cell levels
// Tree-like schedules (every row read by at most one edge, unread rows = roots): ONE
// persistent launch runs the dA GEMM of every level d = D..2 (the reverse
// sweep), and each tile's epilogue turns the edge gradients dA[e] straight into the child's
// backward pointwise step -- for edge e = (cell c, slot k) with child x (its single
// consumer is e): dh(x) = dA[e], dc(x) = dCe[e] (written by c's own pointwise step), then
// dz(x) -> dZ row of x and dCe of x's two edges. The dA rows never reach memory except for
// leaf children (the embedding gradient reads them). Dependencies are per 256-row tile, not
// per level: every tile has a counter (keyed by its first cell) that the epilogues of its
// rows' consumers raise by the number of columns of each row they complete; the tile's TMA
// producer waits for rows x S, so a tile starts as soon as ITS rows are ready, and the
// depth order of PAPER.md L49 holds without level-wide drains. Roots' dZ come from a seeded
// pointwise pass launched before (their counts are pre-set by k_bwd_prelude).
// Epilogue layout: each warp owns 32 accumulator rows; per 64-column slab it moves the
// fp32 values TMEM -> registers -> a padded smem transpose, then walks the rows with the
// 32 lanes across columns, so every global access of the pointwise step is a coalesced
// row segment.
struct BwdLevels {
  const int32_t *lo;
  int D, S, nl, ld_u;
  int narrow_below;  // a level with fewer 256-column pair tiles than this uses 128 columns
  int pf;            // L2 prefetch distance of the dZ (A operand) boxes in k-blocks (0: off)
  int ksplit_max;    // split-K units allowed per level (0: no split; else the number of CTA pairs)
  int KB;            // k-blocks of the full K = GATES*S reduction
  int ks256;         // split-K also for 256-column tiles
  // per-level tile tables (k_bwd_tiles): per level D..2 its critical units, then some of its
  // deferred (leaf-children-only) column tiles inline; after all levels the rest of the
  // deferred tiles of levels D..2. x = first unit, y = units, z = N / 128 | KS << 2 | v << 4
  // (critical entries: v = the level's first split-unit ordinal; deferred entries: their first
  // level-local tile), w = first column tile | column tiles << 16
  const int4 *tcrit, *tinl, *tend;
  const int *total;  // units in all sections
};
// Per-level tiling (k_bwd_tiles): N (128 or 256 columns) and KS (1, or 2 = split-K in two
// k-halves). A latency-bound level whose critical tiles fit one wave of CTA pairs twice over
// runs each tile as two k-half units on two pairs: each pair accumulates half of the
// K = GATES*S reduction, hands the partial of the OTHER half's columns to its partner through
// L2 (ring slots) and finishes its own half of the columns, so a level's mainloop and
// epilogue both halve.
struct BwdCursor {  // per level D..2: critical units, inline deferred tiles; then the end section
  int d, t0, nt, r0, r1, N, NTn, KS, ctlo, lt_off, sbase, sec;
  __device__ void load(const BwdLevels &L) {
    r0 = __ldg(L.lo + d); r1 = __ldg(L.lo + d + 1);
    const int4 c = sec == 0 ? L.tcrit[d] : sec == 1 ? L.tinl[d] : L.tend[d];
    t0 = c.x; nt = c.y; N = (c.z & 3) * 128; KS = (c.z >> 2) & 3;
    lt_off = sec == 0 ? 0 : c.z >> 4;  // critical entries carry the split ordinal base instead
    sbase = sec == 0 ? c.z >> 4 : 0;
    ctlo = c.w & 0xffff; NTn = c.w >> 16;
  }
  __device__ void init(const BwdLevels &L) { d = L.D; sec = 0; load(L); }
  __device__ void seek(const BwdLevels &L, int T) {
    while (T >= t0 + nt) {
      if (sec == 0) sec = 1;
      else if (sec == 1) {
        if (--d < 2) { sec = 2; d = L.D; }
        else sec = 0;
      } else if (--d < 2) return;  // past the last unit (callers stay below *L.total)
      load(L);
    }
  }
  // level-local unit lt = ((row tile) * NTn + column tile - ctlo) * KS + k-half
  __device__ int row_tile(int lt) const { return (lt + lt_off) / (NTn * KS); }
  __device__ int col_tile(int lt) const { return ctlo + ((lt + lt_off) / KS) % NTn; }
  __device__ int khalf(int lt) const { return (lt + lt_off) % KS; }
  __device__ int first_cell(const BwdLevels &L, int lt) const { return (r0 - L.nl) + row_tile(lt) * PM; }
  // k-block range of tile lt: the whole K, or one half of it
  __device__ void krange(const BwdLevels &L, int lt, int &k0, int &k1) const {
    const int h = L.KB / 2;
    if (KS == 1) { k0 = 0; k1 = L.KB; }
    else if (khalf(lt) == 0) { k0 = 0; k1 = h; }
    else { k0 = h; k1 = L.KB; }
  }
};

// k-blocks per stage of a backward tile (see fwd_kps): dZ box of bx0 rows + N/2 U columns
__host__ __device__ inline int bwd_kps(int N, int bx0) {
  const int k = DA_STAGE / (bx0 * 128 + (N / 128) * MN_CHUNK);
  return k < 1 ? 1 : k > 8 ? 8 : k;
}

// epilogue load flavours: the read-once operands of the pointwise step (the child's gates
// and c, its children's c, dCe) stream with evict-first loads (ld.global.cs) so they do not
// displace the dZ rows and U the MMAs read from L2 (FOLD_BWD_LDG build switch: plain loads)
#ifndef FOLD_BWD_LDG
#define BWD_LDG(p) __ldcs(p)
#define BWD_LDC(p) __ldcs(p)
#else
#define BWD_LDG(p) __ldg(p)
#define BWD_LDC(p) __ldcg(p)
#endif
#ifndef FOLD_BW_ST
#define FOLD_BW_ST 4
#endif
// rows per epilogue load group (FOLD_BWD_R build switch) and the one-wave-level L2 prefetch
// of the pointwise operands (FOLD_BWD_PF1=0 disables it)
#ifndef FOLD_BWD_R
#define FOLD_BWD_R 4
#endif
#ifndef FOLD_BWD_PF1
#define FOLD_BWD_PF1 0
#endif
// U (the B operand every tile of every level re-reads): TMA loads with an L2 evict_last
// policy (FOLD_BWD_U_NOHINT build switch: none). With the evict-first epilogue loads:
// C4 dA 11.7 -> 11.55 ms, C3 0.577 -> 0.563 ms
#ifndef FOLD_BWD_U_NOHINT
#define BWD_TMA_U(m, bar, dst, x, y) ptx::tma_load_2d_pair_hint(m, bar, dst, x, y, pol_u)
#else
#define BWD_TMA_U(m, bar, dst, x, y) ptx::tma_load_2d_pair(m, bar, dst, x, y)
#endif
constexpr int BW_ST = FOLD_BW_ST;
constexpr int BW_EPI = 8;                       // epilogue warps
constexpr int BW_THREADS = 128 + 32 * BW_EPI;
// floats per warp transpose buffer: 32 rows x 64 columns, unpadded; float2 granules XOR-
// swizzled by the row (column c of row r at r * 64 + (c ^ 2r)): the row-wise float2 writes and
// the column-wise float2 reads are both conflict-free per half-warp, and the 2 KB the padding
// took leaves room for a fifth pipeline stage
constexpr int BW_XS = 32 * 64;
// split-K hand-over ring: kKsRing slots of [2 CTAs][128 rows][128 columns] fp32 partial sums;
// split unit o (its ordinal among the split units, k_bwd_tiles) uses slot o % kKsRing (use
// o / kKsRing), with a written count and a read
// count per slot (k_bwd_levels waits for the previous use's read before reusing a slot)
constexpr int BW_SMEM = BW_ST * DA_STAGE + BW_EPI * BW_XS * 4 + 1024;

template <int GATES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(BW_THREADS, 1)
    k_bwd_levels(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmZ16,
                 const __grid_constant__ CUtensorMap tmZ64, const __grid_constant__ CUtensorMap tmU, BwdLevels L,
                 int KB, int total_tiles, const int32_t *__restrict__ gather,
                 const __nv_bfloat16 *__restrict__ Gact, int ld_g, const float *__restrict__ C, int ld, float *dA,
                 float *dCe, __nv_bfloat16 *dZ, int ld_z, int *rt_cnt, const int32_t *__restrict__ tstart,
                 int slabs, int dbg, float *ks_ring, int *ks_wr, int *ks_cons) {
  constexpr int ST = BW_ST;
  total_tiles = min(total_tiles, __ldg(L.total));  // the host passes an upper bound
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  float *xs_all = reinterpret_cast<float *>(smem + ST * DA_STAGE);
  __shared__ __align__(8) uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int S = L.S, nl = L.nl;
  const int Sp = (int)round_up(S, BK);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], 2 * BW_EPI); }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmZ);
    ptx::prefetch_tmap(&tmZ16);
    ptx::prefetch_tmap(&tmZ64);
    ptx::prefetch_tmap(&tmU);
  }
  if (warp == 2) { ptx::tmem_alloc2(&tmem_base_sh, 512); ptx::tmem_relinquish2(); }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  if (warp == 0) {
    if (lane == 0) {
      BwdCursor cur;
      cur.init(L);
      int it = 0;
#ifndef FOLD_BWD_U_NOHINT
      const uint64_t pol_u = ptx::createpolicy_evict_last();
#endif
      // A-operand box rows for a CTA holding m rows (narrow tiles load only their rows)
      auto box_of = [](int m) { return m <= 0 ? 0 : m <= 16 ? 16 : m <= 64 ? 64 : BM; };
      // this CTA's dZ box (map, first row) of tile T (bx = 0: the CTA holds no rows)
      auto zbox = [&](const BwdCursor &c, int T, const CUtensorMap *&m, int &row) {
        const int ctt = c.first_cell(L, T - c.t0);
        const int rw = min(PM, c.r1 - nl - ctt);
        const int b = rank ? box_of(rw - BM) : box_of(min(rw, BM));
        m = b == 16 ? &tmZ16 : b == 64 ? &tmZ64 : &tmZ;
        row = ctt + (int)rank * BM;
        return b;
      };
      const int pf = L.pf;
      for (int T = pair; T < total_tiles; T += npairs) {
        cur.seek(L, T);
        const int lt = T - cur.t0, N = cur.N;
        const int ct = cur.first_cell(L, lt);  // first cell of the pair tile
        const int rows = min(PM, cur.r1 - nl - ct);
        int k0, k1;  // this unit's k-blocks (all, or one k-half)
        cur.krange(L, lt, k0, k1);
        const int nkb = k1 - k0;
        // narrow tiles load only the dZ rows they hold (see k_fwd_levels)
        const int bx0 = box_of(min(rows, BM)), bx1 = box_of(rows - BM), bx = rank ? bx1 : bx0;
        const CUtensorMap *mZ = bx == 16 ? &tmZ16 : bx == 64 ? &tmZ64 : &tmZ;
        const int mt = ct + (int)rank * BM;
        // L2 prefetch: the dZ rows of a level were written one level earlier and mostly left
        // L2 since; every column tile of the row tile requests the same k-block at about the
        // same time, so without a prefetch each k-block costs a DRAM round trip that the
        // 4-stage ring does not cover. Boxes pf k-blocks ahead are prefetched into L2, and
        // the last pf k-blocks of a tile prefetch the head of this pair's next tile.
        const CUtensorMap *mZn = nullptr;
        int mtn = 0, bxn = 0;
        int kn0 = 0;
        if (pf > 0 && T + npairs < total_tiles) {
          BwdCursor nx = cur;
          nx.seek(L, T + npairs);
          bxn = zbox(nx, T + npairs, mZn, mtn);
          int kn1;
          nx.krange(L, T + npairs - nx.t0, kn0, kn1);
        }
        const int nb = cur.col_tile(lt) * N + (int)rank * (N / 2);
        const uint32_t bytes = (uint32_t)(bx0 + bx1) * 128 + N * 128;
        // the first stages' U boxes are issued before the dependency wait; narrow tiles pack
        // kps k-blocks per stage
        const int kps = bwd_kps(N, bx0), abox = bx0 * 128, ubox = (N / 128) * MN_CHUNK;
        const int nst = (nkb + kps - 1) / kps;
        if (rank == 0) btrace(dbg, 0, T);
#ifndef FOLD_BWD_EARLY_U
        // wait for the tile's inputs before issuing any of its boxes: issuing the first stages'
        // U boxes before the wait (FOLD_BWD_EARLY_U, the round-1 design) left the tile's whole
        // mainloop ~25% slower on latency-bound levels (C4 B=1024: 27.1 -> 21.6 us per tile,
        // per-tile stamps; dA 13.0 -> 11.7 ms)
        ptx::wait_counter(rt_cnt + ct, rows * slabs);
#endif
        const bool ready = ptx::ld_acquire_gpu(rt_cnt + ct) >= rows * slabs;
        if (ready) ptx::fence_proxy_async_global();
        if (ready && rank == 0) btrace(dbg, 1, T);
        const int pre = ready ? 0 : (nst < ST ? nst : ST);
        if (ready && kps == 1) {  // inputs published: one (A, U) box set per stage
          for (int kb = k0; kb < k1; kb++, it++) {
            if (pf > 0) {
              if (kb + pf < k1) {
                if (bx) ptx::tma_prefetch_2d(mZ, (kb + pf) * BK, mt);
              } else if (bxn && kb + pf - k1 < KB) {
                ptx::tma_prefetch_2d(mZn, (kn0 + kb + pf - k1) * BK, mtn);
              }
            }
            const int s = it % ST;
            const uint32_t ph = (it / ST) & 1;
            ptx::mbar_wait(&empty[s], ph ^ 1);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], bytes);
            uint8_t *A = smem + s * DA_STAGE;
            if (bx) ptx::tma_load_2d_pair(mZ, &full[s], A, kb * BK, mt);
            for (int ch = 0; ch < N / 128; ch++)
              BWD_TMA_U(&tmU, &full[s], A + DA_A_BYTES + ch * MN_CHUNK, nb + ch * 64, kb * BK);
          }
          continue;
        }
        const int uoff = kps == 1 ? DA_A_BYTES : kps * abox;
        for (int q = 0; q < nst; q++) {
          const int s = (it + q) % ST;
          const uint32_t ph = ((it + q) / ST) & 1;
          const int kb0 = k0 + q * kps, nk = min(kps, k1 - kb0);
          uint8_t *stg = smem + s * DA_STAGE;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)nk * bytes);
          for (int j = 0; j < nk; j++)
            for (int ch = 0; ch < N / 128; ch++)
              BWD_TMA_U(&tmU, &full[s], stg + uoff + j * ubox + ch * MN_CHUNK, nb + ch * 64, (kb0 + j) * BK);
          if (q < pre - 1) continue;
          if (q == pre - 1) {
            // this pair tile's dZ rows (and their dCe) complete
            ptx::wait_counter(rt_cnt + ct, rows * slabs);
            ptx::fence_proxy_async_global();
            if (rank == 0) btrace(dbg, 1, T);
            if (bx)
              for (int q2 = 0; q2 < pre; q2++) {
                const int s2 = (it + q2) % ST;
                for (int j = 0; j < kps && q2 * kps + j < nkb; j++)
                  ptx::tma_load_2d_pair(mZ, &full[s2], smem + s2 * DA_STAGE + j * abox, (k0 + q2 * kps + j) * BK,
                                        mt);
              }
            continue;
          }
          if (bx)
            for (int j = 0; j < nk; j++) ptx::tma_load_2d_pair(mZ, &full[s], stg + j * abox, (kb0 + j) * BK, mt);
        }
        it += nst;
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // converged warp, elected lane issues (ptx::elect_one)
      BwdCursor cur;
      cur.init(L);
      int it = 0, tc = 0;
      for (int T = pair; T < total_tiles; T += npairs, tc++) {
        cur.seek(L, T);
        const uint32_t idesc = ptx::idesc_bf16(PM, cur.N, 0, 1);
        const int acc = tc & 1;
        ptx::mbar_wait(&tempty[acc], ((tc >> 1) & 1) ^ 1);
        __syncwarp();
        ptx::tc_fence_after();
        if (lane == 0) btrace(dbg, 2, T);
        const uint32_t dst = tbase + acc * 256;
        const int ct = cur.first_cell(L, T - cur.t0);
        const int rows0 = min(BM, cur.r1 - nl - ct);
        const int bx0 = rows0 <= 16 ? 16 : rows0 <= 64 ? 64 : BM;
        const int kps = bwd_kps(cur.N, bx0), abox = bx0 * 128, ubox = (cur.N / 128) * MN_CHUNK;
        int k0, k1;
        cur.krange(L, T - cur.t0, k0, k1);
        const int nst = (k1 - k0 + kps - 1) / kps;
        if (kps == 1) {  // one k-block per stage, U at the fixed offset DA_A_BYTES
          for (int kb = k0; kb < k1; kb++, it++) {
            int s = it % ST;
            uint32_t ph = (it / ST) & 1;
            ptx::mbar_wait(&full[s], ph);
            __syncwarp();
            ptx::tc_fence_after();
            if (kb == k0 && lane == 0) btrace(dbg, 8, T);
            const uint32_t a0 = ptx::smem_u32(smem + s * DA_STAGE), b0 = a0 + DA_A_BYTES;
            const uint64_t da = ptx::sdesc_sw128(a0, 16, 1024), db = ptx::sdesc_sw128(b0, MN_CHUNK, 1024);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / 16; k++)
                ptx::umma_bf16_2cta(dst, ptx::desc_add(da, 32 * k), ptx::desc_add(db, 2048 * k), idesc,
                                    (kb != k0 || k != 0));
              ptx::umma_commit_2cta(&empty[s]);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) {
            ptx::umma_commit_2cta(&tfull[acc]);
            btrace(dbg, 3, T);
          }
          __syncwarp();
          continue;
        }
        for (int q = 0; q < nst; q++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&full[s], ph);
          __syncwarp();
          ptx::tc_fence_after();
          if (q == 0 && lane == 0) btrace(dbg, 8, T);
          const uint32_t st0 = ptx::smem_u32(smem + s * DA_STAGE);
          const int nk = min(kps, k1 - k0 - q * kps);
          for (int j = 0; j < nk; j++) {
            const uint64_t da = ptx::sdesc_sw128(st0 + j * abox, 16, 1024);
            const uint64_t db = ptx::sdesc_sw128(st0 + kps * abox + j * ubox, MN_CHUNK, 1024);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / 16; k++)
                ptx::umma_bf16_2cta(dst, ptx::desc_add(da, 32 * k), ptx::desc_add(db, 2048 * k), idesc,
                                    (q | j | k) != 0);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::umma_commit_2cta(&empty[s]);
          __syncwarp();
        }
        if (ptx::elect_one()) {
          ptx::umma_commit_2cta(&tfull[acc]);
          btrace(dbg, 3, T);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3, grp = (warp - 4) >> 2;
    float *xs = xs_all + (warp - 4) * BW_XS;
    BwdCursor cur;
    cur.init(L);
    int tc = 0;
    // TMEM (thread = row) -> this warp's smem transpose buffer: 32 rows x the 64 columns of
    // accumulator slab `slab` (row r's column c at r * 64 + (c ^ 2r), float2 granules)
    auto slab_to_xs = [&](uint32_t tl, int slab) {
      float v[64];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        float t8[8];
        ptx::tmem_ld8(tl + slab * 64 + k * 8, t8);
#pragma unroll
        for (int u = 0; u < 8; u++) v[k * 8 + u] = t8[u];
      }
      ptx::tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 64; k += 2)
        *reinterpret_cast<float2 *>(xs + lane * 64 + (k ^ (2 * lane))) = make_float2(v[k], v[k + 1]);
      __syncwarp();
    };
    for (int T = pair; T < total_tiles; T += npairs, tc++) {
      cur.seek(L, T);
      const int N = cur.N, KS = cur.KS;
      const int acc = tc & 1;
      const int lt = T - cur.t0;
      const int ct = cur.first_cell(L, lt);
      {  // order this warp's dCe reads after the tile's publication (already complete)
        if (lane == 0) ptx::wait_counter(rt_cnt + ct, min(PM, cur.r1 - nl - ct) * slabs);
        __syncwarp();
      }
      const int c_row0 = ct + (int)rank * BM + q * 32;  // cell of row 0
      const int c_end = cur.r1 - nl;
      const int n0 = cur.col_tile(lt) * N;
      // this unit's own 64-column slabs (all N / 64, or its k-half's half of them) and, on a
      // split-K level, the partner's slabs whose partial sums it hands over
      const int nsl = N / 64, kh = cur.khalf(lt);
      const int own_n = KS == 1 ? nsl : nsl / 2, own_lo = KS == 1 ? 0 : kh * own_n;
      const int oth_n = KS == 1 ? 0 : nsl / 2, oth_lo = (1 - kh) * oth_n;
      // a unit owning one slab: the two warps of a lane quarter split its 32 rows
      const bool rsplit = own_n == 1;
      const int i_lo = rsplit ? 16 * grp : 0, i_hi = rsplit ? i_lo + 16 : 32;
      const int w0 = rsplit ? 0 : grp, wstep = rsplit ? 1 : 2;
      // per-row metadata for this warp's 32 rows: lane i <-> row i
      const int my_c = c_row0 + lane;
      const bool my_valid = my_c < c_end;
      const bool my_rows = lane >= i_lo && lane < i_hi;  // rows this warp finishes
      int my_x[2] = {-1, -1}, my_xl[2] = {-1, -1}, my_xr[2] = {-1, -1}, my_ts[2] = {-1, -1};
      if (my_valid) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          my_x[h] = __ldg(gather + 2 * (int64_t)(my_c + nl) + h);
          if (my_x[h] >= nl) {
            my_xl[h] = __ldg(gather + 2 * (int64_t)my_x[h]);
            my_xr[h] = __ldg(gather + 2 * (int64_t)my_x[h] + 1);
            my_ts[h] = __ldg(tstart + (my_x[h] - nl));
          }
        }
      }
      // warm L2 with this warp's pointwise operands (the child's gates and c, its children's
      // c, dCe) while the tile's MMAs run: on latency-bound levels (chains) the epilogue's
      // HBM round trips are otherwise on every level's critical path (only on levels that
      // fit one wave of tiles: on wide levels the epilogue overlaps the next tile anyway)
      if (FOLD_BWD_PF1 && my_valid && my_rows && cur.nt <= npairs) {
#pragma unroll 1
        for (int w = w0; w < own_n; w += wstep) {
          const int np = n0 + (own_lo + w) * 64;
          const int half = np >= Sp;
          const int col = np - half * Sp;
          const int x = my_x[half];
          if (col >= S || x < nl) continue;
          const int last = min(64, S - col) - 1;
          const __nv_bfloat16 *gx = Gact + (int64_t)(x - nl) * ld_g + col;
#pragma unroll
          for (int g = 0; g < GATES; g++) { ptx::prefetch_l2(gx + g * ld); ptx::prefetch_l2(gx + g * ld + last); }
          if constexpr (GATES == 5) {
            const int rows[3] = {x, my_xl[half], my_xr[half]};
#pragma unroll
            for (int k = 0; k < 3; k++) {
              if (rows[k] < nl) continue;
              const float *cx = C + (int64_t)rows[k] * ld + col;
              ptx::prefetch_l2(cx); ptx::prefetch_l2(cx + last / 2); ptx::prefetch_l2(cx + last);
            }
            const float *dx = dCe + (2 * (int64_t)my_c + half) * S + col;
            ptx::prefetch_l2(dx); ptx::prefetch_l2(dx + last / 2); ptx::prefetch_l2(dx + last);
          }
        }
      }
      int slab_cnt[2] = {0, 0};  // columns this warp completes (its 64-column slabs), per half
      ptx::mbar_wait(&tfull[acc], (tc >> 1) & 1);
      ptx::tc_fence_after();
      if (warp == 4 && lane == 0 && rank == 0) btrace(dbg, 4, T);
      const uint32_t tl = tbase + acc * 256 + ((uint32_t)(q * 32) << 16);
#ifdef FOLD_DBG_TMEM  // diagnostic: stamp 9 = one probe TMEM load (8 columns) complete
      {
        float t8[8];
        ptx::tmem_ld8(tl, t8);
        ptx::tmem_ld_wait();
        if (warp == 4 && lane == 0 && rank == 0) btrace(dbg, 9, T + (t8[0] == 12345.f));
      }
#endif
      // split-K, phase A: the partner's slabs' partial sums -> this unit's ring slot (fp32,
      // [CTA rank][128 rows][128 columns], rows through the transpose buffer so each store
      // is a coalesced row segment); every epilogue warp of the pair then raises the slot's
      // written count (release), 2 * BW_EPI per use
      const float *pp = nullptr;
      int pslot = 0;
      if (KS == 2) {
        const int ord = cur.sbase + lt;  // this unit's ordinal among all split units
        const int slot = ord % kKsRing, use = ord / kKsRing;
        float *dst = ks_ring + (size_t)slot * kKsSlotFloats + (size_t)rank * BM * 128 + (size_t)q * 32 * 128;
        if (use > 0) {  // the slot's previous unit (tile T - kKsRing) has been read by its partner
          if (lane == 0) ptx::wait_counter(ks_cons + slot, use * 2 * BW_EPI);
          __syncwarp();
        }
#pragma unroll 1
        for (int o = (grp + 1) & 1; o < oth_n; o += 2) {
          slab_to_xs(tl, oth_lo + o);
#pragma unroll 4
          for (int i = 0; i < 32; i++)
            *reinterpret_cast<float2 *>(dst + i * 128 + o * 64 + 2 * lane) =
                *reinterpret_cast<const float2 *>(xs + i * 64 + ((2 * lane) ^ (2 * i)));
          __syncwarp();
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(ks_wr + slot, 1);
        // the partner unit's partial sums of this unit's slabs
        const int Tp = kh == 0 ? ord + 1 : ord - 1;  // the partner's ordinal
        pslot = Tp % kKsRing;
        if (lane == 0) ptx::wait_counter(ks_wr + pslot, (Tp / kKsRing + 1) * 2 * BW_EPI);
        __syncwarp();
        pp = ks_ring + (size_t)pslot * kKsSlotFloats + (size_t)rank * BM * 128 + (size_t)q * 32 * 128;
      }
#pragma unroll 1
      for (int w = w0; w < own_n; w += wstep) {
        const int slab = own_lo + w;
        slab_to_xs(tl, slab);
        if (warp == 4 && lane == 0 && rank == 0 && w == w0) btrace(dbg, 6, T);
        const int np = n0 + slab * 64;  // padded column of the slab (the slab lies in one half)
        const int half = np >= Sp;
        const int col = np - half * Sp + 2 * lane;  // this lane's 2 state columns
        const bool colok = col < S;                  // S even (checked by the host)
        if (np - half * Sp < S) slab_cnt[half] += min(64, S - (np - half * Sp));
        // rows in groups of R: all loads of the group first (memory-level parallelism),
        // then the math and the stores
        constexpr int R = FOLD_BWD_R;
#pragma unroll 1
        for (int i0 = i_lo; i0 < i_hi && c_row0 + i0 < c_end; i0 += R) {
          int xs_[R], xls[R], xrs[R];
          bool ok[R];
          float2 dh[R], cc[R], cl[R], cr[R], dc[R], pv[R];
          uint32_t graw[R][GATES];
#pragma unroll
          for (int j = 0; j < R; j++) {
            const int i = i0 + j;
            xs_[j] = __shfl_sync(0xffffffffu, half ? my_x[1] : my_x[0], i);
            xls[j] = __shfl_sync(0xffffffffu, half ? my_xl[1] : my_xl[0], i);
            xrs[j] = __shfl_sync(0xffffffffu, half ? my_xr[1] : my_xr[0], i);
            ok[j] = colok && i < i_hi && c_row0 + i < c_end;
            dh[j] = *reinterpret_cast<const float2 *>(xs + (i & 31) * 64 + ((2 * lane) ^ (2 * (i & 31))));
            // split-K: the partner's partial sum, added below (fixed order: own + partner); the
            // add waits for the load, so it stays out of this loop of loads
            pv[j] = pp && ok[j] ? __ldcg(reinterpret_cast<const float2 *>(pp + i * 128 + w * 64 + 2 * lane))
                                : make_float2(0.f, 0.f);
            const int64_t e = 2 * (int64_t)(c_row0 + i) + half;
            if (ok[j] && xs_[j] >= nl) {
              const int64_t xc = xs_[j] - nl;
              const __nv_bfloat16 *gx = Gact + xc * ld_g + col;
#pragma unroll
              for (int g = 0; g < GATES; g++) graw[j][g] = BWD_LDG(reinterpret_cast<const uint32_t *>(gx + g * ld));
              if constexpr (GATES == 5) {
#ifdef FOLD_DIAG_NOC  // diagnostic only (results invalid): the c operands are not loaded
                cc[j] = make_float2(0.5f, 0.5f); cl[j] = cc[j]; cr[j] = cc[j];
                dc[j] = BWD_LDC(reinterpret_cast<const float2 *>(dCe + e * S + col));
              }
              if constexpr (false) {
#endif
                cc[j] = BWD_LDC(reinterpret_cast<const float2 *>(C + (int64_t)xs_[j] * ld + col));
                cl[j] = xls[j] >= nl ? BWD_LDC(reinterpret_cast<const float2 *>(C + (int64_t)xls[j] * ld + col))
                                     : make_float2(0.f, 0.f);
                cr[j] = xrs[j] >= nl ? BWD_LDC(reinterpret_cast<const float2 *>(C + (int64_t)xrs[j] * ld + col))
                                     : make_float2(0.f, 0.f);
                dc[j] = BWD_LDC(reinterpret_cast<const float2 *>(dCe + e * S + col));
              }
            }
          }
#pragma unroll
          for (int j = 0; j < R; j++) {
            if (!ok[j]) continue;
            const int64_t e = 2 * (int64_t)(c_row0 + i0 + j) + half;
            if (pp) {
              dh[j].x += pv[j].x;
              dh[j].y += pv[j].y;
            }
            if (xs_[j] < nl) {  // leaf child: the embedding gradient reads dA (bf16 on this path)
              *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<__nv_bfloat16 *>(dA) + e * S + col) =
                  __floats2bfloat162_rn(dh[j].x, dh[j].y);
              continue;
            }
            const int64_t xc = xs_[j] - nl;
            __nv_bfloat16 *dz = dZ + xc * ld_z + col;
            float2 gg[GATES];
#pragma unroll
            for (int g = 0; g < GATES; g++) gg[g] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&graw[j][g]));
            if constexpr (GATES == 1) {
              const float2 h = gg[0];
              *reinterpret_cast<__nv_bfloat162 *>(dz) =
                  __floats2bfloat162_rn(dh[j].x * (1.f - h.x * h.x), dh[j].y * (1.f - h.y * h.y));
            } else {
              float zz[5][2], el[2], er[2];
              const float dhv[2] = {dh[j].x, dh[j].y}, dcv[2] = {dc[j].x, dc[j].y}, ccv[2] = {cc[j].x, cc[j].y};
              const float clv[2] = {cl[j].x, cl[j].y}, crv[2] = {cr[j].x, cr[j].y};
#pragma unroll
              for (int u = 0; u < 2; u++) {
                const float ig = u ? gg[0].y : gg[0].x, fl = u ? gg[1].y : gg[1].x;
                const float fr = u ? gg[2].y : gg[2].x, og = u ? gg[3].y : gg[3].x;
                const float ug = u ? gg[4].y : gg[4].x;
                const float tcv = tanh_fast(ccv[u]);
                const float dO = dhv[u] * tcv;
                const float dcc = dcv[u] + dhv[u] * og * (1.f - tcv * tcv);
                zz[0][u] = dcc * ug * ig * (1.f - ig);
                zz[1][u] = dcc * clv[u] * fl * (1.f - fl);
                zz[2][u] = dcc * crv[u] * fr * (1.f - fr);
                zz[3][u] = dO * og * (1.f - og);
                zz[4][u] = dcc * ig * (1.f - ug * ug);
                el[u] = dcc * fl;
                er[u] = dcc * fr;
              }
#pragma unroll
              for (int g = 0; g < 5; g++)
                *reinterpret_cast<__nv_bfloat162 *>(dz + g * S) = __floats2bfloat162_rn(zz[g][0], zz[g][1]);
              // dc into a leaf is dropped (its c is the constant 0): only cell grandchildren
              if (xls[j] >= nl) *reinterpret_cast<float2 *>(dCe + (2 * xc) * S + col) = make_float2(el[0], el[1]);
              if (xrs[j] >= nl) *reinterpret_cast<float2 *>(dCe + (2 * xc + 1) * S + col) = make_float2(er[0], er[1]);
            }
          }
#ifndef FOLD_DBG_TMEM
          if (warp == 4 && lane == 0 && rank == 0 && w == w0 && i0 == i_lo) btrace(dbg, 9, T);
#endif
        }
        __syncwarp();
        if (warp == 4 && lane == 0 && rank == 0 && w == w0) btrace(dbg, 7, T);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_leader(&tempty[acc]);
      // publish: every lane fences its own dZ / dCe stores, then lane i credits the tiles of
      // row i's children with the columns this warp completed
      ptx::fence_proxy_async_global();
      __threadfence();
      __syncwarp();
      if (KS == 2 && lane == 0) atomicAdd(ks_cons + pslot, 1);  // the partner's slot is read
#pragma unroll
      for (int h = 0; h < 2; h++)
        if (my_valid && my_rows && my_ts[h] >= 0 && slab_cnt[h] > 0) atomicAdd(rt_cnt + my_ts[h], slab_cnt[h]);
      if (warp == 4 && lane == 0 && rank == 0) btrace(dbg, 5, T);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, 512); }
}

// =================================================================== backward: narrow top levels
// The backward's first levels (the tree tops, chains, single trees) are latency bound like
// the forward's last ones. k_bwd_narrow keeps U stationary and swaps the operands: CTA x
// owns 16 dA columns [16x, 16x + 16) of the padded [h_L | h_R] layout and holds U[:, those
// columns] (all GATES*S rows) in shared memory, read from the transposed bf16 copy Ut
// [2 Sp][GATES*S] (K-major A operand). The K = GATES*S reduction is cut into 8 parts of Kp
// rows stacked in M (M row 16 p + c = column c over part p), and a chunk's R dZ rows are
// stacked the same way in N (N row R p + n = row n's dZ over part p; R = 4 for levels of at
// most 4 rows, else 16), so one M = 128, N = 8R MMA advances all 8 parts:
// dA[n][c] = sum_p D[16 p + c][R p + n], Kp/16 MMAs per chunk (an SS-mode MMA costs about
// its operand bytes, so 16 rows cost ~1.6x 4 rows). The chunk's dZ streams through a ring
// of 3 x 16 KB stages (one K-block of all parts per stage for R = 16, four for R = 4). The
// epilogue sums the parts and runs the child's pointwise step for its 16 columns (the same
// arithmetic as k_bwd_levels' epilogue), then credits the child's row tile with the columns
// done, so the wide kernel (launched after it, on the remaining levels) sees the same
// dependency counters.
constexpr int NB_RMAX = 16;       // rows per chunk (levels of <= 4 rows use 4)
constexpr int NB_PARTS = 8;       // K parts stacked in M (16 columns each) and N (R rows each)
constexpr int NB_THREADS = 256;   // warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4-7 epilogue
constexpr int NB_ST = 3;          // dZ ring stages
constexpr int NB_STAGE = NB_PARTS * NB_RMAX * 128;  // 16 KB

template <int GATES>
__global__ void __launch_bounds__(NB_THREADS, 1)
    k_bwd_narrow(const __grid_constant__ CUtensorMap tmU3, const __grid_constant__ CUtensorMap tmZ4a,
                 const __grid_constant__ CUtensorMap tmZ4b, const __grid_constant__ CUtensorMap tmZ4c,
                 const __grid_constant__ CUtensorMap tmU2,
                 const __grid_constant__ CUtensorMap tmZ2a, const __grid_constant__ CUtensorMap tmZ2b, int packed,
                 const int32_t *__restrict__ lo, int D, int d1, int S, int nl, int Kp,
                 const int32_t *__restrict__ gather, const __nv_bfloat16 *__restrict__ Gact, int ld_g,
                 const float *__restrict__ C, int ld, float *dA, float *dCe, __nv_bfloat16 *dZ, int ld_z, int *rt_cnt,
                 const int32_t *__restrict__ tstart) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  const int NSLOT = Kp / BK;              // K-blocks per part
  constexpr int USLOT = NB_PARTS * 16 * 128;   // bytes per K-block slot of the U slice (128 rows)
  uint8_t *Usm = smem, *Bsm = smem + NSLOT * USLOT;  // U: [slot][part][16 rows]; B: ring of stages
  __shared__ __align__(8) uint64_t u_full, full[NB_ST], empty[NB_ST], acc_full[2], acc_empty[2];
  __shared__ float red[NB_PARTS][16][NB_RMAX + 1];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Sp = (int)round_up(S, BK);
  const int col0 = blockIdx.x * 16, half = col0 >= Sp, j0 = col0 - half * Sp;
  const int ncols = min(16, S - j0);
  if (ncols <= 0) return;  // padding columns only (uniform over the CTA)
  if (tid == 0) {
    ptx::mbar_init(&u_full, 1);
    for (int s2 = 0; s2 < NB_ST; s2++) { ptx::mbar_init(&full[s2], 1); ptx::mbar_init(&empty[s2], 1); }
    for (int a = 0; a < 2; a++) { ptx::mbar_init(&acc_full[a], 1); ptx::mbar_init(&acc_empty[a], 4); }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmU3);
    ptx::prefetch_tmap(&tmZ4a);
    ptx::prefetch_tmap(&tmZ4b);
    ptx::prefetch_tmap(&tmZ4c);
    ptx::prefetch_tmap(&tmU2);
    ptx::prefetch_tmap(&tmZ2a);
    ptx::prefetch_tmap(&tmZ2b);
  }
  if (warp == 2) { ptx::tmem_alloc(&tmem_base_sh, 256); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;

  struct Cur {  // chunks of levels D, D-1, ..., d1; R = rows per chunk of the level
    int d, r, r1, R;
    __device__ bool load(const int32_t *lo, int d1) {
      for (;; d--) {
        if (d < d1) return false;
        r = __ldg(lo + d); r1 = __ldg(lo + d + 1);
        R = r1 - r <= 4 ? 4 : NB_RMAX;
        if (r < r1) return true;
      }
    }
    __device__ bool init(const int32_t *lo, int D, int d1) { d = D; return load(lo, d1); }
    __device__ bool next(const int32_t *lo, int d1) {
      r += R;
      if (r < r1) return true;
      d--;
      return load(lo, d1);
    }
  };
  auto tile_target = [&](const Cur &cu, int &key) {
    const int c = cu.r - nl;
    key = __ldg(tstart + c);
    const int tend = min(key + PM, cu.r1 - nl);
    return (tend - key) * S;
  };

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(&u_full, (uint32_t)(NSLOT * USLOT));
      // packed (GATES*S = 8 Kp): one 3D box per K-block slot; otherwise one 2D box per
      // (part, K-block) whose K columns past GATES*S are zero-filled by the TMA bounds
      for (int q = 0; q < NSLOT; q++) {
        if (packed) {
          ptx::tma_load_3d(&tmU3, &u_full, Usm + q * USLOT, q * BK, col0, 0);
        } else {
          for (int p = 0; p < NB_PARTS; p++)
            ptx::tma_load_2d(&tmU2, &u_full, Usm + q * USLOT + p * 16 * 128, p * Kp + q * BK, col0);
        }
      }
      Cur cu;
      int it = 0;
      for (bool ok = cu.init(lo, D, d1); ok; ok = cu.next(lo, d1)) {
        int key;
        const int target = tile_target(cu, key);
        ptx::wait_counter(rt_cnt + key, target);
        ptx::fence_proxy_async_global();
        const int slot_bytes = NB_PARTS * cu.R * 128, kps = NB_STAGE / slot_bytes;
        const CUtensorMap *m4 = cu.R == 4 ? &tmZ4a : &tmZ4b, *m2 = cu.R == 4 ? &tmZ2a : &tmZ2b;
        if (packed && cu.R == 4 && NSLOT * slot_bytes <= NB_ST * NB_STAGE) {
          // few rows: the whole ring takes all K-blocks in ONE box (one round trip per chunk);
          // every stage is used once so the per-stage phases stay uniform
          for (int k = 0; k < NB_ST; k++) ptx::mbar_wait(&empty[(it + k) % NB_ST], (((it + k) / NB_ST) & 1) ^ 1);
          const int s0 = it % NB_ST;
          ptx::mbar_arrive_expect_tx(&full[s0], (uint32_t)(NSLOT * slot_bytes));
          ptx::tma_load_4d(&tmZ4c, &full[s0], Bsm, 0, cu.r - nl, 0, 0);
          for (int k = 1; k < NB_ST; k++) ptx::mbar_arrive(&full[(it + k) % NB_ST]);
          it += NB_ST;
          continue;
        }
        for (int q0 = 0; q0 < NSLOT; q0 += kps, it++) {
          const int s2 = it % NB_ST;
          ptx::mbar_wait(&empty[s2], ((it / NB_ST) & 1) ^ 1);
          const int nk = min(kps, NSLOT - q0);
          uint8_t *stg = Bsm + s2 * NB_STAGE;
          if (packed) {  // one 4D box = kps K-blocks of all parts (K-blocks past the end zero-filled)
            ptx::mbar_arrive_expect_tx(&full[s2], (uint32_t)(kps * slot_bytes));
            ptx::tma_load_4d(m4, &full[s2], stg, 0, cu.r - nl, 0, q0);
            continue;
          }
          ptx::mbar_arrive_expect_tx(&full[s2], (uint32_t)(nk * slot_bytes));
          for (int j = 0; j < nk; j++) {
            const int q = q0 + j;
            {
              for (int p = 0; p < NB_PARTS; p++)
                ptx::tma_load_2d(m2, &full[s2], stg + j * slot_bytes + p * cu.R * 128, p * Kp + q * BK, cu.r - nl);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // converged warp, elected lane issues (ptx::elect_one)
      ptx::mbar_wait(&u_full, 0);
      Cur cu;
      int i = 0, it = 0;
      const uint64_t du = ptx::sdesc_sw128(ptx::smem_u32(Usm), 16, 1024);
      const uint64_t dbb = ptx::sdesc_sw128(ptx::smem_u32(Bsm), 16, 1024);
      for (bool ok = cu.init(lo, D, d1); ok; ok = cu.next(lo, d1), i++) {
        const int acc = i & 1;
        const uint32_t idesc = ptx::idesc_bf16(128, NB_PARTS * cu.R, 0, 0);
        const int slot_bytes = NB_PARTS * cu.R * 128, kps = NB_STAGE / slot_bytes;
        ptx::mbar_wait(&acc_empty[acc], ((i >> 1) & 1) ^ 1);
        __syncwarp();
        ptx::tc_fence_after();
        const uint32_t dst = tbase + acc * NB_PARTS * NB_RMAX;
        if (packed && cu.R == 4 && NSLOT * slot_bytes <= NB_ST * NB_STAGE) {  // one box in the whole ring
          for (int k = 0; k < NB_ST; k++) ptx::mbar_wait(&full[(it + k) % NB_ST], ((it + k) / NB_ST) & 1);
          __syncwarp();
          ptx::tc_fence_after();
          for (int q = 0; q < NSLOT; q++) {
            const uint64_t dq = ptx::desc_add(du, q * USLOT), bq = ptx::desc_add(dbb, q * slot_bytes);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / 16; k++)
                ptx::umma_bf16(dst, ptx::desc_add(dq, 32 * k), ptx::desc_add(bq, 32 * k), idesc, (q | k) != 0);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) {
            for (int k = 0; k < NB_ST; k++) ptx::umma_commit(&empty[(it + k) % NB_ST]);
            ptx::umma_commit(&acc_full[acc]);
          }
          __syncwarp();
          it += NB_ST;
          continue;
        }
        for (int q0 = 0; q0 < NSLOT; q0 += kps, it++) {
          const int s2 = it % NB_ST;
          ptx::mbar_wait(&full[s2], (it / NB_ST) & 1);
          __syncwarp();
          ptx::tc_fence_after();
          const int nk = min(kps, NSLOT - q0);
          for (int j = 0; j < nk; j++) {
            const int q = q0 + j;
            const uint64_t dq = ptx::desc_add(du, q * USLOT);
            const uint64_t bq = ptx::desc_add(dbb, s2 * NB_STAGE + j * slot_bytes);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / 16; k++)
                ptx::umma_bf16(dst, ptx::desc_add(dq, 32 * k), ptx::desc_add(bq, 32 * k), idesc, (q | k) != 0);
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::umma_commit(&empty[s2]);
          __syncwarp();
        }
        if (ptx::elect_one()) ptx::umma_commit(&acc_full[acc]);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int t = tid - 128;           // 0..127
    const int qw = warp & 3;           // TMEM lane quarter = M rows 32 qw .. 32 qw + 31
    const int c = t & 15, nb = t >> 4; // this thread's column; rows nb and nb + 8 of the chunk
    const int j = j0 + c;
    Cur cu;
    int i = 0;
    for (bool ok = cu.init(lo, D, d1); ok; ok = cu.next(lo, d1), i++) {
      const int acc = i & 1;
      const int R = cu.R;
      const int rows = min(R, cu.r1 - cu.r);
      // operands of the children's pointwise steps (G / C from the forward; dCe of each edge
      // was written by its row's own pointwise step, published with its dZ)
      int64_t x[2] = {-1, -1};
      float gg[2][GATES], cc[2] = {0.f, 0.f}, cl[2] = {0.f, 0.f}, cr[2] = {0.f, 0.f}, dc[2] = {0.f, 0.f};
      bool gcl[2] = {false, false}, gcr[2] = {false, false};  // grandchildren that are cells
      bool waited = false;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int n = nb + 8 * h;
        if (n >= rows || c >= ncols) continue;
        const int64_t r = cu.r + n;
        const int64_t xx = __ldg(gather + 2 * r + half);
        x[h] = xx;
        if (xx >= nl) {
          const int64_t xc = xx - nl;
          const __nv_bfloat16 *gx = Gact + xc * ld_g + j;
#pragma unroll
          for (int g = 0; g < GATES; g++) gg[h][g] = __bfloat162float(gx[g * ld]);
          if constexpr (GATES == 5) {
            const int64_t xl = __ldg(gather + 2 * xx), xr = __ldg(gather + 2 * xx + 1);
            cc[h] = __ldcg(C + xx * ld + j);
            gcl[h] = xl >= nl;
            gcr[h] = xr >= nl;
            if (gcl[h]) cl[h] = __ldcg(C + xl * ld + j);
            if (gcr[h]) cr[h] = __ldcg(C + xr * ld + j);
            if (!waited) {
              int key;
              const int target = tile_target(cu, key);
              ptx::wait_counter(rt_cnt + key, target);
              waited = true;
            }
            dc[h] = __ldcg(dCe + (2 * (r - nl) + half) * S + j);
          }
        }
      }
      ptx::mbar_wait(&acc_full[acc], (i >> 1) & 1);
      ptx::tc_fence_after();
      {  // M row 32 qw + lane = (part p = 2 qw + lane / 16, column lane % 16); its rows are the
         // D columns R p .. R p + R - 1
        const int hi = lane >> 4, p = 2 * qw + hi;
        const uint32_t ta = tbase + acc * NB_PARTS * NB_RMAX + ((uint32_t)(qw * 32) << 16);
        if (R == 4) {
          float z[8];
          ptx::tmem_ld8(ta + qw * 8, z);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 4; k++) red[p][lane & 15][k] = hi ? z[4 + k] : z[k];
        } else {
          float z[32];
#pragma unroll
          for (int b = 0; b < 4; b++) ptx::tmem_ld8(ta + qw * 32 + b * 8, *reinterpret_cast<float(*)[8]>(z + 8 * b));
          ptx::tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; k++) red[p][lane & 15][k] = hi ? z[16 + k] : z[k];
        }
      }
      ptx::tc_fence_before();
      ptx::named_bar_sync(1, 128);
      if (lane == 0) ptx::mbar_arrive(&acc_empty[acc]);
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int n = nb + 8 * h;
        if (n >= rows || c >= ncols) continue;
        float dh = 0.f;
#pragma unroll
        for (int p = 0; p < NB_PARTS; p++) dh += red[p][c][n];
        const int64_t r = cu.r + n;
        const int64_t e = 2 * (r - nl) + half;
        if (x[h] < nl) {  // leaf child: the embedding gradient reads dA (bf16 on this path)
          reinterpret_cast<__nv_bfloat16 *>(dA)[e * S + j] = __float2bfloat16_rn(dh);
          continue;
        }
        const int64_t xc = x[h] - nl;
        __nv_bfloat16 *dz = dZ + xc * ld_z + j;
        if constexpr (GATES == 1) {
          dz[0] = __float2bfloat16_rn(dh * (1.f - gg[h][0] * gg[h][0]));
        } else {
          const float ig = gg[h][0], fl = gg[h][1], fr = gg[h][2], og = gg[h][3], ug = gg[h][4];
          const float tcv = tanh_fast(cc[h]);
          const float dO = dh * tcv;
          const float dcc = dc[h] + dh * og * (1.f - tcv * tcv);
          dz[0] = __float2bfloat16_rn(dcc * ug * ig * (1.f - ig));
          dz[S] = __float2bfloat16_rn(dcc * cl[h] * fl * (1.f - fl));
          dz[2 * S] = __float2bfloat16_rn(dcc * cr[h] * fr * (1.f - fr));
          dz[3 * S] = __float2bfloat16_rn(dO * og * (1.f - og));
          dz[4 * S] = __float2bfloat16_rn(dcc * ig * (1.f - ug * ug));
          if (gcl[h]) dCe[(2 * xc) * S + j] = dcc * fl;  // (dc into a leaf is dropped)
          if (gcr[h]) dCe[(2 * xc + 1) * S + j] = dcc * fr;
        }
      }
      ptx::fence_proxy_async_global();
      ptx::named_bar_sync(1, 128);
      // publish: each cell child of the chunk's rows gets this CTA's columns
      if (t < rows) {
        const int64_t rr = cu.r + t;
        const int64_t xx = __ldg(gather + 2 * rr + half);
        if (xx >= nl) {
          __threadfence();
          atomicAdd(rt_cnt + __ldg(tstart + (xx - nl)), ncols);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 256); }
}

// Row-tile bookkeeping for k_bwd_levels: tstart[c] = first cell of c's 256-row tile (tiles
// start at each level's first row), and the counters of tiles holding roots start at the
// roots' share (their dZ rows come from the seeded pass before the kernel). rt_cnt must be
// zeroed before.
__global__ void k_bwd_prelude(const int32_t *__restrict__ lo, int D, int nl, int n_cells,
                              const int32_t *__restrict__ cons_off, int32_t *__restrict__ tstart, int *rt_cnt,
                              int slabs, const int32_t *__restrict__ gather, int *lvl_flags) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += stride) {
    const int r = (int)c + nl;
    int a = 2, b = D;  // level d with lo[d] <= r < lo[d + 1]
    while (a < b) { const int m = (a + b + 1) >> 1; if (__ldg(lo + m) <= r) a = m; else b = m - 1; }
    const int r0 = __ldg(lo + a);
    const int ts = (r0 - nl) + ((r - r0) / PM) * PM;
    tstart[c] = ts;
    if (__ldg(cons_off + r + 1) == __ldg(cons_off + r)) atomicAdd(rt_cnt + ts, slabs);
    if (lvl_flags) {  // bit k: some cell of level a has a cell (not a leaf) in child slot k
      const int bits = (__ldg(gather + 2 * (int64_t)r) >= nl ? 1 : 0) | (__ldg(gather + 2 * (int64_t)r + 1) >= nl ? 2 : 0);
      if (bits && (__ldcg(lvl_flags + a) & bits) != bits) atomicOr(lvl_flags + a, bits);
    }
  }
}

// Tile tables of k_bwd_levels (one block; levels in parallel, offsets by a block scan):
// per level d = Dw..2 the CRITICAL units -- the
// column tiles that touch a child slot holding a cell somewhere in the level (their epilogue
// produces the next level's dZ) -- then, after all levels, the DEFERRED tiles: column tiles
// that lie entirely in a slot whose children are all leaves in that level (chains: the
// right child of every cell). A deferred tile only writes the leaves' dA for the embedding
// gradient, so it leaves the dependent sweep; the critical tiles of a level that then fits
// one wave of CTA pairs twice over run split-K (KS = 2). defer = 0: every tile critical.
__global__ void __launch_bounds__(1024) k_bwd_tiles(const int32_t *__restrict__ lo, int D, int Dw, int Sp, int ld_u,
                                                    int KB, int npairs, int ksplit_max, int ks256, int defer, int *tab) {
  int4 *crit = reinterpret_cast<int4 *>(tab), *inl = crit + (D + 2), *endt = inl + (D + 2);
  const int *flags = reinterpret_cast<const int *>(endt + (D + 2));
  int *total = const_cast<int *>(flags) + (D + 2);
  __shared__ int sc[1024], sc2[1024];
  __shared__ int carry, carry2;
  const int tid = threadIdx.x, nt = blockDim.x;
  // column tiles [lo_t, lo_t + n) of width N touching (crit = true) / lying outside (false)
  // the child slots set in mask (bit 0: columns [0, Sp), bit 1: [Sp, 2 Sp))
  auto range = [&](int N, int mask, bool want_crit, int &lo_t, int &n) {
    const int NT = (ld_u + N - 1) / N;
    const int lc = (Sp + N - 1) / N, rc0 = Sp / N;  // tiles touching slot 0: [0, lc); slot 1: [rc0, NT)
    int a = 0, b = 0;                               // critical range [a, b)
    if ((mask & 3) == 3) { a = 0; b = NT; }
    else if (mask & 1) { a = 0; b = lc; }
    else if (mask & 2) { a = rc0; b = NT; }
    if (want_crit) { lo_t = a; n = b - a; return; }
    if (b == a) { lo_t = 0; n = NT; }               // nothing critical: all deferred
    else if (a == 0) { lo_t = b; n = NT - b; }      // the tiles after the critical range
    else { lo_t = 0; n = a; }                       // the tiles before it
  };
  const int nlev = Dw - 1;  // levels Dw, Dw - 1, ..., 2 (index i = Dw - d)
  if (tid == 0) { carry = 0; carry2 = 0; }
  __syncthreads();
  for (int sec = 0; sec < 2; sec++) {  // 0: critical + inline deferred per level, 1: the end section
    for (int base = 0; base < nlev; base += nt) {
      const int i = base + tid, d = Dw - i;
      int4 vc = make_int4(0, 0, 0, 0), vi = vc, ve = vc;
      int cnt = 0, c = 0, cs = 0;  // cs: split units (the ring's ordinals)
      if (i < nlev) {
        const int M = __ldg(lo + d + 1) - __ldg(lo + d), rt = (M + PM - 1) / PM;
        const int mask = defer ? flags[d] : 3;
        int l128, n128, l256, n256;
        range(128, mask, true, l128, n128);
        range(256, mask, true, l256, n256);
        int N = 256, KS = 1, lt0 = l256, n = n256;
        if (ksplit_max > 0 && KB >= 8 && n128 > 0 && 2 * rt * n128 <= ksplit_max) { N = 128; KS = 2; lt0 = l128; n = n128; }
        else if (ksplit_max > 0 && KB >= 8 && ks256 && n256 > 0 && 2 * rt * n256 <= ksplit_max) { KS = 2; }
        else if (rt * n256 < npairs) { N = 128; lt0 = l128; n = n128; }
        c = rt * n * KS;
        cs = KS == 2 ? c : 0;
        vc = make_int4(0, c, (N >> 7) | (KS << 2), lt0 | (n << 16));
        // deferred tiles (256 columns): as many as fill the level's last round of CTA pairs
        // run right after its critical units (pairs the level leaves idle), the rest at the end
        int ld0, nd;
        range(256, mask, false, ld0, nd);
        if (mask == 3) nd = 0;
        const int e = rt * nd, fill = (npairs - c % npairs) % npairs, ni = c > 0 ? min(e, fill) : 0;
        vi = make_int4(0, ni, 2 | (1 << 2), ld0 | (nd << 16));
        ve = make_int4(0, e - ni, 2 | (1 << 2) | (ni << 4), ld0 | (nd << 16));
        cnt = sec == 0 ? c + ni : e - ni;
      }
      sc[tid] = cnt;  // inclusive scans over the chunk (Hillis-Steele)
      sc2[tid] = cs;
      __syncthreads();
      for (int o = 1; o < nt; o <<= 1) {
        const int add = tid >= o ? sc[tid - o] : 0, add2 = tid >= o ? sc2[tid - o] : 0;
        __syncthreads();
        sc[tid] += add;
        sc2[tid] += add2;
        __syncthreads();
      }
      if (i < nlev) {
        const int off = carry + sc[tid] - cnt;
        if (sec == 0) {
          vc.x = off;
          vc.z |= (carry2 + sc2[tid] - cs) << 4;
          vi.x = off + c;
          crit[d] = vc;
          inl[d] = vi;
        } else {
          ve.x = off;
          endt[d] = ve;
        }
      }
      __syncthreads();
      if (tid == 0) { carry += sc[nt - 1]; carry2 += sc2[nt - 1]; }
      __syncthreads();
    }
  }
  if (tid == 0) *total = carry;
}

// Forward row-tile bookkeeping: tstart[c] as for the backward; a tile's counter counts the
// h columns pushed into its A rows (2 S per cell when complete), leaf children are credited
// here (the embedding kernel, launched before, pushed them).
__global__ void k_fwd_prelude(const int32_t *__restrict__ lo, int D, int nl, int n_cells, int S,
                              const int32_t *__restrict__ gather, int32_t *__restrict__ tstart, int *rt_cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += stride) {
    const int r = (int)c + nl;
    int a = 2, b = D;
    while (a < b) { const int m = (a + b + 1) >> 1; if (__ldg(lo + m) <= r) a = m; else b = m - 1; }
    const int r0 = __ldg(lo + a);
    const int ts = (r0 - nl) + ((r - r0) / PM) * PM;
    tstart[c] = ts;
    const int leaves = (__ldg(gather + 2 * (int64_t)r) < nl) + (__ldg(gather + 2 * (int64_t)r + 1) < nl);
    if (leaves) atomicAdd(rt_cnt + ts, leaves * S);
  }
}

// =================================================================== dU = dZ^T * Acat (all cells)
// CTA pairs: pair tile = 256 gate rows (i) x 256 state columns (j) of one half (L / R);
// each CTA stages its 128 rows of dZ^T and 128 of the 256 columns of the A plane.
constexpr int DU_N = 256;
constexpr int DU_A_BYTES = BM * 128;         // 2 MN chunks x 64 K-rows x 128 B
constexpr int DU_B_BYTES = (DU_N / 2) * 128; // 2 MN chunks x 64 K-rows x 128 B
constexpr int DU_STAGE = DU_A_BYTES + DU_B_BYTES;
constexpr int DU_DB_BYTES = 128 * 8 * 4;       // db: per-thread partial sums, reduced across k groups
constexpr int DU_SMEM = ST * DU_STAGE + DU_DB_BYTES + 1024;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_dU_tc(const __grid_constant__ CUtensorMap tmZ2, const __grid_constant__ CUtensorMap tmAL,
                 const __grid_constant__ CUtensorMap tmAR, int n_cells, int S, int Mg, int NT, int kb_per_split,
                 float *__restrict__ out_base, int64_t split_stride, int accumulate, float *__restrict__ db_base,
                 int db_accumulate, int pf) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t full[ST], empty[ST], tfull, dbfree[ST];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int px = blockIdx.x >> 1;
  const int half = px / NT, jt = px - half * NT;
  const int i0 = blockIdx.y * PM + (int)rank * BM;   // this CTA's gate rows
  const int jn0 = jt * DU_N;                          // the pair's state columns
  // split-K over cells: this pair reduces k-blocks [kb0, kb1) into its own partial slab
  const int KBall = (int)cdiv(n_cells, BK);
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(KBall, kb0 + kb_per_split);
  const int KB = kb1 > kb0 ? kb1 - kb0 : 0;
  float *dU = out_base + (int64_t)blockIdx.z * split_stride;
  // db = column sums of dZ: the first column tile's pair also sums the
  // dZ^T stage tiles it streams anyway (each CTA's idle epilogue warps, for its own 128
  // gate rows, after the MMA has consumed the stage and before it is refilled)
  const bool is_db = db_base != nullptr && px == 0 && KB > 0;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&dbfree[s], 4);  // the 4 epilogue warps
    }
    ptx::mbar_init(&tfull, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmZ2);
    ptx::prefetch_tmap(&tmAL);
    ptx::prefetch_tmap(&tmAR);
  }
  if (warp == 2) { ptx::tmem_alloc2(&tmem_base_sh, 256); ptx::tmem_relinquish2(); }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  if (warp == 0 && lane == 0) {
    // A' = dZ^T chunk (2 boxes of 64 gate-rows x 64 cells), B' = this CTA's 128 columns of
    // the cells' h_L / h_R rows in the A operand planes written by the forward
    const CUtensorMap *tmB = half ? &tmAR : &tmAL;
    const int jb = jn0 + (int)rank * (DU_N / 2);
    for (int it = 0; it < KB; it++) {
      const int kb = kb0 + it;
      // L2 prefetch pf k-blocks ahead: dZ and the A planes stream from DRAM once, and the
      // pairs sharing a row (column) tile request each k-block at about the same time
      if (pf > 0 && it + pf < KB) {
        const int kp = (kb + pf) * BK;
        ptx::tma_prefetch_2d(&tmZ2, i0, kp);
        ptx::tma_prefetch_2d(&tmZ2, i0 + 64, kp);
        ptx::tma_prefetch_2d(tmB, jb, kp);
        ptx::tma_prefetch_2d(tmB, jb + 64, kp);
      }
      int s = it % ST;
      uint32_t ph = (it / ST) & 1;
      ptx::mbar_wait(&empty[s], ph ^ 1);
      if (is_db) ptx::mbar_wait(&dbfree[s], ph ^ 1);
      if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * DU_STAGE);
      uint8_t *A = smem + s * DU_STAGE;
      uint8_t *B = A + DU_A_BYTES;
      ptx::tma_load_2d_pair(&tmZ2, &full[s], A, i0, kb * BK);
      ptx::tma_load_2d_pair(&tmZ2, &full[s], A + MN_CHUNK, i0 + 64, kb * BK);
      ptx::tma_load_2d_pair(tmB, &full[s], B, jb, kb * BK);
      ptx::tma_load_2d_pair(tmB, &full[s], B + MN_CHUNK, jb + 64, kb * BK);
    }
  } else if (warp == 1) {
    if (rank == 0) {  // converged warp, elected lane issues (ptx::elect_one)
      constexpr uint32_t idesc = ptx::idesc_bf16(PM, DU_N, 1, 1);
      for (int it = 0; it < KB; it++) {
        int s = it % ST;
        uint32_t ph = (it / ST) & 1;
        ptx::mbar_wait(&full[s], ph);
        __syncwarp();
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(smem + s * DU_STAGE), b0 = a0 + DU_A_BYTES;
        const uint64_t da = ptx::sdesc_sw128(a0, MN_CHUNK, 1024), db = ptx::sdesc_sw128(b0, MN_CHUNK, 1024);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; k++)
            ptx::umma_bf16_2cta(tbase, ptx::desc_add(da, 2048 * k), ptx::desc_add(db, 2048 * k), idesc, (it | k) != 0);
          ptx::umma_commit_2cta(&empty[s]);
        }
        __syncwarp();
      }
      if (KB > 0 && ptx::elect_one()) ptx::umma_commit_2cta(&tfull);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    if (is_db) {
      // thread t: 16-byte chunk bc of this CTA's 128 gate rows (box bc / 8, chunk bc % 8 =
      // 8 rows) over cells 8 kg .. 8 kg + 7 of every k-block; a stage is read after the MMA
      // has consumed it (empty) and released on dbfree before the producer refills it
      const int t = tid - 128, bc = t & 15, kg = t >> 4;
      const uint32_t smem_base = ptx::smem_u32(smem);
      float acc[8];
#pragma unroll
      for (int u = 0; u < 8; u++) acc[u] = 0.f;
      for (int it = 0; it < KB; it++) {
        const int s = it % ST;
        ptx::mbar_wait(&empty[s], (it / ST) & 1);
        const uint32_t base = smem_base + (uint32_t)(s * DU_STAGE + (bc >> 3) * MN_CHUNK + kg * 8 * 128);
#pragma unroll
        for (int kk = 0; kk < 8; kk++) {
          const uint4 a = ptx::lds128(base + kk * 128 + ((((uint32_t)bc & 7) ^ (uint32_t)kk) << 4));
          const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&aw[u]));
            acc[2 * u] += f.x;
            acc[2 * u + 1] += f.y;
          }
        }
        // release the stage to the producer's next TMA (async proxy) only after this
        // warp's generic-proxy reads: shared-window loads (LDS, ordered with the arrive in
        // the shared-memory pipe) plus the cross-proxy fence. The first version read the
        // tile through a generic pointer (LD.E), the arrive overtook those loads and under
        // load the refill landed first (GPUTEST_r01: db differed between identical calls
        // in whole 64-row boxes while dZ and dU matched)
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&dbfree[s]);
      }
      // reduce the 8 k groups (fixed order) and write this split's 128 gate rows
      float *red = reinterpret_cast<float *>(smem + ST * DU_STAGE);
#pragma unroll
      for (int u = 0; u < 8; u++) red[t * 8 + u] = acc[u];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      {
        const int r = t, bcx = (r >> 6) * 8 + ((r >> 3) & 7), u = r & 7;
        float v = 0.f;
        for (int g = 0; g < 8; g++) v += red[(g * 16 + bcx) * 8 + u];
        const int row = i0 + r;
        if (row < Mg) {
          float *dst = db_base + (int64_t)blockIdx.z * Mg + row;
          *dst = db_accumulate ? *dst + v : v;
        }
      }
    }
    if (KB > 0) ptx::mbar_wait(&tfull, 0);
    ptx::tc_fence_after();
    const int i = i0 + q * 32 + lane;
    const uint32_t tl = tbase + ((uint32_t)(q * 32) << 16);
    float *out = dU + (int64_t)i * 2 * S + half * S;
#pragma unroll 1
    for (int nc = 0; nc < DU_N / 8; nc++) {
      float v[8];
      ptx::tmem_ld8(tl + nc * 8, v);
      ptx::tmem_ld_wait();
      int j = jn0 + nc * 8;
      if (i >= Mg || j >= S) continue;
      if (KB == 0) {
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = 0.f;
      }
      if (j + 8 <= S && (S & 3) == 0 && !accumulate) {
        *reinterpret_cast<float4 *>(out + j) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(out + j + 4) = make_float4(v[4], v[5], v[6], v[7]);
      } else {
        for (int u = 0; u < 8 && j + u < S; u++) out[j + u] = accumulate ? out[j + u] + v[u] : v[u];
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, 256); }
}

// out[i] = (accumulate ? out[i] : 0) + sum_{s < nsplit} part[s][i]   (fixed order).
// float4 lanes only when every slab start and out are 16-byte aligned (vec != 0: n % 4 == 0
// and aligned bases, checked on the host); otherwise scalar (e.g. db with gates * S odd).
__global__ void k_reduce_splits(int64_t n, int nsplit, const float *__restrict__ part, float *__restrict__ out,
                                int accumulate, int vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (int64_t i4 = t0 * 4; i4 < n; i4 += stride * 4) {
      float4 acc = accumulate ? *reinterpret_cast<const float4 *>(out + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < nsplit; s++) {
        const float4 v = *reinterpret_cast<const float4 *>(part + (int64_t)s * n + i4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      *reinterpret_cast<float4 *>(out + i4) = acc;
    }
  } else {
    for (int64_t i = t0; i < n; i += stride) {
      float acc = accumulate ? out[i] : 0.f;
      for (int s = 0; s < nsplit; s++) acc += part[(int64_t)s * n + i];
      out[i] = acc;
    }
  }
}

}  // namespace

fold_status launch_reduce_splits(int64_t n, int nsplit, const float *part, float *out, int accumulate,
                                 cudaStream_t st) {
  if (n <= 0) return FOLD_OK;
  const int vec = (n % 4 == 0) && ((((uintptr_t)part) | ((uintptr_t)out)) & 15) == 0;
  int64_t blocks = cdiv(vec ? cdiv(n, 4) : n, 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_reduce_splits<<<(unsigned)blocks, 256, 0, st>>>(n, nsplit, part, out, accumulate, vec);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

namespace {

// =================================================================== weight prep
// Ub[r][half*Sp + k] = bf16(U[r][half*S + k]) for k < S, 0 for k in [S, Sp) (Sp =
// round_up(S, 64)): the one bf16 copy of U serves the forward (K-major B operand, each K
// half starting 128 B aligned) and dA (MN-major B operand over the padded 2*Sp columns).
// With il_gates > 0 the output rows are gate-interleaved in blocks of 8 state columns
// (Uil8, the forward's B operand): out row (j/8)*8*G + g*8 + j%8 <- U row g*S + j (zero for
// j >= S).
__global__ void k_prep_U(int64_t rows, int S, int Sp, const float *__restrict__ U, __nv_bfloat16 *__restrict__ Ub,
                         int il_gates) {
  const int cpr = Sp / 4;  // 8-element chunks per row (2*Sp / 8)
  const int64_t total = rows * cpr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = (S & 3) == 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / cpr;
    const int kp = (int)(i - r * cpr) * 8;
    const int half = kp >= Sp, k = kp - half * Sp;
    int K = S;
    int64_t src_row = r;
    if (il_gates) {
      const int64_t blk = r / (8 * il_gates), rem = r - blk * 8 * il_gates;
      const int64_t j = blk * 8 + (rem & 7), g = rem >> 3;
      src_row = g * S + j;
      if (j >= S) K = 0;  // padding rows of the last 8-column block
    }
    const float *src = U + src_row * 2 * S + half * S + k;
    float v[8];
    if (vec && k + 8 <= K) {
      float4 a = __ldg(reinterpret_cast<const float4 *>(src)), b = __ldg(reinterpret_cast<const float4 *>(src + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = k + u < K ? __ldg(src + u) : 0.f;
    }
    *reinterpret_cast<uint4 *>(Ub + r * 2 * Sp + kp) =
        make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
  }
}

}  // namespace

// =================================================================== host helpers
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 2D tensor map: `cols` contiguous elements per row, `rows` rows, `row_bytes` stride.
fold_status make_map_ex(CUtensorMap *m, const void *ptr, CUtensorMapDataType dt, uint64_t cols, uint64_t rows,
                        uint64_t row_bytes, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return FOLD_E_CUDA;
  if (rows < 1) rows = 1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void *>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FOLD_OK : FOLD_E_CUDA;
}
namespace {

// bf16 operand map with 128B swizzle (UMMA operand tiles)
fold_status make_map(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows, uint64_t row_bytes,
                     uint32_t box_cols, uint32_t box_rows) {
  return make_map_ex(m, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cols, rows, row_bytes, box_cols, box_rows,
                     CU_TENSOR_MAP_SWIZZLE_128B);
}

// cudaFuncSetAttribute once per kernel and size (it is a host round trip worth avoiding
// inside the level loop)
template <typename K>
fold_status set_smem(K kernel, int bytes) {
  static thread_local std::unordered_map<const void *, int> set;  // per host thread (and device)
  int dev = 0;
  cudaGetDevice(&dev);
  const void *key = (const char *)(const void *)kernel + dev;
  auto it = set.find(key);
  if (it != set.end() && it->second >= bytes) return FOLD_OK;
  FOLD_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  set[key] = bytes;
  return FOLD_OK;
}

int num_sms() {
  static int n[kMaxDevices] = {};
  const int dev = cur_dev();
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

// SMs the persistent level kernels leave free for concurrent work (fold_set_reserved_sms)
std::atomic<int> g_reserved_sms{0};
int reserve_pairs(int npairs) {
  const int r = npairs - (g_reserved_sms.load(std::memory_order_relaxed) + 1) / 2;
  return r < 1 ? 1 : r;
}

// Max co-resident CTA pairs of a kernel (the persistent kernels' spin waits need every CTA
// of the grid resident: the grid never exceeds this).
template <typename K>
int max_pairs(K kernel, int threads, int smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (num_sms() / 2));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (const void *)kernel, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = num_sms() / 2;
  }
  return n < num_sms() / 2 ? n : num_sms() / 2;
}

// L2 prefetch distance (k-blocks) of the wide GEMMs' streamed operands, FOLD_PF_FWD /
// FOLD_PF_BWD / FOLD_PF_DU (default 0 = off: measured at C2 B=1024, distances 4 / 8 / 16 made
// dA +7%, dU +8-10% and C5 +15-25% slower; the ring's operands mostly hit L2 already)
int l2_prefetch_dist(const char *env) {
  const char *e = getenv(env);
  return e ? atoi(e) : 0;
}

int dbg_bwd() {
  static int v = [] { const char *e = getenv("FOLD_DBG_BWD"); return e ? atoi(e) : 0; }();
  return v;
}
int dbg_fwd() {
  static int v = [] { const char *e = getenv("FOLD_DBG_FWD"); return e ? atoi(e) : 0; }();
  return v;
}

// First level of the forward's narrow tail: every level d0..D has at most narrow_max rows
// (FOLD_FWD_NARROW_MAX, default 32; 0 disables k_fwd_narrow). D + 1 if there is none or S is
// too large for the stationary U slice.
int fwd_narrow_start(const int32_t *lo, int D, int S) {
  static const int narrow_max = [] {
    const char *e = getenv("FOLD_FWD_NARROW_MAX");
    return e ? atoi(e) : 32;
  }();
  if (narrow_max <= 0 || S > NW_MAX_S || S < 1) return D + 1;
  int d0 = D + 1;
  while (d0 - 1 >= 2 && lo[d0] - lo[d0 - 1] <= narrow_max) d0--;
  return d0;
}

template <int GATES>
fold_status launch_fwd_levels(const TcFwdArgs &a, cudaStream_t st) {
  using Cfg = FwdCfg<GATES>;
  const int S = a.S, nc = a.n_cells;
  CUtensorMap tmAL, tmAR, tmUw, tmUn, tmGw, tmGn, tmUm, tmGm;
  FOLD_TRY(make_map(&tmAL, a.sc.AL, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, BM));
  FOLD_TRY(make_map(&tmAR, a.sc.AR, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, BM));
  CUtensorMap tmAL16, tmAR16, tmAL64, tmAR64;  // narrow tiles: boxes of the rows they hold
  FOLD_TRY(make_map(&tmAL16, a.sc.AL, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, 16));
  FOLD_TRY(make_map(&tmAR16, a.sc.AR, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, 16));
  FOLD_TRY(make_map(&tmAL64, a.sc.AL, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, 64));
  FOLD_TRY(make_map(&tmAR64, a.sc.AR, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, 64));
  const uint64_t il_rows = (uint64_t)cdiv(S, 8) * 8 * GATES;
  FOLD_TRY(make_map(&tmUw, a.Ub, (uint64_t)a.ld_u, il_rows, (uint64_t)a.ld_u * 2, BK, GATES * Cfg::WMAX / 2));
  FOLD_TRY(make_map(&tmUn, a.Ub, (uint64_t)a.ld_u, il_rows, (uint64_t)a.ld_u * 2, BK, GATES * Cfg::WNAR / 2));
  FOLD_TRY(make_map(&tmUm, a.Ub, (uint64_t)a.ld_u, il_rows, (uint64_t)a.ld_u * 2, BK, GATES * Cfg::WMID / 2));
  // epilogue bulk stores: G [n_cells][GATES*S] bf16 and the pool's C [N][S] fp32, plain
  // (unswizzled) boxes of W columns x 128 rows
  FOLD_TRY(make_map_ex(&tmGw, a.Gact, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (uint64_t)a.ld_g, (uint64_t)nc,
                       (uint64_t)a.ld_g * 2, Cfg::WMAX, BM, CU_TENSOR_MAP_SWIZZLE_NONE));
  FOLD_TRY(make_map_ex(&tmGn, a.Gact, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (uint64_t)a.ld_g, (uint64_t)nc,
                       (uint64_t)a.ld_g * 2, Cfg::WNAR, BM, CU_TENSOR_MAP_SWIZZLE_NONE));
  FOLD_TRY(make_map_ex(&tmGm, a.Gact, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (uint64_t)a.ld_g, (uint64_t)nc,
                       (uint64_t)a.ld_g * 2, Cfg::WMID, BM, CU_TENSOR_MAP_SWIZZLE_NONE));
  auto kern = k_fwd_levels<GATES>;
  const int smem_bytes = Cfg::SMEM;
  FOLD_TRY(set_smem(kern, smem_bytes));
  static thread_local int npairs_dev[kMaxDevices] = {};
  int &npairs_dev_max = npairs_dev[cur_dev()];
  if (!npairs_dev_max) npairs_dev_max = max_pairs(kern, Cfg::THREADS, smem_bytes);
  const int npairs_max = reserve_pairs(npairs_dev_max);
  FwdLevels L{a.level_off, a.D, S, Cfg::WMAX, Cfg::WNAR, npairs_max / 2, Cfg::WMID, GATES, npairs_max,
              l2_prefetch_dist("FOLD_PF_FWD")};
  // the narrow tail: levels d0..D all of at most narrow_max rows go to k_fwd_narrow
  const int d0 = fwd_narrow_start(a.level_off_host, a.D, S);
  int64_t total = 0;
  for (int d = 2; d < d0; d++) {
    const int M = a.level_off_host[d + 1] - a.level_off_host[d];
    total += cdiv(M, PM) * cdiv(S, fwd_level_W(L, M));
  }
  if (total > INT32_MAX) return FOLD_E_INVALID;
  if (total <= 0 && d0 > a.D) return FOLD_OK;
  FOLD_CUDA_TRY(cudaMemsetAsync(a.rt_cnt, 0, (size_t)nc * sizeof(int), st));
  {
    int64_t blocks = cdiv(nc, 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_fwd_prelude<<<(unsigned)blocks, 256, 0, st>>>(a.level_off, a.D, a.nl, nc, S, a.gather, a.tstart, a.rt_cnt);
    FOLD_LAUNCH_CHECK();
  }
  if (total > 0) {
    const int npairs = total < npairs_max ? (int)total : npairs_max;
    kern<<<2 * npairs, Cfg::THREADS, smem_bytes, st>>>(tmAL, tmAR, tmAL16, tmAR16, tmAL64, tmAR64, tmUw, tmUn, tmGw,
                                                        tmGn, tmUm, tmGm, L, (int)total, a.nl, a.ld, a.gather, a.b,
                                                        a.H, a.C, a.Gact, a.ld_g, a.sc, a.rt_cnt, a.tstart,
                                                        dbg_fwd());
    FOLD_LAUNCH_CHECK();
  }
  if (d0 <= a.D) {
    using NC = NwCfg<GATES>;
    CUtensorMap tmUs, tmAL8, tmAR8;
    FOLD_TRY(make_map(&tmUs, a.Ub, (uint64_t)a.ld_u, il_rows, (uint64_t)a.ld_u * 2, BK, NC::UROWS));
    FOLD_TRY(make_map(&tmAL8, a.sc.AL, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, NW_ROWS));
    FOLD_TRY(make_map(&tmAR8, a.sc.AR, (uint64_t)S, (uint64_t)nc, (uint64_t)a.sc.ld * 2, BK, NW_ROWS));
    // 4D view of the two planes as [K-block][half][row][64 columns] (S % 64 == 0 and A_R at a
    // fixed offset from A_L): one box = the chunk's 8 rows of both halves and all K-blocks,
    // landing slot-major with the halves interleaved (the B operand's 8-row groups)
    CUtensorMap tmA4;
    const int64_t half_off = (const char *)a.sc.AR - (const char *)a.sc.AL;
    int use3d = (S % BK == 0) && (S / BK) <= 256 && half_off > 0 && half_off % 16 == 0;
    if (use3d) {
      auto enc = encode_fn();
      if (!enc) return FOLD_E_CUDA;
      cuuint64_t dims[4] = {(cuuint64_t)BK, (cuuint64_t)nc, 2, (cuuint64_t)(S / BK)};
      cuuint64_t strides[3] = {(cuuint64_t)a.sc.ld * 2, (cuuint64_t)half_off, (cuuint64_t)BK * 2};
      cuuint32_t box[4] = {(cuuint32_t)BK, (cuuint32_t)NW_ROWS, 2, (cuuint32_t)(S / BK)};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = enc(&tmA4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void *)a.sc.AL, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) use3d = 0;
    }
    if (!use3d) tmA4 = tmAL8;
    const int nsm = NC::smem((int)cdiv(S, BK));
    auto nk = k_fwd_narrow<GATES>;
    FOLD_TRY(set_smem(nk, nsm));
    const int grid = (int)cdiv(S, 8);
    const int32_t *lo = a.level_off;
    int D = a.D, nl = a.nl, ld = a.ld, ld_g = a.ld_g;
    const int32_t *gather = a.gather;
    const float *bias = a.b;
    __nv_bfloat16 *H = a.H, *G = a.Gact;
    float *C = a.C;
    ScatterA sc = a.sc;
    int *rt = a.rt_cnt;
    const int32_t *ts = a.tstart;
    int d0v = d0, Sv = S, dbgv = dbg_fwd() == 2;
    void *args[] = {(void *)&tmUs, (void *)&tmAL8, (void *)&tmAR8, (void *)&tmA4, (void *)&use3d,
                    (void *)&lo, (void *)&d0v, (void *)&D,
                    (void *)&Sv, (void *)&nl, (void *)&ld, (void *)&gather, (void *)&bias, (void *)&H, (void *)&C,
                    (void *)&G, (void *)&ld_g, (void *)&sc, (void *)&rt, (void *)&ts, (void *)&dbgv};
    // cooperative: every CTA must be resident (they wait on each other's published columns)
    FOLD_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)nk, dim3(grid), dim3(NW_THREADS), args, (size_t)nsm, st));
    FOLD_LAUNCH_CHECK();
  }
  return FOLD_OK;
}

}  // namespace

int tc_ld_u(int S) { return 2 * (int)round_up(S, BK); }

int tc_debug_bwd_trace(unsigned long long *host, int n) {
  if (n > kTraceTiles) n = kTraceTiles;
  for (int p = 0; p < 10; p++)
    if (cudaMemcpyFromSymbol(host + (size_t)p * n, g_bwd_trace, (size_t)n * 8, (size_t)p * kTraceTiles * 8) !=
        cudaSuccess)
      return -1;
  for (int p = 0; p < 2; p++)
    if (cudaMemcpyFromSymbol(host + (size_t)(10 + p) * n, g_bwd_clk, (size_t)n * 8, (size_t)p * kTraceTiles * 8) !=
        cudaSuccess)
      return -1;
  return n;
}

int tc_debug_fwd_trace(unsigned long long *host, int n) {
  if (n > kTraceTiles) n = kTraceTiles;
  for (int p = 0; p < 9; p++)
    if (cudaMemcpyFromSymbol(host + (size_t)p * n, g_fwd_trace, (size_t)n * 8, (size_t)p * kTraceTiles * 8) !=
        cudaSuccess)
      return -1;
  return n;
}

size_t tc_weights_bytes(int gates, int S) { return round_up(cdiv(S, 8) * 8 * gates * tc_ld_u(S) * 2, 256); }

fold_status tc_prepare_Uil(int gates, int S, const float *U, __nv_bfloat16 *Uil, cudaStream_t st) {
  const int Sp = tc_ld_u(S) / 2;
  const int64_t rows = cdiv(S, 8) * 8 * gates;
  int64_t blocks = cdiv(rows * (Sp / 4), 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_prep_U<<<(unsigned)blocks, 256, 0, st>>>(rows, S, Sp, U, Uil, gates);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status tc_prepare_U(int gates, int S, const float *U, __nv_bfloat16 *Ub, cudaStream_t st) {
  const int64_t rows = (int64_t)gates * S;
  const int Sp = tc_ld_u(S) / 2;
  int64_t blocks = cdiv(rows * (Sp / 4), 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_prep_U<<<(unsigned)blocks, 256, 0, st>>>(rows, S, Sp, U, Ub, 0);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

// Ut[r][k] = U[k][half * S + j] in bf16 for the padded column r = half * Sp + j (0 for
// j >= S): the narrow backward's K-major copy of U's columns. 32 x 32 tiles through shared
// memory (coalesced reads of U rows and writes of Ut rows).
__global__ void k_prep_Ut(int K, int Kt, int S, int Sp, const float *__restrict__ U, __nv_bfloat16 *__restrict__ Ut) {
  __shared__ float tile[32][33];
  const int R = 2 * Sp;
  const int ntk = (K + 31) / 32, ntr = (R + 31) / 32;
  for (int t = blockIdx.x; t < ntk * ntr; t += gridDim.x) {
    const int k0 = (t / ntr) * 32, r0 = (t % ntr) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // rows k0 + i of U, columns r0 + tx
      const int k = k0 + i, r = r0 + threadIdx.x;
      const int half = r >= Sp, j = r - half * Sp;
      tile[i][threadIdx.x] = (k < K && r < R && j < S) ? __ldg(U + (int64_t)k * 2 * S + half * S + j) : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // rows r0 + i of Ut, columns k0 + tx
      const int r = r0 + i, k = k0 + threadIdx.x;
      if (r < R && k < K) Ut[(int64_t)r * Kt + k] = __float2bfloat16_rn(tile[threadIdx.x][i]);
    }
    __syncthreads();
  }
}

fold_status tc_prepare_Ut(int gates, int S, const float *U, __nv_bfloat16 *Ut, cudaStream_t st) {
  if (!U || !Ut) return FOLD_E_INVALID;
  const int Sp = (int)round_up(S, BK), K = gates * S;
  int64_t tiles = cdiv(K, 32) * cdiv(2 * Sp, 32);
  unsigned grid = (unsigned)(tiles < 148 * 16 ? tiles : 148 * 16);
  k_prep_Ut<<<grid, dim3(32, 8), 0, st>>>(K, (int)round_up(K, 8), S, Sp, U, Ut);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}
size_t tc_ut_bytes(int gates, int S) { return round_up((size_t)2 * round_up(S, BK) * round_up(gates * S, 8) * 2, 256); }

fold_status tc_fwd_levels(int cell, const TcFwdArgs &a, cudaStream_t st) {
  if (a.D < 2) return FOLD_OK;
  if (cell == FOLD_CELL_TREELSTM) return launch_fwd_levels<5>(a, st);
  return launch_fwd_levels<1>(a, st);
}

fold_status tc_gemm_dA(int c0, int M, int n_cells, int S, int gates, const __nv_bfloat16 *dZ, int ld_z,
                       const __nv_bfloat16 *Ub, float *dA, cudaStream_t st) {
  if (M <= 0) return FOLD_OK;
  CUtensorMap tmZ, tmU;
  FOLD_TRY(make_map(&tmZ, dZ, (uint64_t)gates * S, (uint64_t)n_cells, (uint64_t)ld_z * 2, BK, BM));
  const int ld_u = tc_ld_u(S);
  FOLD_TRY(make_map(&tmU, Ub, (uint64_t)ld_u, (uint64_t)gates * S, (uint64_t)ld_u * 2, 64, BK));
  FOLD_TRY(set_smem(k_gemm_dA_tc, DA_SMEM));
  const int NTn = (int)cdiv(ld_u, DA_N);
  const int ntiles = NTn * (int)cdiv(M, PM);
  const int np = ntiles < num_sms() / 2 ? ntiles : num_sms() / 2;
  int KB = (int)cdiv(gates * S, BK);
  k_gemm_dA_tc<<<2 * np, kThreads, DA_SMEM, st>>>(tmZ, tmU, c0, M, KB, S, NTn, ntiles, dA);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

// backward dependency credits: a child row is complete once all S columns of its pointwise
// step are written (credits are columns, so tiles of any width can publish)
int tc_bwd_slabs(int S) { return S; }

fold_status tc_bwd_prelude(const TcBwdArgs &a, const int32_t *cons_off, cudaStream_t st) {
  if (a.n_cells <= 0) return FOLD_OK;
  FOLD_CUDA_TRY(cudaMemsetAsync(a.rt_cnt, 0, (size_t)a.n_cells * sizeof(int), st));
  if (a.ks_cnt) FOLD_CUDA_TRY(cudaMemsetAsync(a.ks_cnt, 0, (size_t)2 * kKsRing * sizeof(int), st));
  int *lvl_flags = a.lvl_tab ? a.lvl_tab + 12 * (a.D + 2) : nullptr;
  if (lvl_flags) FOLD_CUDA_TRY(cudaMemsetAsync(lvl_flags, 0, (size_t)(a.D + 2) * sizeof(int), st));
  int64_t blocks = cdiv(a.n_cells, 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_bwd_prelude<<<(unsigned)blocks, 256, 0, st>>>(a.level_off, a.D, a.nl, a.n_cells, cons_off, a.tstart, a.rt_cnt,
                                                  tc_bwd_slabs(a.S), a.gather, lvl_flags);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

// First level (from the top) handled by the wide backward: levels d1..D all of at most
// FOLD_BWD_NARROW_MAX rows (default 128; 0 disables) run in k_bwd_narrow, which needs
// S <= 1024 (the stationary U slice). D + 1 if none.
int bwd_narrow_start(const int32_t *lo, int D, int S, int gates) {
  // measured: levels of <= 64 rows, and only when there are at least 4 of them. Round 1 chose
  // 128 rows (16-row chunks beat the wide tiles below it); with the wide kernel's split-K
  // units on latency-bound levels, 32-64 rows measure 1-5% better than 128 on C2 B=4..64 and
  // C3, while chains keep needing the narrow kernel (C4 B=64: 9.9 ms with it, 10.9 without);
  // a separate launch for one or two top levels (C2 B=64: the 64-row root level) costs more
  // than it saves
  static const int narrow_max = [] {
    const char *e = getenv("FOLD_BWD_NARROW_MAX");
    return e ? atoi(e) : 64;
  }();
  if (narrow_max <= 0 || S > 1024) return D + 1;
  int d1 = D + 1;
  while (d1 - 1 >= 2 && lo[d1] - lo[d1 - 1] <= narrow_max) d1--;
  static const bool forced = getenv("FOLD_BWD_NARROW_MAX") != nullptr;  // test hook: no minimum
  if (!forced && D + 1 - d1 < 4) return D + 1;
  return d1;
}

fold_status tc_bwd_levels(int cell, const TcBwdArgs &a, cudaStream_t st) {
  if (a.D < 2) return FOLD_OK;
  const int S = a.S, gates = cell == FOLD_CELL_TREELSTM ? 5 : 1;
  if (S & 1) return FOLD_E_UNSUPPORTED;
  CUtensorMap tmZ, tmZ16, tmZ64, tmU;
  FOLD_TRY(make_map(&tmZ, a.dZ, (uint64_t)gates * S, (uint64_t)a.n_cells, (uint64_t)a.ld_z * 2, BK, BM));
  FOLD_TRY(make_map(&tmZ16, a.dZ, (uint64_t)gates * S, (uint64_t)a.n_cells, (uint64_t)a.ld_z * 2, BK, 16));
  FOLD_TRY(make_map(&tmZ64, a.dZ, (uint64_t)gates * S, (uint64_t)a.n_cells, (uint64_t)a.ld_z * 2, BK, 64));
  const int ld_u = tc_ld_u(S);
  FOLD_TRY(make_map(&tmU, a.Ub, (uint64_t)ld_u, (uint64_t)gates * S, (uint64_t)ld_u * 2, 64, BK));
  auto kern = gates == 5 ? k_bwd_levels<5> : k_bwd_levels<1>;
  FOLD_TRY(set_smem(kern, BW_SMEM));
  static thread_local int npairs_dev[kMaxDevices] = {};
  int &npairs_dev_max = npairs_dev[cur_dev()];
  if (!npairs_dev_max) npairs_dev_max = max_pairs(kern, BW_THREADS, BW_SMEM);
  const int npairs_max = reserve_pairs(npairs_dev_max);
  // the narrow top: levels D..d1 (all of at most FOLD_BWD_NARROW_MAX rows) run first in
  // k_bwd_narrow, the wide kernel takes levels d1-1..2
  const int d1 = bwd_narrow_start(a.level_off_host, a.D, S, gates);
  if (d1 <= a.D) {
    const int Kp = (int)round_up(cdiv(gates * S, NB_PARTS), BK);
    int packed = (gates * S) % (NB_PARTS * BK) == 0;
    const int nsm = (Kp / BK) * (NB_PARTS * 16 * 128) + NB_ST * NB_STAGE + 1024;
    auto enc = encode_fn();
    if (!enc) return FOLD_E_CUDA;
    FOLD_TRY(tc_prepare_Ut(gates, S, a.U, a.Ut, st));
    CUtensorMap tmU3, tmZ4a, tmZ4b, tmZ4c, tmU2, tmZ2a, tmZ2b;
    // per-(part, K-block) 2D boxes for S where GATES*S is not 8 K-blocks' multiple (K past
    // GATES*S out of bounds = zero)
    const int Kt = (int)round_up(gates * S, 8);  // Ut row stride (16-byte aligned rows)
    FOLD_TRY(make_map(&tmU2, a.Ut, (uint64_t)gates * S, (uint64_t)ld_u, (uint64_t)Kt * 2, BK, 16));
    FOLD_TRY(make_map(&tmZ2a, a.dZ, (uint64_t)gates * S, (uint64_t)a.n_cells, (uint64_t)a.ld_z * 2, BK, 4));
    FOLD_TRY(make_map(&tmZ2b, a.dZ, (uint64_t)gates * S, (uint64_t)a.n_cells, (uint64_t)a.ld_z * 2, BK, NB_RMAX));
    tmU3 = tmU2;  // (replaced below when packed)
    tmZ4a = tmZ2a;
    tmZ4b = tmZ2b;
    tmZ4c = tmZ2a;
    if (packed) {
      {  // Ut [2 Sp][GATES*S] viewed as [part][row][K in part]: box 64 K x 16 rows x 8 parts
        const int K = gates * S;
        cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)ld_u, (cuuint64_t)NB_PARTS};
        cuuint64_t strides[2] = {(cuuint64_t)Kt * 2, (cuuint64_t)Kp * 2};
        cuuint32_t box[3] = {(cuuint32_t)BK, 16, (cuuint32_t)NB_PARTS};
        cuuint32_t es[3] = {1, 1, 1};
        if (enc(&tmU3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void *)a.Ut, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return FOLD_E_CUDA;
      }
      for (int v = 0; v < 3; v++) {  // dZ viewed as [K-block][part][row][64]: box = R rows x 8 parts x K-blocks
        const int R = v == 1 ? NB_RMAX : 4;
        const int nslot_box = v == 2 ? Kp / BK : NB_STAGE / (NB_PARTS * R * 128);
        if (v == 2 && (nslot_box > 256 || nslot_box * NB_PARTS * 4 * 128 > NB_ST * NB_STAGE)) { tmZ4c = tmZ4a; continue; }
        cuuint64_t dims[4] = {(cuuint64_t)BK, (cuuint64_t)a.n_cells, (cuuint64_t)NB_PARTS, (cuuint64_t)(Kp / BK)};
        cuuint64_t strides[3] = {(cuuint64_t)a.ld_z * 2, (cuuint64_t)Kp * 2, (cuuint64_t)BK * 2};
        cuuint32_t box[4] = {(cuuint32_t)BK, (cuuint32_t)R, (cuuint32_t)NB_PARTS, (cuuint32_t)nslot_box};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (enc(v == 2 ? &tmZ4c : v ? &tmZ4b : &tmZ4a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void *)a.dZ, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return FOLD_E_CUDA;
      }
    }
    auto nk = gates == 5 ? k_bwd_narrow<5> : k_bwd_narrow<1>;
    FOLD_TRY(set_smem(nk, nsm));
    const int grid = ld_u / 16;
    const int32_t *lo = a.level_off;
    int D = a.D, d1v = d1, Sv = S, nl = a.nl, Kpv = Kp, ld_g = a.ld_g, ld = a.ld, ld_z = a.ld_z;
    const int32_t *gather = a.gather, *ts = a.tstart;
    const __nv_bfloat16 *G = a.Gact;
    const float *C = a.C;
    float *dA = a.dA, *dCe = a.dCe;
    __nv_bfloat16 *dZ = a.dZ;
    int *rt = a.rt_cnt;
    void *args[] = {(void *)&tmU3, (void *)&tmZ4a, (void *)&tmZ4b, (void *)&tmZ4c, (void *)&tmU2, (void *)&tmZ2a, (void *)&tmZ2b,
                    (void *)&packed, (void *)&lo, (void *)&D, (void *)&d1v, (void *)&Sv, (void *)&nl,
                    (void *)&Kpv, (void *)&gather, (void *)&G, (void *)&ld_g, (void *)&C, (void *)&ld, (void *)&dA,
                    (void *)&dCe, (void *)&dZ, (void *)&ld_z, (void *)&rt, (void *)&ts};
    FOLD_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)nk, dim3(grid), dim3(NB_THREADS), args, (size_t)nsm, st));
    FOLD_LAUNCH_CHECK();
  }
  // FOLD_BWD_KSPLIT=0 disables the split-K units of latency-bound levels, 2 keeps them to
  // 128-column tiles (A/B switches; C3 B=1024 dA 0.60 -> 0.50 ms, C4 12.1 -> 11.2-11.5 ms)
  static const int ksplit_on = [] { const char *e = getenv("FOLD_BWD_KSPLIT"); return e ? atoi(e) : 1; }();
  const int KB = (int)cdiv(gates * S, BK);
  if (!a.lvl_tab) return FOLD_E_INVALID;
  const int4 *tcrit = reinterpret_cast<const int4 *>(a.lvl_tab), *tinl = tcrit + (a.D + 2), *tend = tinl + (a.D + 2);
  const int *ttotal = a.lvl_tab + 13 * (a.D + 2);
  BwdLevels L{a.level_off, d1 - 1, S, a.nl, ld_u, npairs_max, l2_prefetch_dist("FOLD_PF_BWD"),
              (ksplit_on && a.ks_ring && a.ks_cnt && npairs_max >= 2) ? npairs_max : 0, KB, ksplit_on != 2,
              tcrit, tinl, tend, ttotal};
  // an upper bound of the units (128-column tiles, all split): the tables are built on the
  // device from the levels' child slots; the kernel reads the exact count
  int64_t total = 0;
  for (int d = 2; d < d1; d++) total += cdiv(a.level_off_host[d + 1] - a.level_off_host[d], PM) * cdiv(ld_u, 128) * 2;
  if (total <= 0) return FOLD_OK;
  if (total > INT32_MAX) return FOLD_E_INVALID;
  static const int defer = [] { const char *e = getenv("FOLD_BWD_DEFER"); return e ? atoi(e) : 1; }();
  k_bwd_tiles<<<1, 1024, 0, st>>>(a.level_off, a.D, d1 - 1, (int)round_up(S, BK), ld_u, KB, npairs_max, L.ksplit_max,
                                L.ks256, defer, a.lvl_tab);
  FOLD_LAUNCH_CHECK();
  const int npairs = total < npairs_max ? (int)total : npairs_max;
  kern<<<2 * npairs, BW_THREADS, BW_SMEM, st>>>(tmZ, tmZ16, tmZ64, tmU, L, KB, (int)total, a.gather,
                                               a.Gact, a.ld_g, a.C, a.ld, a.dA, a.dCe, a.dZ, a.ld_z, a.rt_cnt,
                                               a.tstart, tc_bwd_slabs(S), dbg_bwd(), a.ks_ring, a.ks_cnt,
                                               a.ks_cnt ? a.ks_cnt + kKsRing : nullptr);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

int tc_dU_splits(int n_cells, int gates, int S) {
  // split-K count minimising (waves of CTA pairs) x (k-blocks per split) + the partial
  // slabs' round trip: one CTA pair per SM pair, ~0.27 us per k-block of a pair tile at
  // S = 1024 (scaled by the tile count below), ~14 us per extra 42 MB partial at S = 1024
  // (C2 B=1024: 2 splits ran 4.3 waves, the last one third full; 6 splits run 13.0)
  const int64_t pairs = 2 * cdiv(S, DU_N) * cdiv((int64_t)gates * S, PM);  // CTA pairs per split
  const int64_t per_wave = num_sms() / 2;
  const int64_t kbs = cdiv(n_cells, BK);
  const int64_t cap = kbs / 32;  // keep >= 32 k-blocks (2048 cells) per split
  const double part = 14.0 * ((double)gates * S * 2 * S) / (5.0 * 1024 * 2048) / 0.27;  // in k-block units
  int64_t best = 1;
  double best_t = 1e300;
  for (int64_t sp = 1; sp <= 16 && (sp == 1 || sp <= cap); sp++) {
    const double t = (double)cdiv(pairs * sp, per_wave) * (double)cdiv(kbs, sp) + (sp > 1 ? sp * part : 0.0);
    if (t < best_t - 1e-9) { best_t = t; best = sp; }
  }
  return (int)best;
}

fold_status tc_gemm_dU(int n_cells, int S, int gates, const __nv_bfloat16 *dZ, int ld_z, const ScatterA &sc,
                       float *dU, int accumulate, float *split_ws, float *db, float *db_ws, cudaStream_t st) {
  CUtensorMap tmZ2, tmAL, tmAR;
  const uint64_t ncr = (uint64_t)(n_cells > 0 ? n_cells : 1);
  FOLD_TRY(make_map(&tmZ2, dZ, (uint64_t)gates * S, ncr, (uint64_t)ld_z * 2, 64, BK));
  FOLD_TRY(make_map(&tmAL, sc.AL, (uint64_t)S, ncr, (uint64_t)sc.ld * 2, 64, BK));
  FOLD_TRY(make_map(&tmAR, sc.AR, (uint64_t)S, ncr, (uint64_t)sc.ld * 2, 64, BK));
  FOLD_TRY(set_smem(k_gemm_dU_tc, DU_SMEM));
  const int NT = (int)cdiv(S, DU_N);
  const int splits = tc_dU_splits(n_cells, gates, S);
  const int KBall = (int)cdiv(n_cells, BK);
  const int kbps = (int)cdiv(KBall, splits);
  dim3 grid((unsigned)(2 * 2 * NT), (unsigned)cdiv(gates * S, PM), (unsigned)splits);
  const int64_t n = (int64_t)gates * S * 2 * S;
  // db (optional): straight into db with one split, else per-split partials in db_ws
  if (db && splits > 1 && !db_ws) return FOLD_E_WORKSPACE;
  float *dbo = db ? (splits == 1 ? db : db_ws) : nullptr;
  const int dbacc = splits == 1 ? accumulate : 0;
  if (splits == 1) {
    k_gemm_dU_tc<<<grid, kThreads, DU_SMEM, st>>>(tmZ2, tmAL, tmAR, n_cells, S, gates * S, NT, kbps, dU, 0,
                                                  accumulate, dbo, dbacc, l2_prefetch_dist("FOLD_PF_DU"));
    FOLD_LAUNCH_CHECK();
    return FOLD_OK;
  }
  if (!split_ws) return FOLD_E_WORKSPACE;
  k_gemm_dU_tc<<<grid, kThreads, DU_SMEM, st>>>(tmZ2, tmAL, tmAR, n_cells, S, gates * S, NT, kbps, split_ws, n, 0,
                                                dbo, 0, l2_prefetch_dist("FOLD_PF_DU"));
  FOLD_LAUNCH_CHECK();
  FOLD_TRY(launch_reduce_splits(n, splits, split_ws, dU, accumulate, st));
  if (db) FOLD_TRY(launch_reduce_splits((int64_t)gates * S, splits, db_ws, db, accumulate, st));
  return FOLD_OK;
}

int set_reserved_sms(int n) { return g_reserved_sms.exchange(n < 0 ? 0 : n); }

}  // namespace fold

// gemm_tf32.cu — the contractions of the FP32 and TF32 precision modes on the 5th-gen tensor
// cores (tcgen05.mma kind::tf32), plus the per-level gather / pointwise kernels around them.
//
// The three GEMM passes of the method (SURVEY §8(a) a8 Z = [h_L | h_R] U^T, a12 dA = dZ U,
// a14 dU = dZ^T [h_L | h_R]; PAPER.md L47 / L49) run in one generic kernel, k_gemm_tf32:
// one CTA per 128 x BN output tile, TMA streams 128-byte (32 x fp32) K blocks of A and B
// (each K-major or MN-major, 128B-swizzled) into a 3-4 stage ring, one elected thread issues
// the MMAs into a TMEM accumulator, four epilogue warps read it back (tcgen05.ld) and store
// (or accumulate) fp32 rows.
//   npass = 1 (FOLD_PREC_TF32): one MMA per K step; the tensor core reads the fp32
//             containers as TF32 (10 explicit mantissa bits): ~1e-3 relative per product.
//   npass = 3 (FOLD_PREC_FP32, "3xTF32"): x = hi + lo with hi = x truncated to TF32 (what
//             the tensor core reads from the raw tile) and lo = x - hi (exact in fp32, then
//             read as TF32): A B ~ A_hi B_hi + A_hi B_lo + A_lo B_hi, error ~2^-21 relative per
//             product (the dropped lo*lo and TF32-of-lo terms) — fp32-class results at a third
//             of the TF32 rate. The lo tiles are made in shared memory by the (otherwise idle)
//             epilogue warps after each stage lands, so HBM traffic is that of one fp32 pass.
// Split-K over the reduction (the all-cells dU GEMM at small state sizes) writes per-split
// partial slabs reduced in fixed order (deterministic: no float atomics).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <unordered_map>

#include "exec.cuh"
#include "ptx.cuh"

namespace fold {

fold_status make_map_ex(CUtensorMap *m, const void *ptr, CUtensorMapDataType dt, uint64_t cols, uint64_t rows,
                        uint64_t row_bytes, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw);

namespace {

constexpr int TM = 128;          // output rows per CTA (MMA M)
constexpr int TK = 32;           // K elements per stage block (128 B of fp32 = one swizzle row)
constexpr int TF_THREADS = 256;  // warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4-7 split + epilogue
constexpr int A_TILE = TM * 128;  // bytes of one A block (128 rows or 4 MN chunks x 32 K rows)

template <int BN, int NPASS>
struct TfCfg {
  static constexpr int B_TILE = BN * 128;
  static constexpr int RAW = A_TILE + B_TILE;
  static constexpr int STAGE = NPASS == 3 ? 2 * RAW : RAW;  // raw tiles, then their lo parts
  static constexpr int NST = (200 * 1024) / STAGE > 6 ? 6 : (200 * 1024) / STAGE;
  static constexpr int SMEM = NST * STAGE + 1024;
  static_assert(NST >= 2, "pipeline depth");
};

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
  return p + ((1024u - (ptx::smem_u32(p) & 1023u)) & 1023u);
}

// kind::tf32 instruction descriptor: D fp32 (bit 4), A / B format TF32 (2 at bits 7, 10),
// majors (bits 15, 16), N >> 3 (17..22), M >> 4 (24..28)
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// shared-memory descriptor of K step k (8 fp32 of K = 32 bytes) of an operand block:
// K-major: 128B swizzle (16-byte chunks XOR row mod 8), rows of 128 B along K, 8-row atoms
//   1024 B apart (SBO), the step advances 32 B within the rows;
// MN-major: TF32 MN-major operands take the "128B swizzle with 32-byte atoms" layout
//   (descriptor layout type 1; TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: 32-byte chunks XOR
//   row mod 4): 128 B (32 elements) of M/N per K row, 4-row atoms 512 B apart (SBO), so a
//   K step (8 rows) is two atoms and advances 1024 B; MN chunks of 32 K rows 4096 B apart (LBO)
__device__ __forceinline__ uint64_t sdesc_mn32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(4096 >> 4) << 16;  // LBO: next 32-element MN chunk
  d |= (uint64_t)(512 >> 4) << 32;   // SBO: next 4-row K atom
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)1 << 61;            // SWIZZLE_128B_BASE32B
  return d;
}
__device__ __forceinline__ uint64_t tf_desc(uint32_t base, int k, int mn_major) {
  return mn_major ? sdesc_mn32(base + 1024u * (uint32_t)k) : ptx::sdesc_sw128(base + 32u * (uint32_t)k, 16, 1024);
}

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t lo_part(uint32_t x) {
  // x - trunc_tf32(x): exact in fp32 (Sterbenz); the tensor core then reads it as TF32
  const float f = __uint_as_float(x), hi = __uint_as_float(x & 0xFFFFE000u);
  return __float_as_uint(f - hi);
}

// Load one operand block (rows x 32 K) of operand X at (row0, k0) into dst:
//   K-major: one box (32 K x rows) at (k0, row0);  MN-major: rows / 32 boxes (32 MN x 32 K)
//   at (row0 + 32 c, k0).
__device__ __forceinline__ void load_block(const CUtensorMap *m, uint64_t *bar, uint8_t *dst, int mn_major, int rows,
                                           int row0, int k0) {
  if (!mn_major) {
    ptx::tma_load_2d(m, bar, dst, k0, row0);
  } else {
    for (int c = 0; c < rows / 32; c++) ptx::tma_load_2d(m, bar, dst + c * 4096, row0 + 32 * c, k0);
  }
}

// One output tile (m0, n0) of one problem, K blocks [kb0, kb0 + kb_per_split) (the body of
// the single-problem and the grouped kernels below).
template <int BN, int NPASS>
__device__ __forceinline__ void gemm_tf32_tile(const CUtensorMap *pA, const CUtensorMap *pB, int a_mn, int b_mn,
                                               int M, int N, int K, int kb_per_split, float *__restrict__ C,
                                               int64_t ldc, int64_t split_stride, int accumulate, int m0, int n0,
                                               int split) {
  using Cfg = TfCfg<BN, NPASS>;
  constexpr int ST = Cfg::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t full[ST], ready[ST], empty[ST], tfull;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KBall = (K + TK - 1) / TK;
  const int kb0 = split * kb_per_split;
  const int kb1 = min(KBall, kb0 + kb_per_split);
  const int KB = kb1 > kb0 ? kb1 - kb0 : 0;
  float *Cz = C + (int64_t)split * split_stride;
  const CUtensorMap &tmA = *pA, &tmB = *pB;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&ready[s], 4);  // the 4 splitter warps (3xTF32)
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(&tfull, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 2) { ptx::tmem_alloc(&tmem_base_sh, BN); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < KB; it++) {
        const int s = it % ST;
        const uint32_t ph = (it / ST) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], Cfg::RAW);
        uint8_t *A = smem + s * Cfg::STAGE;
        const int k0 = (kb0 + it) * TK;
        load_block(&tmA, &full[s], A, a_mn, TM, m0, k0);
        load_block(&tmB, &full[s], A + A_TILE, b_mn, BN, n0, k0);
      }
    }
  } else if (warp == 1) {
    {  // converged warp, elected lane issues (ptx::elect_one)
      constexpr int kN = BN;
      const uint32_t idesc = idesc_tf32(TM, kN, a_mn, b_mn);
      for (int it = 0; it < KB; it++) {
        const int s = it % ST;
        const uint32_t ph = (it / ST) & 1;
        ptx::mbar_wait(NPASS == 3 ? &ready[s] : &full[s], ph);
        __syncwarp();
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(smem + s * Cfg::STAGE), b0 = a0 + A_TILE;
        uint64_t ad[TK / 8], bd[TK / 8], al[TK / 8], bl[TK / 8];
#pragma unroll
        for (int k = 0; k < TK / 8; k++) {
          ad[k] = tf_desc(a0, k, a_mn); bd[k] = tf_desc(b0, k, b_mn);
          al[k] = tf_desc(a0 + Cfg::RAW, k, a_mn); bl[k] = tf_desc(b0 + Cfg::RAW, k, b_mn);
        }
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < TK / 8; k++) {
            umma_tf32(tbase, ad[k], bd[k], idesc, (it | k) != 0);
            if constexpr (NPASS == 3) {
              umma_tf32(tbase, ad[k], bl[k], idesc, 1);  // A_hi B_lo
              umma_tf32(tbase, al[k], bd[k], idesc, 1);  // A_lo B_hi
            }
          }
          ptx::umma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (KB > 0 && ptx::elect_one()) ptx::umma_commit(&tfull);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int t = tid - 128;
    if constexpr (NPASS == 3) {
      // split each landed stage: lo = x - trunc_tf32(x) into the stage's second half
      for (int it = 0; it < KB; it++) {
        const int s = it % ST;
        ptx::mbar_wait(&full[s], (it / ST) & 1);
        const uint32_t raw = ptx::smem_u32(smem + s * Cfg::STAGE);
        for (int i = t; i < Cfg::RAW / 16; i += 128) {
          const uint4 v = ptx::lds128(raw + 16 * i);
          sts128(raw + Cfg::RAW + 16 * i, make_uint4(lo_part(v.x), lo_part(v.y), lo_part(v.z), lo_part(v.w)));
        }
        ptx::fence_proxy_async_smem();  // generic writes -> the MMA's (async proxy) reads
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ready[s]);
      }
    }
    // epilogue: TMEM lane = output row, 8 columns per tcgen05.ld
    if (KB > 0) ptx::mbar_wait(&tfull, 0);
    ptx::tc_fence_after();
    const int q = warp & 3, row = m0 + q * 32 + lane;
    const uint32_t tl = tbase + ((uint32_t)(q * 32) << 16);
    float *out = Cz + (int64_t)row * ldc;
    const bool vec = ((ldc & 3) == 0) && ((((uintptr_t)Cz) & 15) == 0);
#pragma unroll 1
    for (int nc = 0; nc < BN / 8; nc++) {
      float v[8];
      ptx::tmem_ld8(tl + nc * 8, v);
      ptx::tmem_ld_wait();
      const int j = n0 + nc * 8;
      if (row >= M || j >= N) continue;
      if (KB == 0) {
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = 0.f;
      }
      if (vec && j + 8 <= N && !accumulate) {
        *reinterpret_cast<float4 *>(out + j) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(out + j + 4) = make_float4(v[4], v[5], v[6], v[7]);
      } else {
        for (int u = 0; u < 8 && j + u < N; u++) out[j + u] = accumulate ? out[j + u] + v[u] : v[u];
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, BN); }
}

template <int BN, int NPASS>
__global__ void __launch_bounds__(TF_THREADS, 1)
    k_gemm_tf32(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int a_mn, int b_mn,
                int M, int N, int K, int kb_per_split, float *__restrict__ C, int64_t ldc, int64_t split_stride,
                int accumulate) {
  gemm_tf32_tile<BN, NPASS>(&tmA, &tmB, a_mn, b_mn, M, N, K, kb_per_split, C, ldc, split_stride, accumulate,
                            blockIdx.y * TM, blockIdx.x * BN, blockIdx.z);
}

// Grouped: up to kTfGroupMax independent problems in ONE launch (the multi-op executor's
// per-level operations, "each iteration of the loop will evaluate all of the
// operations at a particular depth"); blockIdx.x enumerates the problems' output tiles
// (problem p owns tiles [tile_start[p], tile_start[p + 1])), blockIdx.z the K split.
template <int BN, int NPASS>
__global__ void __launch_bounds__(TF_THREADS, 1) k_gemm_tf32_grouped(const __grid_constant__ TfGroupArgs P) {
  int p = 0;
  while (p + 1 < P.n && (int)blockIdx.x >= P.tile_start[p + 1]) p++;
  if ((int)blockIdx.z >= P.nsplit[p]) return;  // another problem of the launch uses more splits
  const int lt = (int)blockIdx.x - P.tile_start[p];
  const int m0 = (lt / P.ntn[p]) * TM, n0 = (lt % P.ntn[p]) * BN;
  gemm_tf32_tile<BN, NPASS>(&P.ta[p], &P.tb[p], P.a_mn[p], P.b_mn[p], P.M[p], P.N[p], P.K[p], P.kbps[p], P.C[p],
                            P.ldc[p], P.split_stride[p], P.accumulate[p], m0, n0, blockIdx.z);
}

// ---------------------------------------------------------------- CTA-pair variant
// Pair tile 256 rows x BN (cluster of 2, tcgen05.mma.cta_group::2.kind::tf32, M = 256): each
// CTA stages its 128 A rows and BN/2 of the B rows (columns), so per SM the tensor core's
// shared-memory operand reads and the TMA ingress per FLOP are those of a 128 x 2BN tile
// (B200 guide: "in 2CTA mode two SMs share operands -> per-SM smem bandwidth halves"; the
// single-CTA 128 x 128 TF32 tile reads 128 B/clk of operands, the whole shared-memory port).
// 3xTF32: each CTA's splitter warps split their own stage (A rows + B half) and arrive on the
// leader's `ready` barrier (8 warps); the leader's MMA warp waits on it and issues
// A_hi B_hi + A_hi B_lo + A_lo B_hi for the pair.
template <int BN, int NPASS>
struct TfPairCfg {
  static constexpr int A_T = TM * 128;          // 128 rows x 32 fp32
  static constexpr int B_T = (BN / 2) * 128;    // this CTA's BN / 2 rows (columns) of B
  static constexpr int RAW = A_T + B_T;
  static constexpr int STAGE = NPASS == 3 ? 2 * RAW : RAW;
  static constexpr int NST = (200 * 1024) / STAGE > 6 ? 6 : (200 * 1024) / STAGE;
  static constexpr int SMEM = NST * STAGE + 1024;
  static_assert(NST >= 2, "pipeline depth");
};

__device__ __forceinline__ void umma_tf32_2cta(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// release at cluster scope: the arriving CTA's generic shared-memory writes (the lo tiles) are
// made visible to the async proxy first (fence.proxy.async), then the leader's MMA reads them
__device__ __forceinline__ void arrive_leader_cluster(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ptx::smem_u32(bar) &
                                                                                     ptx::kLeaderMask)
               : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D_%=;\n\t"
      "bra W_%=;\n"
      "D_%=:\n\t}" ::"r"(ptx::smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// load_block into this CTA of a pair: `pair_bar` (NPASS = 1) completes on the leader's barrier
__device__ __forceinline__ void load_block_pair(const CUtensorMap *m, uint64_t *bar, uint8_t *dst, int mn_major,
                                                int rows, int row0, int k0, bool to_leader) {
  if (!mn_major) {
    if (to_leader) ptx::tma_load_2d_pair(m, bar, dst, k0, row0);
    else ptx::tma_load_2d(m, bar, dst, k0, row0);
  } else {
    for (int c = 0; c < rows / 32; c++) {
      if (to_leader) ptx::tma_load_2d_pair(m, bar, dst + c * 4096, row0 + 32 * c, k0);
      else ptx::tma_load_2d(m, bar, dst + c * 4096, row0 + 32 * c, k0);
    }
  }
}

// one pair tile: rows [m0, m0 + 256) (this CTA: m0 + 128 rank ..), columns [n0, n0 + BN)
template <int BN, int NPASS>
__device__ __forceinline__ void gemm_tf32_pair_tile(const CUtensorMap *pA, const CUtensorMap *pB, int a_mn, int b_mn,
                                                    int M, int N, int K, int kb_per_split, float *__restrict__ C,
                                                    int64_t ldc, int64_t split_stride, int accumulate, int m0, int n0,
                                                    int split) {
  using Cfg = TfPairCfg<BN, NPASS>;
  constexpr int ST = Cfg::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t full[ST], ready[ST], empty[ST], tfull;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int KBall = (K + TK - 1) / TK;
  const int kb0 = split * kb_per_split;
  const int kb1 = min(KBall, kb0 + kb_per_split);
  const int KB = kb1 > kb0 ? kb1 - kb0 : 0;
  float *Cz = C + (int64_t)split * split_stride;
  const CUtensorMap &tmA = *pA, &tmB = *pB;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&ready[s], 8);  // the 4 splitter warps of both CTAs (3xTF32; leader's copy)
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(&tfull, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 2) { ptx::tmem_alloc2(&tmem_base_sh, BN); ptx::tmem_relinquish2(); }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  const int arow = m0 + (int)rank * TM, brow = n0 + (int)rank * (BN / 2);

  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < KB; it++) {
        const int s = it % ST;
        const uint32_t ph = (it / ST) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        uint8_t *A = smem + s * Cfg::STAGE;
        const int k0 = (kb0 + it) * TK;
        if constexpr (NPASS == 3) {  // each CTA's own barrier: its splitter waits on it
          ptx::mbar_arrive_expect_tx(&full[s], Cfg::RAW);
          load_block_pair(&tmA, &full[s], A, a_mn, TM, arow, k0, false);
          load_block_pair(&tmB, &full[s], A + Cfg::A_T, b_mn, BN / 2, brow, k0, false);
        } else {  // both CTAs' bytes complete on the leader's barrier (the MMA issuer's)
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * Cfg::RAW);
          load_block_pair(&tmA, &full[s], A, a_mn, TM, arow, k0, true);
          load_block_pair(&tmB, &full[s], A + Cfg::A_T, b_mn, BN / 2, brow, k0, true);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // converged warp, elected lane issues
      const uint32_t idesc = idesc_tf32(2 * TM, BN, a_mn, b_mn);
      for (int it = 0; it < KB; it++) {
        const int s = it % ST;
        const uint32_t ph = (it / ST) & 1;
        if constexpr (NPASS == 3) wait_cluster(&ready[s], ph);
        else ptx::mbar_wait(&full[s], ph);
        __syncwarp();
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(smem + s * Cfg::STAGE), b0 = a0 + Cfg::A_T;
        uint64_t ad[TK / 8], bd[TK / 8], al[TK / 8], bl[TK / 8];
#pragma unroll
        for (int k = 0; k < TK / 8; k++) {
          ad[k] = tf_desc(a0, k, a_mn); bd[k] = tf_desc(b0, k, b_mn);
          al[k] = tf_desc(a0 + Cfg::RAW, k, a_mn); bl[k] = tf_desc(b0 + Cfg::RAW, k, b_mn);
        }
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < TK / 8; k++) {
            umma_tf32_2cta(tbase, ad[k], bd[k], idesc, (it | k) != 0);
            if constexpr (NPASS == 3) {
              umma_tf32_2cta(tbase, ad[k], bl[k], idesc, 1);  // A_hi B_lo
              umma_tf32_2cta(tbase, al[k], bd[k], idesc, 1);  // A_lo B_hi
            }
          }
          ptx::umma_commit_2cta(&empty[s]);
        }
        __syncwarp();
      }
      if (KB > 0 && ptx::elect_one()) ptx::umma_commit_2cta(&tfull);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int t = tid - 128;
    if constexpr (NPASS == 3) {
      for (int it = 0; it < KB; it++) {
        const int s = it % ST;
        ptx::mbar_wait(&full[s], (it / ST) & 1);
        const uint32_t raw = ptx::smem_u32(smem + s * Cfg::STAGE);
        for (int i = t; i < Cfg::RAW / 16; i += 128) {
          const uint4 v = ptx::lds128(raw + 16 * i);
          sts128(raw + Cfg::RAW + 16 * i, make_uint4(lo_part(v.x), lo_part(v.y), lo_part(v.z), lo_part(v.w)));
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) arrive_leader_cluster(&ready[s]);
      }
    }
    if (KB > 0) ptx::mbar_wait(&tfull, 0);
    ptx::tc_fence_after();
    const int q = warp & 3, row = arow + q * 32 + lane;
    const uint32_t tl = tbase + ((uint32_t)(q * 32) << 16);
    float *out = Cz + (int64_t)row * ldc;
    const bool vec = ((ldc & 3) == 0) && ((((uintptr_t)Cz) & 15) == 0);
#pragma unroll 1
    for (int nc = 0; nc < BN / 8; nc++) {
      float v[8];
      ptx::tmem_ld8(tl + nc * 8, v);
      ptx::tmem_ld_wait();
      const int j = n0 + nc * 8;
      if (row >= M || j >= N) continue;
      if (KB == 0) {
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = 0.f;
      }
      if (vec && j + 8 <= N && !accumulate) {
        *reinterpret_cast<float4 *>(out + j) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(out + j + 4) = make_float4(v[4], v[5], v[6], v[7]);
      } else {
        for (int u = 0; u < 8 && j + u < N; u++) out[j + u] = accumulate ? out[j + u] + v[u] : v[u];
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, BN); }
}

template <int BN, int NPASS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TF_THREADS, 1)
    k_gemm_tf32_p(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int a_mn,
                  int b_mn, int M, int N, int K, int kb_per_split, float *__restrict__ C, int64_t ldc,
                  int64_t split_stride, int accumulate) {
  gemm_tf32_pair_tile<BN, NPASS>(&tmA, &tmB, a_mn, b_mn, M, N, K, kb_per_split, C, ldc, split_stride, accumulate,
                                 blockIdx.y * 2 * TM, (blockIdx.x >> 1) * BN, blockIdx.z);
}

template <int BN, int NPASS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TF_THREADS, 1)
    k_gemm_tf32_grouped_p(const __grid_constant__ TfGroupArgs P) {
  const int tile = (int)(blockIdx.x >> 1);
  int p = 0;
  while (p + 1 < P.n && tile >= P.tile_start[p + 1]) p++;
  if ((int)blockIdx.z >= P.nsplit[p]) return;  // (both CTAs of the pair return together)
  const int lt = tile - P.tile_start[p];
  const int m0 = (lt / P.ntn[p]) * 2 * TM, n0 = (lt % P.ntn[p]) * BN;
  gemm_tf32_pair_tile<BN, NPASS>(&P.ta[p], &P.tb[p], P.a_mn[p], P.b_mn[p], P.M[p], P.N[p], P.K[p], P.kbps[p],
                                 P.C[p], P.ldc[p], P.split_stride[p], P.accumulate[p], m0, n0, blockIdx.z);
}

template <typename K>
fold_status set_smem_tf(K kernel, int bytes) {
  static thread_local std::unordered_map<const void *, int> set;
  const void *key = (const char *)(const void *)kernel + cur_dev();
  auto it = set.find(key);
  if (it != set.end() && it->second >= bytes) return FOLD_OK;
  FOLD_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  set[key] = bytes;
  return FOLD_OK;
}

int sm_count() {
  static int n[kMaxDevices] = {};
  const int dev = cur_dev();
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

// operand map: K-major = rows x K (box 32 K x rows), MN-major = K rows x MN (box 32 x 32)
fold_status tf_map(CUtensorMap *m, const TfOperand &x, int rows_mn, int K, int box_rows) {
  if (((uintptr_t)x.p & 15) || (x.ld & 3)) return FOLD_E_INVALID;
  if (!x.mn_major)
    return make_map_ex(m, x.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (uint64_t)K, (uint64_t)rows_mn, (uint64_t)x.ld * 4,
                       TK, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
  return make_map_ex(m, x.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (uint64_t)rows_mn, (uint64_t)K, (uint64_t)x.ld * 4, 32,
                     TK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

// BN = 128 for 3xTF32 (the stage holds raw + lo tiles), 256 for one pass when N is wide
int tf_bn(int N, int npass) { return (npass == 1 && N > 128) ? 256 : 128; }

// CTA pairs (k_gemm_tf32_p) when the tile has more than 128 rows: FOLD_TF32_PAIR=0 keeps the
// single-CTA kernels (A/B switch)
bool tf_pair_enabled() {
  static const bool v = [] { const char *e = getenv("FOLD_TF32_PAIR"); return !(e && atoi(e) == 0); }();
  return v;
}
// Measured (C2 B=1024 / C3 / C6): pairs pay on large GEMMs in 3xTF32 (FP32 mode: forward
// 18.0 -> 14.7 ms, dA 14.7 -> 11.3, dU 16.3 -> 15.0) and on the MN-major TF32 passes (dA, dU),
// not on the one-pass K-major forward, nor at S = 300 (C3 / SST / C6: 128-column pair tiles
// measured 4-8% slower), so pairs run 256-column tiles where those pad N by little
int tf_pair_bn(int N) { return (N % 256 == 0 || N >= 2048) ? 256 : 128; }
bool tf_use_pair(int M, int N, int npass, bool any_mn) {
  return tf_pair_enabled() && M >= 2048 && tf_pair_bn(N) == 256 && (npass == 3 || any_mn);
}

int tf_splits_any(int M, int N, int K, int npass, bool pair) {
  const int BN = pair ? tf_pair_bn(N) : tf_bn(N, npass);
  const int64_t ctas = (pair ? 2 * cdiv(M, 2 * TM) : cdiv(M, TM)) * cdiv(N, BN);
  const int64_t kbs = cdiv(K, TK);
  int sp = 1;
  // fill about one wave of CTAs when the tile grid is small and the reduction long
  while (sp < 16 && ctas * sp * 2 <= sm_count() && kbs / (2 * sp) >= 16) sp *= 2;
  return sp;
}

int tf_splits_mn(int M, int N, int K, int npass, bool any_mn) {
  return tf_splits_any(M, N, K, npass, tf_use_pair(M, N, npass, any_mn));
}

template <int BN, int NPASS, bool PAIR = false>
fold_status launch_tf(const CUtensorMap &ma, const CUtensorMap &mb, const TfOperand &A, const TfOperand &B, int M,
                      int N, int K, float *C, int64_t ldc, int accumulate, int splits, float *split_ws,
                      cudaStream_t st) {
  auto kern = PAIR ? k_gemm_tf32_p<BN, NPASS> : k_gemm_tf32<BN, NPASS>;
  const int smem = PAIR ? TfPairCfg<BN, NPASS>::SMEM : TfCfg<BN, NPASS>::SMEM;
  FOLD_TRY(set_smem_tf(kern, smem));
  const int KBall = (int)cdiv(K, TK);
  const int kbps = (int)cdiv(KBall, splits);
  dim3 grid((unsigned)((PAIR ? 2 : 1) * cdiv(N, BN)), (unsigned)cdiv(M, PAIR ? 2 * TM : TM), (unsigned)splits);
  if (splits == 1) {
    kern<<<grid, TF_THREADS, smem, st>>>(ma, mb, A.mn_major, B.mn_major, M, N, K, kbps, C, ldc, 0, accumulate);
    FOLD_LAUNCH_CHECK();
    return FOLD_OK;
  }
  // partial slabs [splits][M][N] (dense, ld N), then the fixed-order sum into C
  if (ldc != N) return FOLD_E_INVALID;
  kern<<<grid, TF_THREADS, smem, st>>>(ma, mb, A.mn_major, B.mn_major, M, N, K, kbps, split_ws, N,
                                            (int64_t)M * N, 0);
  FOLD_LAUNCH_CHECK();
  return launch_reduce_splits((int64_t)M * N, splits, split_ws, C, accumulate, st);
}

// Grouped launch: every problem's tiles in one grid (BN = 128), per-problem split-K into
// partial slabs of split_ws (reduced per problem in fixed order, deterministic).
int tf_group_splits(const TfProblem &q, int npass, bool pair) {
  if (q.M <= 0 || q.N <= 0) return 1;
  return tf_splits_any(q.M, q.N, q.K, npass, pair);
}
// a group runs on CTA pairs when some problem has more than 128 rows (BN = 256 if some N
// exceeds 128), else on single-CTA 128 x 128 tiles
bool tf_group_pair(const TfProblem *q, int n, int npass, int &bn) {
  int mmax = 0, nmax = 0;
  bool mn = false;
  for (int i = 0; i < n; i++) {
    mmax = std::max(mmax, q[i].M); nmax = std::max(nmax, q[i].N);
    mn = mn || q[i].A.mn_major || q[i].B.mn_major;
  }
  bn = tf_pair_bn(nmax);
  return tf_use_pair(mmax, nmax, npass, mn);
}

template <int BN, int NPASS, bool PAIR>
fold_status launch_tf_grouped(TfGroupArgs &P, int zmax, cudaStream_t st) {
  auto kern = PAIR ? k_gemm_tf32_grouped_p<BN, NPASS> : k_gemm_tf32_grouped<BN, NPASS>;
  const int smem = PAIR ? TfPairCfg<BN, NPASS>::SMEM : TfCfg<BN, NPASS>::SMEM;
  FOLD_TRY(set_smem_tf(kern, smem));
  kern<<<dim3((unsigned)((PAIR ? 2 : 1) * P.tile_start[P.n]), 1, (unsigned)zmax), TF_THREADS, smem, st>>>(P);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

// ---------------------------------------------------------------- level helpers (FP32 / TF32 modes)
// Acat[c] = [H[gL] | H[gR]] (PAPER.md L47's gather, materialised for the GEMM's dense A
// operand and kept for the weight-gradient GEMM). One warp per (row, 128-column block).
__global__ void k_gather_cat(int r0, int r1, int nl, int S, int ld, const int32_t *__restrict__ gather,
                             const float *__restrict__ H, float *__restrict__ Acat, int64_t ld_a) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nblk = (int)cdiv(2 * S, 128);
  const int64_t ntask = (int64_t)(r1 - r0) * nblk;
  const bool vec = (S & 3) == 0;
  for (int64_t task = w; task < ntask; task += nw) {
    const int64_t r = r0 + task / nblk;
    const int jb = (int)(task % nblk) * 128;
    float *dst = Acat + (r - nl) * ld_a;
    if (vec) {
      const int j = jb + lane * 4;
      if (j < 2 * S) {
        const int half = j >= S;
        const int64_t src = gather[2 * r + half];
        *reinterpret_cast<float4 *>(dst + j) = *reinterpret_cast<const float4 *>(H + src * ld + (j - half * S));
      }
    } else {
      for (int u = 0; u < 4; u++) {
        const int j = jb + lane + 32 * u;
        if (j >= 2 * S) break;
        const int half = j >= S;
        dst[j] = H[gather[2 * r + half] * (int64_t)ld + (j - half * S)];
      }
    }
  }
}

// Cell forward pointwise step on the level's GEMM output (already in Gact, gate g of column
// j at g*ld + j): TreeLSTM gates (Tai et al. eqs 9-14 with x = 0, cited at PAPER.md
// L301-304), c = i u + fL cL + fR cR, h = o tanh(c); TreeRNN h = tanh(z + b) (Fig. 1 cell).
template <int GATES>
__global__ void k_cell_fwd_pw(int r0, int r1, int nl, int S, int ld, int ld_g, const int32_t *__restrict__ gather,
                              const float *__restrict__ b, float *__restrict__ H, float *__restrict__ C,
                              float *__restrict__ Gact) {
  const int64_t total = (int64_t)(r1 - r0) * S;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = r0 + i / S;
    const int j = (int)(i % S);
    const int64_t c = r - nl;
    float *ga = Gact + c * ld_g;
    if constexpr (GATES == 1) {
      const float h = tanhf(ga[j] + b[j]);
      ga[j] = h;
      H[r * ld + j] = h;
      C[r * ld + j] = 0.f;
    } else {
      const float ig = 1.f / (1.f + expf(-(ga[j] + b[j])));
      const float fl = 1.f / (1.f + expf(-(ga[ld + j] + b[S + j])));
      const float fr = 1.f / (1.f + expf(-(ga[2 * ld + j] + b[2 * S + j])));
      const float og = 1.f / (1.f + expf(-(ga[3 * ld + j] + b[3 * S + j])));
      const float ug = tanhf(ga[4 * ld + j] + b[4 * S + j]);
      // (rows below nl: the §3.5 leaf cell, no children: c_L = c_R = 0)
      const int64_t gl = gather[2 * r], gr = gather[2 * r + 1];
      const float cl = gl >= 0 ? C[gl * ld + j] : 0.f, cr = gr >= 0 ? C[gr * ld + j] : 0.f;
      const float cc = ig * ug + fl * cl + fr * cr;
      C[r * ld + j] = cc;
      H[r * ld + j] = og * tanhf(cc);
      ga[j] = ig; ga[ld + j] = fl; ga[2 * ld + j] = fr; ga[3 * ld + j] = og; ga[4 * ld + j] = ug;
    }
  }
}

// Ufwd[g*ld + j][k] = U[g*S + j][k] (0 for j >= S), Ubwd[i][k] = U[i][k]; k < 2S, rows padded to ld_u
__global__ void k_prep_U_tf(int gates, int S, int ld, int64_t ld_u, const float *__restrict__ U,
                            float *__restrict__ Ufwd, float *__restrict__ Ubwd) {
  const int64_t rows_f = (int64_t)gates * ld;
  const int64_t total = rows_f * ld_u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t row = i / ld_u, k = i % ld_u;
    const int g = (int)(row / ld), j = (int)(row % ld);
    const float v = (j < S && k < 2 * S) ? U[((int64_t)g * S + j) * 2 * S + k] : 0.f;
    if (Ufwd) Ufwd[i] = v;
    if (Ubwd && j < S) Ubwd[((int64_t)g * S + j) * ld_u + k] = v;
  }
}

}  // namespace

int64_t gemm_tf32_split_floats(int M, int N, int K) {
  int sp = 1;
  for (int np : {1, 3})
    for (bool pr : {false, true}) sp = std::max(sp, tf_splits_any(M, N, K, np, pr));
  return sp > 1 ? (int64_t)sp * M * N : 0;
}

fold_status gemm_tf32(const TfOperand &A, const TfOperand &B, int M, int N, int K, float *C, int64_t ldc,
                      int accumulate, int npass, float *split_ws, int64_t split_ws_floats, cudaStream_t st) {
  if (M <= 0 || N <= 0) return FOLD_OK;
  if (npass != 1 && npass != 3) return FOLD_E_INVALID;
  const int BN = tf_bn(N, npass);
  int splits = tf_splits_mn(M, N, K, npass, A.mn_major || B.mn_major);
  if (splits > 1 && (!split_ws || split_ws_floats < (int64_t)splits * M * N || ldc != N)) splits = 1;
  CUtensorMap ma, mb;
  FOLD_TRY(tf_map(&ma, A, M, K > 0 ? K : 1, TM));
  FOLD_TRY(tf_map(&mb, B, N, K > 0 ? K : 1, BN));
  if (tf_use_pair(M, N, npass, A.mn_major || B.mn_major)) {
    const int PBN = tf_pair_bn(N);
    CUtensorMap mbp;
    FOLD_TRY(tf_map(&mbp, B, N, K > 0 ? K : 1, PBN / 2));
    if (npass == 3)
      return PBN == 256 ? launch_tf<256, 3, true>(ma, mbp, A, B, M, N, K, C, ldc, accumulate, splits, split_ws, st)
                        : launch_tf<128, 3, true>(ma, mbp, A, B, M, N, K, C, ldc, accumulate, splits, split_ws, st);
    return PBN == 256 ? launch_tf<256, 1, true>(ma, mbp, A, B, M, N, K, C, ldc, accumulate, splits, split_ws, st)
                      : launch_tf<128, 1, true>(ma, mbp, A, B, M, N, K, C, ldc, accumulate, splits, split_ws, st);
  }
  if (npass == 3) return launch_tf<128, 3>(ma, mb, A, B, M, N, K, C, ldc, accumulate, splits, split_ws, st);
  if (BN == 256) return launch_tf<256, 1>(ma, mb, A, B, M, N, K, C, ldc, accumulate, splits, split_ws, st);
  return launch_tf<128, 1>(ma, mb, A, B, M, N, K, C, ldc, accumulate, splits, split_ws, st);
}

fold_status launch_gather_cat(int r0, int r1, int nl, int S, int ld, const int32_t *gather, const float *H,
                              float *Acat, int64_t ld_a, cudaStream_t st) {
  if (r1 <= r0) return FOLD_OK;
  const int64_t warps = (int64_t)(r1 - r0) * cdiv(2 * S, 128);
  int64_t blocks = cdiv(warps, 8);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_gather_cat<<<(unsigned)blocks, 256, 0, st>>>(r0, r1, nl, S, ld, gather, H, Acat, ld_a);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status launch_cell_fwd_pw(int cell, int r0, int r1, int nl, int S, int ld, int ld_g, const int32_t *gather,
                               const float *b, float *H, float *C, float *Gact, cudaStream_t st) {
  if (r1 <= r0) return FOLD_OK;
  int64_t blocks = cdiv((int64_t)(r1 - r0) * S, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (cell == FOLD_CELL_TREELSTM)
    k_cell_fwd_pw<5><<<(unsigned)blocks, 256, 0, st>>>(r0, r1, nl, S, ld, ld_g, gather, b, H, C, Gact);
  else
    k_cell_fwd_pw<1><<<(unsigned)blocks, 256, 0, st>>>(r0, r1, nl, S, ld, ld_g, gather, b, H, C, Gact);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

int64_t tf_ld_u(int S) { return round_up(2 * (int64_t)S, 4); }

fold_status launch_prep_U_tf(int gates, int S, int ld, const float *U, float *Ufwd, float *Ubwd, cudaStream_t st) {
  const int64_t total = (int64_t)gates * ld * tf_ld_u(S);
  int64_t blocks = cdiv(total, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_prep_U_tf<<<(unsigned)blocks, 256, 0, st>>>(gates, S, ld, tf_ld_u(S), U, Ufwd, Ubwd);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

int64_t gemm_tf32_grouped_ws_floats(const TfProblem *q, int n, int npass) {
  int64_t best = 0;
  for (bool pr : {false, true}) {
    int64_t tot = 0;
    for (int i = 0; i < n; i++) {
      const int sp = tf_group_splits(q[i], npass, pr);
      if (sp > 1) tot += (int64_t)sp * q[i].M * q[i].N;
    }
    best = std::max(best, tot);
  }
  return best;
}

fold_status gemm_tf32_grouped(const TfProblem *q, int n, int npass, float *split_ws, int64_t split_ws_floats,
                              cudaStream_t st) {
  if (npass != 1 && npass != 3) return FOLD_E_INVALID;
  if (n > kTfGroupMax) return FOLD_E_INVALID;
  TfGroupArgs P{};
  int pbn = 128;
  const bool pair = tf_group_pair(q, n, npass, pbn);
  const int BN = pair ? pbn : 128, TMt = pair ? 2 * TM : TM;
  int64_t ws_off = 0;
  int zmax = 1, tiles = 0;
  int red_n = 0, red_sp[kTfGroupMax] = {};
  float *red_part[kTfGroupMax] = {}, *red_out[kTfGroupMax] = {};
  int64_t red_cnt[kTfGroupMax] = {};
  int red_acc[kTfGroupMax] = {};
  for (int i = 0; i < n; i++) {
    const TfProblem &x = q[i];
    if (x.M <= 0 || x.N <= 0) continue;
    const int k = P.n;
    FOLD_TRY(tf_map(&P.ta[k], x.A, x.M, x.K > 0 ? x.K : 1, TM));
    FOLD_TRY(tf_map(&P.tb[k], x.B, x.N, x.K > 0 ? x.K : 1, pair ? BN / 2 : 128));
    P.a_mn[k] = x.A.mn_major; P.b_mn[k] = x.B.mn_major;
    P.M[k] = x.M; P.N[k] = x.N; P.K[k] = x.K;
    int sp = tf_group_splits(x, npass, pair);
    if (sp > 1 && (!split_ws || ws_off + (int64_t)sp * x.M * x.N > split_ws_floats || x.ldc != x.N)) sp = 1;
    const int KBall = (int)cdiv(x.K > 0 ? x.K : 1, TK);
    P.kbps[k] = (int)cdiv(KBall, sp);
    P.nsplit[k] = sp;
    if (sp > 1) {
      P.C[k] = split_ws + ws_off; P.ldc[k] = x.N; P.split_stride[k] = (int64_t)x.M * x.N; P.accumulate[k] = 0;
      red_part[red_n] = split_ws + ws_off; red_out[red_n] = x.C; red_cnt[red_n] = (int64_t)x.M * x.N;
      red_sp[red_n] = sp; red_acc[red_n] = x.accumulate; red_n++;
      ws_off += (int64_t)sp * x.M * x.N;
    } else {
      P.C[k] = x.C; P.ldc[k] = x.ldc; P.split_stride[k] = 0; P.accumulate[k] = x.accumulate;
    }
    P.ntn[k] = (int)cdiv(x.N, BN);
    P.tile_start[k] = tiles;
    tiles += (int)(cdiv(x.M, TMt) * P.ntn[k]);
    if (sp > zmax) zmax = sp;
    P.n++;
  }
  if (P.n == 0) return FOLD_OK;
  P.tile_start[P.n] = tiles;
  fold_status ls;
  if (!pair) ls = npass == 3 ? launch_tf_grouped<128, 3, false>(P, zmax, st) : launch_tf_grouped<128, 1, false>(P, zmax, st);
  else if (BN == 256) ls = npass == 3 ? launch_tf_grouped<256, 3, true>(P, zmax, st) : launch_tf_grouped<256, 1, true>(P, zmax, st);
  else ls = npass == 3 ? launch_tf_grouped<128, 3, true>(P, zmax, st) : launch_tf_grouped<128, 1, true>(P, zmax, st);
  FOLD_TRY(ls);
  for (int r = 0; r < red_n; r++)
    FOLD_TRY(launch_reduce_splits(red_cnt[r], red_sp[r], red_part[r], red_out[r], red_acc[r], st));
  return FOLD_OK;
}

}  // namespace fold

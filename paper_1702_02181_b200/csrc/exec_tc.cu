// exec_tc.cu — tcgen05 (5th-gen tensor core) kernels for the BF16 path.
//
//  k_cell_fwd_tc   one level of the forward (gather -> operation -> concat)
//                  in one kernel. The gather is moved to production time: whoever
//                  produces a pool row (embedding kernel, or this kernel's epilogue for
//                  the previous level) also writes it into the A-operand row of each
//                  consumer edge (planes A_L / A_R, row = consumer cell). So the level's
//                  A rows are contiguous and TMA streams them as dense 128B-swizzled boxes;
//                  tcgen05.mma multiplies them with a gate-interleaved slab of U into a
//                  TMEM accumulator; the epilogue warps apply the gates, append (h, c) to
//                  the level's pool rows (the concat becomes an append) and push h to its
//                  consumers' A rows.
//  k_gemm_dA_tc    backward edge gradients of one level: dA = dZ_level * U  (K-major).
//  k_gemm_dU_tc    weight gradient over all cells at once: dU = dZ^T * [A_L | A_R], both
//                  operands MN-major dense TMA boxes; split-K over cells with a
//                  fixed-order reduction (deterministic).
// Warp roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer (one lane),
// warp 2 TMEM allocator, warps 4-7 epilogue (warp w reads TMEM lanes 32(w%4)..+31).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "exec.cuh"
#include "ptx.cuh"

namespace fold {

namespace {

constexpr int BM = 128;     // rows per tile (UMMA M)
constexpr int BK = 64;      // K elements per stage (128 B of bf16 = one swizzle row)
constexpr int ST = 4;       // pipeline stages
constexpr int kThreads = 256;

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
  return (uint8_t *)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

constexpr int tmem_cols_for(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}

// =================================================================== forward cell level
template <int GATES, int W>
struct FwdCfg {
  static constexpr int N = GATES * W;
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = N * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int ACC_STRIDE = 256;  // TMEM columns per accumulator buffer (2 buffers)
  static constexpr int TMEM_COLS = 512;
  static constexpr int SMEM = ST * STAGE + 1024;
  static constexpr int EPI_WARPS = 8;     // 2 per SM sub-partition: each owns half the columns
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int CHUNKS = W / 8;
  static_assert(N % 16 == 0 && N <= 256, "UMMA N for M=128");
  static_assert(W % 8 == 0, "gate slab rows must fill 8-row swizzle atoms");
  static_assert(SMEM <= 227 * 1024, "smem");
};

// Persistent: grid = min(#tiles, #SMs); tile t -> (state-column tile t % NT, row tile t / NT)
// (N fast: the CTAs running concurrently share a few A tiles in L2; U is L2-resident).
// Two TMEM accumulators: the epilogue of tile i overlaps the MMA main loop of tile i+1.
// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4..11 epilogue
// (warp w reads TMEM lanes 32 (w % 4) .. +31, column chunks (w - 4) / 4, +2, +4, ...).
template <int GATES, int W>
__global__ void __launch_bounds__(FwdCfg<GATES, W>::THREADS, 1)
    k_cell_fwd_tc(const __grid_constant__ CUtensorMap tmAL, const __grid_constant__ CUtensorMap tmAR,
                  const __grid_constant__ CUtensorMap tmU, int r0, int r1, int nl, int S, int Sp, int ld, int KBh,
                  int NT, int ntiles, const int32_t *__restrict__ gather, const float *__restrict__ bias,
                  __nv_bfloat16 *__restrict__ H, float *__restrict__ C, __nv_bfloat16 *__restrict__ Gact, int ld_g,
                  ScatterA sc, int dbg_epi, int bias_in_smem) {
  using Cfg = FwdCfg<GATES, W>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], Cfg::EPI_WARPS); }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmAL);
    ptx::prefetch_tmap(&tmAR);
    ptx::prefetch_tmap(&tmU);
  }
  if (warp == 2) {
    ptx::tmem_alloc(&tmem_base_sh, Cfg::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  // the whole bias (GATES*S fp32) stays in shared memory when it fits next to the ring
  float *sbias = reinterpret_cast<float *>(smem + ST * Cfg::STAGE);
  if (bias_in_smem)
    for (int i = tid; i < GATES * S; i += blockDim.x) sbias[i] = bias[i];
  const float *bsrc = bias_in_smem ? sbias : bias;
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  const int KB = 2 * KBh;

  if (warp == 0) {
    // TMA producer: per stage one dense box of 128 A rows (the level's contiguous cell rows
    // of the left / right operand plane) + one box of the gate-interleaved U slab.
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int c0 = (r0 - nl) + (t / NT) * BM;
        for (int kb = 0; kb < KB; kb++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full[s], Cfg::STAGE);
          int half = kb >= KBh;
          int kc = (kb - half * KBh) * BK;
          uint8_t *A = smem + s * Cfg::STAGE;
          ptx::tma_load_2d(half ? &tmAR : &tmAL, &full[s], A, kc, c0);
          // U is stored gate-interleaved per state-column tile (tc_prepare_U): one box of
          // GATES*W rows holds (i, fL, fR, o, u) for the tile's W state columns
          ptx::tma_load_2d(&tmU, &full[s], A + Cfg::A_BYTES, half * Sp + kc, (t % NT) * Cfg::N);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(BM, Cfg::N, 0, 0);
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
        const int acc = tc & 1;
        const uint32_t aph = (tc >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], aph ^ 1);
        ptx::tc_fence_after();
        const uint32_t dst = tbase + acc * Cfg::ACC_STRIDE;
        for (int kb = 0; kb < KB; kb++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&full[s], ph);
          ptx::tc_fence_after();
          uint32_t a0 = ptx::smem_u32(smem + s * Cfg::STAGE), b0 = a0 + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; k++)
            ptx::umma_bf16(dst, ptx::sdesc_sw128(a0 + 32 * k, 16, 1024), ptx::sdesc_sw128(b0 + 32 * k, 16, 1024),
                           idesc, (kb | k) != 0);
          ptx::umma_commit(&empty[s]);
        }
        ptx::umma_commit(&tfull[acc]);
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
    auto fetch_meta = [&](int t, Meta &m) {
      const int64_t rr = r0 + (int64_t)(t / NT) * BM + row;
      m.gl = m.gr = m.ce0 = m.ce1 = 0; m.e0 = 0;
      if (t < ntiles && rr < r1) {
        m.gl = gather[2 * rr]; m.gr = gather[2 * rr + 1];
        m.ce0 = sc.cons_off[rr]; m.ce1 = sc.cons_off[rr + 1];
        if (m.ce1 > m.ce0) m.e0 = sc.cons_edge[m.ce0];
      }
    };
    Meta nxt;
    fetch_meta(blockIdx.x, nxt);
    int tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
      const int acc = tc & 1;
      const uint32_t aph = (tc >> 1) & 1;
      const int j0 = (t % NT) * W;
      const int64_t r = r0 + (int64_t)(t / NT) * BM + row;
      const bool valid = r < r1 && dbg_epi != 1;
      const Meta cur = nxt;
      fetch_meta(t + gridDim.x, nxt);
      const int64_t gl = cur.gl, gr = cur.gr;
      const int ce0 = cur.ce0, ce1 = cur.ce1;
      const int64_t c = r - nl;
      // prefetch the first chunk's child cell states before waiting for the accumulator
      float cl[8], cr[8];
      auto load_c = [&](int jb) {
        if (GATES != 5) return;
        // leaf children have c = 0 (their C rows are not materialised in BF16 mode)
        const bool lok = valid && gl >= nl, rok = valid && gr >= nl;
        if (jb + 8 <= S && (S & 7) == 0) {
#pragma unroll
          for (int u = 0; u < 8; u++) { cl[u] = 0.f; cr[u] = 0.f; }
          if (lok) {
            float4 a = __ldg(reinterpret_cast<const float4 *>(C + gl * ld + jb));
            float4 b = __ldg(reinterpret_cast<const float4 *>(C + gl * ld + jb + 4));
            cl[0] = a.x; cl[1] = a.y; cl[2] = a.z; cl[3] = a.w; cl[4] = b.x; cl[5] = b.y; cl[6] = b.z; cl[7] = b.w;
          }
          if (rok) {
            float4 a = __ldg(reinterpret_cast<const float4 *>(C + gr * ld + jb));
            float4 b = __ldg(reinterpret_cast<const float4 *>(C + gr * ld + jb + 4));
            cr[0] = a.x; cr[1] = a.y; cr[2] = a.z; cr[3] = a.w; cr[4] = b.x; cr[5] = b.y; cr[6] = b.z; cr[7] = b.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; u++) {
            cl[u] = (lok && jb + u < S) ? C[gl * ld + jb + u] : 0.f;
            cr[u] = (rok && jb + u < S) ? C[gr * ld + jb + u] : 0.f;
          }
        }
      };
      load_c(j0 + grp * 8);
      ptx::mbar_wait(&tfull[acc], aph);
      ptx::tc_fence_after();
      const uint32_t tl = tbase + acc * Cfg::ACC_STRIDE + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int jc = grp; jc < Cfg::CHUNKS; jc += 2) {
        float z[GATES][8];
#pragma unroll
        for (int g = 0; g < GATES; g++) ptx::tmem_ld8(tl + g * W + jc * 8, z[g]);
        ptx::tmem_ld_wait();
        const int jb = j0 + jc * 8;
        float ccl[8], ccr[8];
#pragma unroll
        for (int u = 0; u < 8; u++) { ccl[u] = cl[u]; ccr[u] = cr[u]; }
        if (jc + 2 < Cfg::CHUNKS) load_c(jb + 16);  // next chunk of this warp, in flight during math
        if (!valid || jb >= S) continue;
        const bool fullc = (jb + 8 <= S) && ((S & 7) == 0);
        float hh[8];
        if constexpr (GATES == 1) {
#pragma unroll
          for (int u = 0; u < 8; u++) hh[u] = tanh_fast(z[0][u] + (jb + u < S ? bsrc[jb + u] : 0.f));
          if (fullc) {
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
#pragma unroll
          for (int g = 0; g < 5; g++) {
            float bz[8];
            if (fullc) {
              float4 x = *reinterpret_cast<const float4 *>(bsrc + g * S + jb);
              float4 y = *reinterpret_cast<const float4 *>(bsrc + g * S + jb + 4);
              bz[0] = x.x; bz[1] = x.y; bz[2] = x.z; bz[3] = x.w; bz[4] = y.x; bz[5] = y.y; bz[6] = y.z; bz[7] = y.w;
            } else {
#pragma unroll
              for (int u = 0; u < 8; u++) bz[u] = jb + u < S ? bsrc[g * S + jb + u] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; u++) gs[g][u] = g == 4 ? tanh_fast(z[g][u] + bz[u]) : sigmoid_fast(z[g][u] + bz[u]);
          }
#pragma unroll
          for (int u = 0; u < 8; u++) {
            cc[u] = gs[0][u] * gs[4][u] + gs[1][u] * ccl[u] + gs[2][u] * ccr[u];
            hh[u] = gs[3][u] * tanh_fast(cc[u]);
          }
          __nv_bfloat16 *ga = Gact + c * ld_g;
          if (dbg_epi == 2) {  // probe: no stores at all (keep the math alive)
            float acc = 0.f;
#pragma unroll
            for (int u = 0; u < 8; u++) acc += cc[u] + hh[u] + gs[0][u] + gs[1][u] + gs[2][u] + gs[3][u] + gs[4][u];
            if (acc == 12345.f) C[r * ld + jb] = acc;
            continue;
          }
          if (fullc) {
            *reinterpret_cast<float4 *>(C + r * ld + jb) = make_float4(cc[0], cc[1], cc[2], cc[3]);
            *reinterpret_cast<float4 *>(C + r * ld + jb + 4) = make_float4(cc[4], cc[5], cc[6], cc[7]);
#pragma unroll
            for (int g = 0; g < 5; g++)
              if (dbg_epi != 3)
              *reinterpret_cast<uint4 *>(ga + g * S + jb) =
                  make_uint4(pack_bf16x2(gs[g][0], gs[g][1]), pack_bf16x2(gs[g][2], gs[g][3]),
                             pack_bf16x2(gs[g][4], gs[g][5]), pack_bf16x2(gs[g][6], gs[g][7]));
          } else {
            for (int u = 0; u < 8 && jb + u < S; u++) {
              int j = jb + u;
              C[r * ld + j] = cc[u];
#pragma unroll
              for (int g = 0; g < 5; g++) ga[g * S + j] = __float2bfloat16_rn(gs[g][u]);
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
            int ed = e == ce0 ? cur.e0 : sc.cons_edge[e];
            *reinterpret_cast<uint4 *>(((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld + jb) = pk;
          }
        } else {
          for (int u = 0; u < 8 && jb + u < S; u++) {
            __nv_bfloat16 hv = __float2bfloat16_rn(hh[u]);
            if (ce1 == ce0) H[r * ld + jb + u] = hv;
            for (int e = ce0; e < ce1; e++) {
              int ed = sc.cons_edge[e];
              (((ed & 1) ? sc.AR : sc.AL) + (int64_t)(ed >> 1) * sc.ld)[jb + u] = hv;
            }
          }
        }
      }
      // this accumulator buffer may be overwritten by the MMA of tile i+2
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, Cfg::TMEM_COLS);
  }
}

// =================================================================== dA = dZ * U (one level)
// Persistent (grid = min(#tiles, #SMs)), tile t -> (N tile t % NTn, row tile t / NTn),
// 128 x 256 tiles, two TMEM accumulators so the fp32 store epilogue of tile i overlaps the
// main loop of tile i+1.
constexpr int DA_N = 256;
constexpr int DA_A_BYTES = BM * 128, DA_B_BYTES = DA_N * 128, DA_STAGE = DA_A_BYTES + DA_B_BYTES;
constexpr int DA_SMEM = ST * DA_STAGE + 1024;

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_dA_tc(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmUt, int c0, int M,
                 int KB, int S, int NTn, int ntiles, float *__restrict__ dA) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t full[ST], empty[ST], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { ptx::mbar_init(&tfull[a], 1); ptx::mbar_init(&tempty[a], 4); }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmZ);
    ptx::prefetch_tmap(&tmUt);
  }
  if (warp == 2) { ptx::tmem_alloc(&tmem_base_sh, 512); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int mt = c0 + (t / NTn) * BM, n0 = (t % NTn) * DA_N;
        for (int kb = 0; kb < KB; kb++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full[s], DA_STAGE);
          uint8_t *A = smem + s * DA_STAGE;
          ptx::tma_load_2d(&tmZ, &full[s], A, kb * BK, mt);
          ptx::tma_load_2d(&tmUt, &full[s], A + DA_A_BYTES, kb * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(BM, DA_N, 0, 0);
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
        const int acc = tc & 1;
        ptx::mbar_wait(&tempty[acc], ((tc >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t dst = tbase + acc * 256;
        for (int kb = 0; kb < KB; kb++, it++) {
          int s = it % ST;
          uint32_t ph = (it / ST) & 1;
          ptx::mbar_wait(&full[s], ph);
          ptx::tc_fence_after();
          uint32_t a0 = ptx::smem_u32(smem + s * DA_STAGE), b0 = a0 + DA_A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; k++)
            ptx::umma_bf16(dst, ptx::sdesc_sw128(a0 + 32 * k, 16, 1024), ptx::sdesc_sw128(b0 + 32 * k, 16, 1024),
                           idesc, (kb | k) != 0);
          ptx::umma_commit(&empty[s]);
        }
        ptx::umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int N2 = 2 * S;
    int tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
      const int acc = tc & 1;
      const int mt = c0 + (t / NTn) * BM, n0 = (t % NTn) * DA_N;
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
        int n = n0 + nc * 8;
        if (!valid || n >= N2) continue;
        if (n + 8 <= N2 && (N2 & 3) == 0) {
          *reinterpret_cast<float4 *>(out + n) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4 *>(out + n + 4) = make_float4(v[4], v[5], v[6], v[7]);
        } else {
          for (int u = 0; u < 8 && n + u < N2; u++) out[n + u] = v[u];
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 512); }
}

// =================================================================== dU = dZ^T * Acat (all cells)
constexpr int DU_N = 256;
constexpr int DU_A_BYTES = BM * 128;     // 2 MN chunks x 64 K-rows x 128 B
constexpr int DU_B_BYTES = DU_N * 128;   // 4 MN chunks x 64 K-rows x 128 B
constexpr int DU_STAGE = DU_A_BYTES + DU_B_BYTES;
constexpr int DU_SMEM = ST * DU_STAGE + 1024;
constexpr int MN_CHUNK = 64 * 128;       // bytes per 64-element MN chunk of 64 K rows

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_dU_tc(const __grid_constant__ CUtensorMap tmZ2, const __grid_constant__ CUtensorMap tmAL,
                 const __grid_constant__ CUtensorMap tmAR, int n_cells, int S, int Mg, int NT, int kb_per_split,
                 float *__restrict__ out_base, int64_t split_stride, int accumulate) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t full[ST], empty[ST], tfull;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = blockIdx.x / NT, jt = blockIdx.x - half * NT;
  const int i0 = blockIdx.y * BM, jn0 = jt * DU_N;
  // split-K over cells: this CTA reduces k-blocks [kb0, kb1) into its own partial slab
  const int KBall = (int)cdiv(n_cells, BK);
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(KBall, kb0 + kb_per_split);
  const int KB = kb1 > kb0 ? kb1 - kb0 : 0;
  float *dU = out_base + (int64_t)blockIdx.z * split_stride;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::mbar_init(&tfull, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmZ2);
    ptx::prefetch_tmap(&tmAL);
    ptx::prefetch_tmap(&tmAR);
  }
  if (warp == 2) { ptx::tmem_alloc(&tmem_base_sh, 256); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
  if (warp == 0 && lane == 0) {
    // A' = dZ^T chunk (2 boxes of 64 gate-rows x 64 cells), B' = the cells' [h_L | h_R]
    // rows from the A operand planes written by the forward (4 boxes of 64 cols x 64 cells)
    const CUtensorMap *tmB = half ? &tmAR : &tmAL;
    for (int it = 0; it < KB; it++) {
      const int kb = kb0 + it;
      int s = it % ST;
      uint32_t ph = (it / ST) & 1;
      ptx::mbar_wait(&empty[s], ph ^ 1);
      ptx::mbar_arrive_expect_tx(&full[s], DU_STAGE);
      uint8_t *A = smem + s * DU_STAGE;
      uint8_t *B = A + DU_A_BYTES;
      ptx::tma_load_2d(&tmZ2, &full[s], A, i0, kb * BK);
      ptx::tma_load_2d(&tmZ2, &full[s], A + MN_CHUNK, i0 + 64, kb * BK);
#pragma unroll
      for (int ch = 0; ch < 4; ch++) ptx::tma_load_2d(tmB, &full[s], B + ch * MN_CHUNK, jn0 + ch * 64, kb * BK);
    }
  } else if (warp == 0) {
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(BM, DU_N, 1, 1);
      for (int it = 0; it < KB; it++) {
        int s = it % ST;
        uint32_t ph = (it / ST) & 1;
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        uint32_t a0 = ptx::smem_u32(smem + s * DU_STAGE), b0 = a0 + DU_A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; k++)
          ptx::umma_bf16(tbase, ptx::sdesc_sw128(a0 + 2048 * k, MN_CHUNK, 1024),
                         ptx::sdesc_sw128(b0 + 2048 * k, MN_CHUNK, 1024), idesc, (it | k) != 0);
        ptx::umma_commit(&empty[s]);
      }
      ptx::umma_commit(&tfull);
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    ptx::mbar_wait(&tfull, 0);
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
  __syncthreads();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 256); }
}

// out[i] = (accumulate ? out[i] : 0) + sum_{s < nsplit} part[s][i]   (fixed order)
__global__ void k_reduce_splits(int64_t n, int nsplit, const float *__restrict__ part, float *__restrict__ out,
                                int accumulate) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i4 < n; i4 += stride * 4) {
    if (i4 + 4 <= n) {
      float4 acc = accumulate ? *reinterpret_cast<const float4 *>(out + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < nsplit; s++) {
        float4 v = *reinterpret_cast<const float4 *>(part + (int64_t)s * n + i4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      *reinterpret_cast<float4 *>(out + i4) = acc;
    } else {
      for (int64_t i = i4; i < n; i++) {
        float acc = accumulate ? out[i] : 0.f;
        for (int s = 0; s < nsplit; s++) acc += part[(int64_t)s * n + i];
        out[i] = acc;
      }
    }
  }
}

// =================================================================== weight prep
// Forward operand: Uil[t*GW + g*W + jj][half*Sp + k] = bf16(U[g*S + t*W + jj][half*S + k])
// (gate-interleaved per W-column tile; K halves padded to Sp = round_up(S, 64) so every TMA
// box starts 128-byte aligned; rows / columns past S are zero).
__global__ void k_prep_Uil(int gates, int W, int NT, int S, int Sp, const float *__restrict__ U,
                           __nv_bfloat16 *__restrict__ Uil, int ld_u) {
  const int GW = gates * W;
  const int64_t total = (int64_t)NT * GW * (2 * Sp);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t ri = i / (2 * Sp);
    const int kp = (int)(i - ri * 2 * Sp);
    const int t = (int)(ri / GW), rem = (int)(ri - (int64_t)t * GW), g = rem / W, j = t * W + (rem - g * W);
    const int half = kp >= Sp, kk = kp - half * Sp;
    float v = (j < S && kk < S) ? U[((int64_t)g * S + j) * 2 * S + half * S + kk] : 0.f;
    Uil[ri * ld_u + kp] = __float2bfloat16_rn(v);
  }
}

// Backward operand: Ut[k][r] = bf16(U[r][k]) (ld_ut), 32x32 smem tiles.
__global__ void k_prep_Ut(int R, int K, const float *__restrict__ U, __nv_bfloat16 *__restrict__ Ut, int ld_ut) {
  __shared__ float t[32][33];
  const int r0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    int r = r0 + i, k = k0 + tx;
    t[i][tx] = (r < R && k < K) ? U[(int64_t)r * K + k] : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    int k = k0 + i, r = r0 + tx;
    if (r < R && k < K) Ut[(int64_t)k * ld_ut + r] = __float2bfloat16_rn(t[tx][i]);
  }
}

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

// 2D bf16 tensor map: `cols` contiguous elements per row, `rows` rows, `row_bytes` stride.
fold_status make_map(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows, uint64_t row_bytes,
                     uint32_t box_cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return FOLD_E_CUDA;
  if (rows < 1) rows = 1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FOLD_OK : FOLD_E_CUDA;
}

template <typename K>
fold_status set_smem(K kernel, int bytes) {
  FOLD_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return FOLD_OK;
}

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

int dbg_fwd_epi() {
  static int v = [] { const char *e = getenv("FOLD_DBG_FWD_EPI"); return e ? atoi(e) : 0; }();
  return v;
}

template <int GATES, int W>
fold_status launch_fwd(int r0, int r1, int nl, int n_cells, const int32_t *gather, int S, int ld, const TcWeights &w,
                       const float *b, __nv_bfloat16 *H, float *C, __nv_bfloat16 *Gact, int ld_g, const ScatterA &sc,
                       cudaStream_t st) {
  using Cfg = FwdCfg<GATES, W>;
  CUtensorMap tmAL, tmAR, tmU;
  FOLD_TRY(make_map(&tmAL, sc.AL, (uint64_t)S, (uint64_t)n_cells, (uint64_t)sc.ld * 2, BK, BM));
  FOLD_TRY(make_map(&tmAR, sc.AR, (uint64_t)S, (uint64_t)n_cells, (uint64_t)sc.ld * 2, BK, BM));
  const int NTu = (int)cdiv(S, W);
  FOLD_TRY(make_map(&tmU, w.U, (uint64_t)w.ld_u, (uint64_t)NTu * Cfg::N, (uint64_t)w.ld_u * 2, BK, Cfg::N));
  auto kern = k_cell_fwd_tc<GATES, W>;
  const int bias_bytes = GATES * S * 4;
  const int bias_in_smem = Cfg::SMEM + bias_bytes <= 227 * 1024 ? 1 : 0;
  const int smem_bytes = Cfg::SMEM + (bias_in_smem ? bias_bytes : 0);
  FOLD_TRY(set_smem(kern, smem_bytes));
  const int NT = (int)cdiv(S, W);
  const int ntiles = NT * (int)cdiv(r1 - r0, BM);
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  int KBh = (int)cdiv(S, BK);
  kern<<<grid, Cfg::THREADS, smem_bytes, st>>>(tmAL, tmAR, tmU, r0, r1, nl, S, w.ld_u / 2, ld, KBh, NT, ntiles,
                                               gather, b, H, C, Gact, ld_g, sc, dbg_fwd_epi(), bias_in_smem);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

}  // namespace

int tc_fwd_W(int gates) { return gates == 5 ? 48 : 128; }

size_t tc_workspace_bytes(int gates, int S) {
  const int W = tc_fwd_W(gates);
  size_t ld_u = 2 * round_up(S, 64), ld_ut = round_up((int64_t)gates * S, 8);
  size_t rows_il = (size_t)cdiv(S, W) * gates * W;
  return round_up((int64_t)(rows_il * ld_u * 2), 256) + round_up((int64_t)2 * S * ld_ut * 2, 256);
}

size_t tc_ut_offset(int gates, int S) {
  const int W = tc_fwd_W(gates);
  size_t ld_u = 2 * round_up(S, 64);
  size_t rows_il = (size_t)cdiv(S, W) * gates * W;
  return round_up((int64_t)(rows_il * ld_u * 2), 256);
}

fold_status tc_prepare_U(int gates, int S, const float *U, TcWeights &w, bool transpose, cudaStream_t st) {
  if (!transpose) {
    const int W = tc_fwd_W(gates), NT = (int)cdiv(S, W), Sp = (int)round_up(S, 64);
    int64_t total = (int64_t)NT * gates * W * 2 * Sp;
    int64_t blocks = cdiv(total, 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_prep_Uil<<<(unsigned)blocks, 256, 0, st>>>(gates, W, NT, S, Sp, U, w.U, w.ld_u);
  } else {
    const int R = gates * S, K = 2 * S;
    dim3 grid((unsigned)cdiv(K, 32), (unsigned)cdiv(R, 32));
    k_prep_Ut<<<grid, 256, 0, st>>>(R, K, U, w.Ut, w.ld_ut);
  }
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

fold_status tc_cell_fwd(int cell, int r0, int r1, int nl, int n_cells, const int32_t *gather, int S, int ld,
                        const TcWeights &w, const float *b, __nv_bfloat16 *H, float *C, __nv_bfloat16 *Gact, int ld_g,
                        const ScatterA &sc, cudaStream_t st) {
  if (r1 <= r0) return FOLD_OK;
  if (cell == FOLD_CELL_TREELSTM)
    return launch_fwd<5, 48>(r0, r1, nl, n_cells, gather, S, ld, w, b, H, C, Gact, ld_g, sc, st);
  return launch_fwd<1, 128>(r0, r1, nl, n_cells, gather, S, ld, w, b, H, C, Gact, ld_g, sc, st);
}

fold_status tc_gemm_dA(int c0, int M, int n_cells, int S, int gates, const __nv_bfloat16 *dZ, int ld_z,
                       const TcWeights &w, float *dA, cudaStream_t st) {
  if (M <= 0) return FOLD_OK;
  CUtensorMap tmZ, tmUt;
  FOLD_TRY(make_map(&tmZ, dZ, (uint64_t)gates * S, (uint64_t)n_cells, (uint64_t)ld_z * 2, BK, BM));
  FOLD_TRY(make_map(&tmUt, w.Ut, (uint64_t)gates * S, (uint64_t)2 * S, (uint64_t)w.ld_ut * 2, BK, DA_N));
  FOLD_TRY(set_smem(k_gemm_dA_tc, DA_SMEM));
  const int NTn = (int)cdiv(2 * S, DA_N);
  const int ntiles = NTn * (int)cdiv(M, BM);
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  int KB = (int)cdiv(gates * S, BK);
  k_gemm_dA_tc<<<grid, kThreads, DA_SMEM, st>>>(tmZ, tmUt, c0, M, KB, S, NTn, ntiles, dA);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

int tc_dU_splits(int n_cells, int gates, int S) {
  int64_t tiles = 2 * cdiv(S, DU_N) * cdiv((int64_t)gates * S, BM);
  int64_t kbs = cdiv(n_cells, BK);
  int64_t want = cdiv(4 * 148, tiles);           // >= ~4 waves of CTAs in total
  int64_t cap = kbs / 32;                         // keep >= 32 k-blocks (2048 cells) per split
  int64_t sp = want < cap ? want : cap;
  if (sp > 16) sp = 16;
  return sp < 1 ? 1 : (int)sp;
}

fold_status tc_gemm_dU(int n_cells, int S, int gates, const __nv_bfloat16 *dZ, int ld_z, const ScatterA &sc,
                       float *dU, int accumulate, float *split_ws, cudaStream_t st) {
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
  dim3 grid((unsigned)(2 * NT), (unsigned)cdiv(gates * S, BM), (unsigned)splits);
  const int64_t n = (int64_t)gates * S * 2 * S;
  if (splits == 1) {
    k_gemm_dU_tc<<<grid, kThreads, DU_SMEM, st>>>(tmZ2, tmAL, tmAR, n_cells, S, gates * S, NT, kbps, dU, 0,
                                                  accumulate);
    FOLD_LAUNCH_CHECK();
    return FOLD_OK;
  }
  if (!split_ws) return FOLD_E_WORKSPACE;
  k_gemm_dU_tc<<<grid, kThreads, DU_SMEM, st>>>(tmZ2, tmAL, tmAR, n_cells, S, gates * S, NT, kbps, split_ws, n, 0);
  FOLD_LAUNCH_CHECK();
  int64_t blocks = cdiv(cdiv(n, 4), 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_reduce_splits<<<(unsigned)blocks, 256, 0, st>>>(n, splits, split_ws, dU, accumulate);
  FOLD_LAUNCH_CHECK();
  return FOLD_OK;
}

}  // namespace fold

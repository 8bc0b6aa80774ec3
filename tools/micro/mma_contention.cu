// What slows a CTA-pair tcgen05 mainloop when an epilogue runs beside it? (the
// wide GEMMs run their MMAs at ~65% of the clock-adjusted peak while their epilogues move
// data, ~89% without; k_gemm_dU_tc, no epilogue traffic, 89%.) One cluster of 2 CTAs per
// TPC; the leader issues M=256, N=256, K=16 bf16 MMAs (cta_group::2) from fixed shared-
// memory operands (4 per 64-deep k-block, one commit per k-block, at most 4 k-blocks in
// flight, like the kernels' ring) while other warps of both CTAs generate one kind of side
// traffic until the MMAs finish:
//   0 none | 1 TMA loads (L2-resident source) into a 4 x 32 KB ring | 2 LDS+STS (8 warps)
//   3 LDG.128 (8 warps, L2-resident) | 4 STG.128 (8 warps) | 5 LDG + STG | 6 TMA + LDG
// Prints the MMA rate as a fraction of 128 cycles per MMA and the side traffic in B/clk/SM.
// Standalone tool (not part of libfold):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1702_02181_b200/csrc \
//        tools/micro/mma_contention.cu -o /tmp/mma_contention -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace fold;

constexpr int OPND = 2 * 32768;   // two k-blocks of A (16 KB) + B half (16 KB)
constexpr int RING = 4 * 32768;   // TMA side-traffic ring
constexpr int SCR = 32768;        // LDS/STS scratch
constexpr int SMEM = OPND + RING + SCR + 1024;
constexpr int ROWS = 16384, COLS = 1024;  // 32 MB bf16 TMA source
constexpr int64_t GBUF = 8 << 20;          // floats per LDG/STG buffer (32 MB)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_probe(const __grid_constant__ CUtensorMap tm, int mode, int kblocks, const float4 *gsrc, float4 *gdst,
            unsigned long long *out) {
  extern __shared__ uint8_t raw[];
  uint8_t *smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  uint8_t *ring = smem + OPND, *scr = smem + OPND + RING;
  __shared__ __align__(8) uint64_t mdone[4], rfull[4];
  __shared__ uint32_t tbase_sh;
  __shared__ volatile int stop;
  __shared__ unsigned long long side_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; i++) { ptx::mbar_init(&mdone[i], 1); ptx::mbar_init(&rfull[i], 1); }
    ptx::fence_mbar_init();
    stop = 0;
    side_bytes = 0;
  }
  if (warp == 2) { ptx::tmem_alloc2(&tbase_sh, 512); ptx::tmem_relinquish2(); }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = tbase_sh;
  unsigned long long my_bytes = 0;
  if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // mode 7: B MN-major (k_bwd_levels' U operand), mode 8: A and B MN-major (k_gemm_dU_tc)
      const int amn = mode == 8, bmn = mode >= 7;
      const uint32_t idesc = ptx::idesc_bf16(256, 256, amn, bmn);
      const unsigned long long c0 = clock64();
      for (int kb = 0; kb < kblocks; kb++) {
        const int s = kb & 3;
        if (kb >= 4) ptx::mbar_wait(&mdone[s], ((kb >> 2) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(smem + (kb & 1) * 32768), b0 = a0 + 16384;
#pragma unroll
        for (int k = 0; k < 4; k++)
          ptx::umma_bf16_2cta(tbase + (kb & 1) * 256,
                              amn ? ptx::sdesc_sw128(a0 + 2048 * k, 8192, 1024) : ptx::sdesc_sw128(a0 + 32 * k, 16, 1024),
                              bmn ? ptx::sdesc_sw128(b0 + 2048 * k, 8192, 1024) : ptx::sdesc_sw128(b0 + 32 * k, 16, 1024),
                              idesc, 1);
        ptx::umma_commit_2cta(&mdone[s]);
      }
      for (int kb = kblocks - 4; kb < kblocks; kb++) ptx::mbar_wait(&mdone[kb & 3], (kb >> 2) & 1);
      const unsigned long long c1 = clock64();
      out[blockIdx.x >> 1] = c1 - c0;
      // stop the side traffic in both CTAs
      stop = 1;
      const uint32_t peer = ptx::smem_u32((const void *)&stop);
      uint32_t pa;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(pa) : "r"(peer));
      asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(pa), "r"(1) : "memory");
    }
  } else if (warp == 0 && (mode == 1 || mode == 6)) {
    if (lane == 0) {
      uint32_t seed = blockIdx.x * 2654435761u + 7u;
      for (int it = 0;; it++) {
        const int s = it & 3;
        if (it >= 4) { ptx::mbar_wait(&rfull[s], ((it >> 2) - 1) & 1); my_bytes += 32768; }
        if (stop) {
          for (int j = it - (it >= 4 ? 3 : it); j < it; j++) ptx::mbar_wait(&rfull[j & 3], (j >> 2) & 1);
          break;
        }
        ptx::mbar_arrive_expect_tx(&rfull[s], 32768);
        seed = seed * 1664525u + 1013904223u;
        const int rb = (int)((seed >> 8) % (ROWS / 256)), cb = (int)((seed >> 20) % (COLS / 64));
        ptx::tma_load_2d(&tm, &rfull[s], ring + s * 32768, cb * 64, rb * 256);
      }
    }
  } else if (warp >= 4) {
    const int t = threadIdx.x - 128;  // 0..255
    if (mode == 2) {
      const uint32_t base = ptx::smem_u32(scr);
      uint32_t x = 0;
      while (!stop) {
#pragma unroll 4
        for (int i = 0; i < 8; i++) {
          const uint32_t off = ((t + i * 256) * 16) & (SCR - 1);
          uint4 v = ptx::lds128(base + off);
          x ^= v.x;
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + (off ^ 4096)), "r"(v.x), "r"(v.y + x), "r"(v.z),
                       "r"(v.w)
                       : "memory");
        }
        my_bytes += 8 * 32;
      }
      if (x == 0x12345678u) out[1000] = x;
    } else if (mode == 3 || mode == 5 || mode == 6) {
      float acc = 0.f;
      int64_t i = ((int64_t)blockIdx.x * 256 + t) * 8;
      const int64_t n4 = GBUF / 4;
      while (!stop) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = __ldcg(gsrc + ((i + u * 37 * 256) % n4));
#pragma unroll
        for (int u = 0; u < 8; u++) acc += v[u].x + v[u].w;
        if (mode == 5) {
#pragma unroll
          for (int u = 0; u < 4; u++) gdst[(i + u * 256 + 7) % n4] = v[u];
          my_bytes += 4 * 16;
        }
        i = (i + 148 * 256 * 8) % n4;
        my_bytes += 8 * 16;
      }
      if (acc == 1234.5f) out[1000] = 1;
    } else if (mode == 4) {
      int64_t i = ((int64_t)blockIdx.x * 256 + t) * 8;
      const int64_t n4 = GBUF / 4;
      const float4 v = make_float4(1.f, 2.f, 3.f, (float)t);
      while (!stop) {
#pragma unroll
        for (int u = 0; u < 8; u++) gdst[(i + u * 256) % n4] = v;
        i = (i + 148 * 256 * 8) % n4;
        my_bytes += 8 * 16;
      }
    }
  }
  if (my_bytes) atomicAdd(&side_bytes, my_bytes);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  __syncthreads();
  if (threadIdx.x == 0) out[256 + blockIdx.x] = side_bytes;
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, 512); }
}

// Realistic pipeline: both CTAs' producers TMA their 128 A rows + 128 B rows per 64-deep
// k-block into an ST-stage ring (completion on the leader's full barrier), the leader's MMA
// thread waits full, issues 4 MMAs, commits to both CTAs' empty barriers (the kernels'
// protocol). Source rows drawn at random from `nrows` rows (32 MB: L2-resident; 512 MB:
// DRAM) in tiles of 16 k-blocks.
__device__ __forceinline__ void tma_pair(const CUtensorMap *m, uint64_t *bar, void *dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar) & ptx::kLeaderMask), "r"(x), "r"(y)
      : "memory");
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_pipe(const __grid_constant__ CUtensorMap tm, int nrows, int ST, int kblocks, unsigned long long *out, int side,
           const float4 *dsrc, float4 *ddst, int64_t dn4) {
  __shared__ volatile int stop;
  __shared__ unsigned long long side_bytes;
  if (threadIdx.x == 0) { stop = 0; side_bytes = 0; }
  extern __shared__ uint8_t raw[];
  uint8_t *smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[8], empty[8];
  __shared__ uint32_t tbase_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; i++) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_mbar_init();
  }
  if (warp == 2) { ptx::tmem_alloc2(&tbase_sh, 512); ptx::tmem_relinquish2(); }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = tbase_sh;
  if (warp == 0 && lane == 0) {
    uint32_t seed = (blockIdx.x >> 1) * 2654435761u + 99u;
    int ra = 0, rb = 0;
    for (int kb = 0; kb < kblocks; kb++) {
      if ((kb & 15) == 0) {
        seed = seed * 1664525u + 1013904223u;
        ra = (int)((seed >> 4) % (uint32_t)(nrows / 256)) * 256;
        seed = seed * 1664525u + 1013904223u;
        rb = (int)((seed >> 4) % (uint32_t)(nrows / 256)) * 256;
      }
      const int s = kb % ST;
      ptx::mbar_wait(&empty[s], ((kb / ST) & 1) ^ 1);
      if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * 32768);
      uint8_t *st = smem + s * 32768;
      tma_pair(&tm, &full[s], st, (kb & 15) * 64, ra + (int)rank * 128);
      tma_pair(&tm, &full[s], st + 16384, (kb & 15) * 64, rb + (int)rank * 128);
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    const uint32_t idesc = ptx::idesc_bf16(256, 256, 0, 0);
    const unsigned long long c0 = clock64();
    for (int kb = 0; kb < kblocks; kb++) {
      const int s = kb % ST;
      ptx::mbar_wait(&full[s], (kb / ST) & 1);
      ptx::tc_fence_after();
      const uint32_t a0 = ptx::smem_u32(smem + s * 32768), b0 = a0 + 16384;
#pragma unroll
      for (int k = 0; k < 4; k++)
        ptx::umma_bf16_2cta(tbase, ptx::sdesc_sw128(a0 + 32 * k, 16, 1024),
                            ptx::sdesc_sw128(b0 + 32 * k, 16, 1024), idesc, (kb & 15) | k);
      ptx::umma_commit_2cta(&empty[s]);
    }
    // all MMAs done: the last commit
    ptx::mbar_wait(&empty[(kblocks - 1) % ST], ((kblocks - 1) / ST) & 1);
    out[blockIdx.x >> 1] = clock64() - c0;
    stop = 1;
    uint32_t pa;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(pa) : "r"(ptx::smem_u32((const void *)&stop)));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(pa), "r"(1) : "memory");
  } else if (warp >= 4 && side) {
    // side traffic like an epilogue: 1 LDG (DRAM-resident), 2 TMEM loads of the other
    // accumulator, 3 STG, 4 LDG + STG, 5 LDG + STG + TMEM loads
    const int t = threadIdx.x - 128;
    unsigned long long mb = 0;
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * 256;
    int64_t i = (int64_t)blockIdx.x * 256 + t;
    const uint32_t tl = tbase + 256 + ((uint32_t)((warp & 3) * 32) << 16);
    int col = 0;
    while (!stop) {
      if (side == 2 || side == 5) {
        float v[8];
        ptx::tmem_ld8(tl + col, v);
        ptx::tmem_ld_wait();
        acc += v[0] + v[7];
        col = (col + 8) & 255;
        mb += 32 * 32 / 32;  // bytes per thread (8 x 4 B)
      }
      if (side == 1 || side == 4 || side == 5 || side == 8) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = side == 8 ? __ldcs(dsrc + i + u * stride) : __ldcg(dsrc + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; u++) acc += v[u].x + v[u].w;
        mb += 64;
        if (side >= 4) {
#pragma unroll
          for (int u = 0; u < 3; u++) {
            if (side == 8) __stcs(ddst + i + u * stride, v[u]);
            else ddst[i + u * stride] = v[u];
          }
          mb += 48;
        }
        i += 4 * stride;
        if (i + 4 * stride >= dn4) i = (int64_t)blockIdx.x * 256 + t;
      } else if (side == 3 || side == 6 || side == 7) {
        const float4 v = make_float4(1.f, 2.f, 3.f, (float)t);
        if (side == 3) {
#pragma unroll
          for (int u = 0; u < 4; u++) ddst[i + u * stride] = v;
        } else if (side == 6) {
#pragma unroll
          for (int u = 0; u < 4; u++) __stcs(ddst + i + u * stride, v);
        } else {
          uint64_t pol;
          asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
          for (int u = 0; u < 4; u++)
            asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ddst + i + u * stride),
                         "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                         : "memory");
        }
        mb += 64;
        i += 4 * stride;
        if (i + 4 * stride >= dn4) i = (int64_t)blockIdx.x * 256 + t;
      }
    }
    if (acc == 1234.5f) out[1000] = 1;
    atomicAdd(&side_bytes, mb);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[256 + blockIdx.x] = side_bytes;
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, 512); }
}

int main() {
  void *src;
  cudaMalloc(&src, (size_t)ROWS * COLS * 2);
  {  // non-zero, non-repeating data (no chance of compressible lines)
    unsigned short *h = (unsigned short *)malloc((size_t)ROWS * COLS * 2);
    uint32_t x = 12345u;
    for (size_t i = 0; i < (size_t)ROWS * COLS; i++) { x = x * 1664525u + 1013904223u; h[i] = (unsigned short)(x >> 16); }
    cudaMemcpy(src, h, (size_t)ROWS * COLS * 2, cudaMemcpyHostToDevice);
    free(h);
  }
  float4 *g1, *g2;
  cudaMalloc(&g1, GBUF * 4);
  cudaMalloc(&g2, GBUF * 4);
  {
    float *h = (float *)malloc(GBUF * 4);
    for (int64_t i = 0; i < GBUF; i++) h[i] = (float)(i % 977) * 0.25f + 1.f;
    cudaMemcpy(g1, h, GBUF * 4, cudaMemcpyHostToDevice);
    free(h);
  }
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {COLS, ROWS};
  cuuint64_t strides[1] = {COLS * 2};
  cuuint32_t box[2] = {64, 256};
  cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  unsigned long long *out;
  cudaMalloc(&out, 2048 * sizeof(unsigned long long));
  unsigned long long h[512];
  const char *names[] = {"none", "tma", "lds_sts", "ldg", "stg", "ldg_stg", "tma_ldg", "B_mn_major", "AB_mn_major"};
  const int kblocks = 8192, grid = 148;
  printf("{\"mma\": \"M256 N256 K16 bf16 cta_group::2, 4 per k-block, peak 128 clk each\", \"rows\": [\n");
  for (int mode = 0; mode < 9; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      k_probe<<<grid, 384, SMEM>>>(tm, mode, kblocks, g1, g2, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, out, 512 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double clk = 0, side = 0;
      for (int p = 0; p < grid / 2; p++) clk += h[p];
      clk /= grid / 2;
      for (int b = 0; b < grid; b++) side += h[256 + b];
      side /= grid;
      if (rep == 1)
        printf("  {\"side\": \"%s\", \"mma_frac_of_peak\": %.3f, \"clk_per_mma\": %.1f, \"side_B_per_clk_per_sm\": %.1f}%s\n",
               names[mode], 128.0 * 4 * kblocks / clk, clk / (4.0 * kblocks), side / clk, mode < 8 ? "," : "");
    }
  }
  printf("]}\n");
  // realistic pipeline: stages x source size
  {
    const int64_t big_rows = 262144;
    void *bsrc;
    cudaMalloc(&bsrc, (size_t)big_rows * COLS * 2);
    cudaMemset(bsrc, 0x3c, (size_t)big_rows * COLS * 2);
    cudaMemcpy(bsrc, src, (size_t)ROWS * COLS * 2, cudaMemcpyDeviceToDevice);
    CUtensorMap tb;
    cuuint64_t dims2[2] = {COLS, (cuuint64_t)big_rows};
    cuuint32_t box2[2] = {64, 128};
    enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bsrc, dims2, strides, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
    const int64_t dn4 = (int64_t)1 << 27;  // 2 GB of float4 (DRAM-resident side traffic)
    float4 *d1, *d2;
    cudaMalloc(&d1, dn4 * 16);
    cudaMalloc(&d2, dn4 * 16);
    cudaMemset(d1, 0x3f, dn4 * 16);
    printf("{\"pipeline\": \"TMA ring -> 2-CTA MMA, 32 KB per CTA per k-block, + side traffic\", \"rows\": [\n");
    const char *sn[] = {"none", "ldg_dram", "tmem_ld", "stg_dram", "ldg_stg_dram", "ldg_stg_tmem", "stg_cs", "stg_evict_first", "ldcs_stcs"};
    for (int big = 0; big < 2; big++)
      for (int side = 0; side < 9; side++) {
        const int st = big ? 6 : 4;
        for (int rep = 0; rep < 2; rep++) {
          k_pipe<<<148, 384, 6 * 32768 + 1024>>>(tb, big ? (int)big_rows : ROWS, st, 8192, out, side, d1, d2, dn4);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        }
        cudaMemcpy(h, out, 512 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double clk = 0, sb = 0;
        for (int p = 0; p < 74; p++) clk += h[p];
        clk /= 74;
        for (int b = 0; b < 148; b++) sb += h[256 + b];
        sb /= 148;
        printf("  {\"source_MB\": %d, \"stages\": %d, \"side\": \"%s\", \"mma_frac_of_peak\": %.3f, \"operand_B_per_clk_per_sm\": %.1f, \"side_B_per_clk_per_sm\": %.1f}%s\n",
               big ? 512 : 32, st, sn[side], 128.0 * 4 * 8192 / clk, 32768.0 * 8192 / clk, sb / clk, (big && side == 8) ? "" : ",");
      }
    printf("]}\n");
  }
  return 0;
}

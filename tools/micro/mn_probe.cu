// Does the B operand's major-ness change the 2-CTA tcgen05 MMA stream rate? Each CTA pair runs
// the kernels' pipeline (TMA ring of ST stages -> elected-lane MMAs M = 256, N in {128, 256},
// K = 16 x 4 per k-block -> commit to both CTAs' empty barriers) over L2-resident bf16 data,
// with B either K-major (box {64 K, N/2 rows}, like the forward's U) or MN-major (boxes of
// {64 N, 64 K} chunks, like the backward's dA = dZ U operand). Prints the MMA rate as a
// fraction of the tensor peak (N/2 cycles per MMA) and the operand bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1702_02181_b200/csrc \
//        tools/micro/mn_probe.cu -o /tmp/mn_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace fold;

constexpr int ROWS = 16384, COLS = 1024;  // 32 MB bf16 (row stride varied below: 1024..5120 elements)

__device__ __forceinline__ void tma_pair(const CUtensorMap *m, uint64_t *bar, void *dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar) & ptx::kLeaderMask), "r"(x), "r"(y)
      : "memory");
}

template <int N, int BMN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_probe(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int ST, int kblocks,
            unsigned long long *out, int rows_a = ROWS, int rows_b = ROWS) {
  constexpr int ABYTES = 128 * 128, BBYTES = (N / 2) * 128, STAGE = ABYTES + BBYTES, CH = 64 * 128;
  extern __shared__ uint8_t raw[];
  uint8_t *smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[8], empty[8];
  __shared__ uint32_t tbase_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1;
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
    for (int kb = 0; kb < kblocks; kb++) {
      const int tile = kb / 16, kk = kb % 16;
      const int ra = ((pair * 7919 + tile * 13) % (rows_a / 256)) * 256;
      const int rb = ((pair * 104729 + tile * 31) % ((BMN ? rows_b - 1024 : rows_b) / 256)) * 256;
      const int s = kb % ST;
      ptx::mbar_wait(&empty[s], ((kb / ST) & 1) ^ 1);
      if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * STAGE);
      uint8_t *st = smem + s * STAGE;
      tma_pair(&tmA, &full[s], st, kk * 64, ra + (int)rank * 128);
      if (BMN) {  // B[k][n]: rows = K, columns = N; this CTA's N/2 columns in 64-column chunks
        for (int ch = 0; ch < N / 128; ch++)
          tma_pair(&tmB, &full[s], st + ABYTES + ch * CH, (pair % 4) * 256 + (int)rank * (N / 2) + ch * 64,
                   rb + kk * 64);
      } else {
        tma_pair(&tmB, &full[s], st + ABYTES, kk * 64, rb + (int)rank * (N / 2));
      }
    }
  } else if (warp == 1 && rank == 0) {
    const uint32_t idesc = ptx::idesc_bf16(256, N, 0, BMN);
    const unsigned long long c0 = clock64();
    for (int kb = 0; kb < kblocks; kb++) {
      const int s = kb % ST;
      ptx::mbar_wait(&full[s], (kb / ST) & 1);
      __syncwarp();
      ptx::tc_fence_after();
      const uint32_t a0 = ptx::smem_u32(smem + s * STAGE), b0 = a0 + ABYTES;
      const uint64_t da = ptx::sdesc_sw128(a0, 16, 1024);
      const uint64_t db = BMN ? ptx::sdesc_sw128(b0, CH, 1024) : ptx::sdesc_sw128(b0, 16, 1024);
      if (ptx::elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; k++)
          ptx::umma_bf16_2cta(tbase, ptx::desc_add(da, 32 * k), ptx::desc_add(db, BMN ? 2048 * k : 32 * k), idesc,
                              (kb % 16) | k);
        ptx::umma_commit_2cta(&empty[s]);
      }
      __syncwarp();
    }
    ptx::mbar_wait(&empty[(kblocks - 1) % ST], ((kblocks - 1) / ST) & 1);
    if (lane == 0) out[pair] = clock64() - c0;
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, 512); }
}

// The C4 backward's exact access pattern: 64 pairs = 4 row tiles x 16 column tiles of a
// 1024-row level; pair (r, c) streams dZ rows [256 r, 256 r + 256) (K = 5120 columns) and U
// (MN-major, K = 5120 rows x 2048 columns) columns [128 c, 128 c + 128), 80 k-blocks per
// tile; `levels` tiles back to back, each level's dZ block 1024 rows further on.
template <int THREADS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_c4(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmU, int levels, int lockstep,
         unsigned long long *out, int npairs_work, int zlev = 3) {
  constexpr int N = 128, ABYTES = 128 * 128, STAGE = ABYTES + (N / 2) * 128, ST = 4, KB = 80;
  extern __shared__ uint8_t raw[];
  uint8_t *smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[ST], empty[ST], done;
  __shared__ uint32_t tbase_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1, r = (pair % 64) / 16, c = pair % 16;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; i++) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) { ptx::tmem_alloc2(&tbase_sh, 512); ptx::tmem_relinquish2(); }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = tbase_sh;
  if (pair >= npairs_work) {
  } else if (warp >= 4) {
    ptx::mbar_wait(&done, 0);  // idle epilogue warps parked on a barrier (try_wait loop)
  } else if (warp == 0 && lane == 0) {
    int it = 0;
    for (int l = 0; l < levels; l++)
      for (int kb = 0; kb < KB; kb++, it++) {
        const int s = it % ST;
        ptx::mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * STAGE);
        uint8_t *st = smem + s * STAGE;
        const int kk = lockstep ? kb : (kb + 5 * c) % KB;
        tma_pair(&tmZ, &full[s], st, kk * 64, (l % zlev) * 1024 + r * 256 + (int)rank * 128);
        tma_pair(&tmU, &full[s], st + ABYTES, c * 128 + (int)rank * 64, kk * 64);
      }
  } else if (warp == 1 && rank == 0) {
    const uint32_t idesc = ptx::idesc_bf16(256, N, 0, 1);
    const unsigned long long c0 = clock64();
    int it = 0;
    for (int l = 0; l < levels; l++)
      for (int kb = 0; kb < KB; kb++, it++) {
        const int s = it % ST;
        ptx::mbar_wait(&full[s], (it / ST) & 1);
        __syncwarp();
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(smem + s * STAGE), b0 = a0 + ABYTES;
        const uint64_t da = ptx::sdesc_sw128(a0, 16, 1024), db = ptx::sdesc_sw128(b0, 64 * 128, 1024);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; k++)
            ptx::umma_bf16_2cta(tbase, ptx::desc_add(da, 32 * k), ptx::desc_add(db, 2048 * k), idesc, kb | k);
          ptx::umma_commit_2cta(&empty[s]);
        }
        __syncwarp();
      }
    ptx::mbar_wait(&empty[(it - 1) % ST], ((it - 1) / ST) & 1);
    if (lane == 0) out[pair] = clock64() - c0;
  }
  if (warp == 1 && lane == 0) ptx::mbar_arrive(&done);
  if (THREADS > 128 && warp == 1 && lane == 0 && pair < npairs_work && rank == 1) {}
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc2(tbase, 512); }
}

// touch a buffer right before the probe: write (dirty lines, home L2 only) or read it
__global__ void k_touch(uint4 *p, size_t n, int write) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (; i < n; i += st) {
    if (write) p[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
    else { uint4 v = p[i]; acc.x ^= v.x; acc.y ^= v.y; }
  }
  if (acc.x == 0x12345678u && acc.y == 7u) p[0] = acc;
}

int main() {
  void *src;
  cudaMalloc(&src, (size_t)ROWS * COLS * 2);
  {
    unsigned short *h = (unsigned short *)malloc((size_t)ROWS * COLS * 2);
    uint32_t x = 12345u;
    for (size_t i = 0; i < (size_t)ROWS * COLS; i++) { x = x * 1664525u + 1013904223u; h[i] = (unsigned short)(x >> 16); }
    cudaMemcpy(src, h, (size_t)ROWS * COLS * 2, cudaMemcpyHostToDevice);
    free(h);
  }
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  auto mk = [&](CUtensorMap *m, int box_cols, int box_rows, int cols = COLS) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(ROWS * COLS / cols)};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUtensorMap tA, tB64, tB128, tMN;
  mk(&tA, 64, 128); mk(&tB64, 64, 64); mk(&tB128, 64, 128); mk(&tMN, 64, 64);
  const int smem = 7 * 32768 + 1024;
  cudaFuncSetAttribute(k_probe<128, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<256, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<256, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *out, h[128];
  cudaMalloc(&out, 128 * sizeof(unsigned long long));
  const int kblocks = 4096;
  printf("{\"probe\": \"B operand K-major vs MN-major, 2-CTA MMA stream (L2-resident)\", \"rows\": [\n");
  bool first = true;
  for (int N : {128, 256})
    for (int mn : {0, 1})
      for (int ST : {4, 6})
        for (int pairs : {64, 74}) {
          for (int rep = 0; rep < 2; rep++) {
            if (N == 128 && !mn) k_probe<128, 0><<<2 * pairs, 128, smem>>>(tA, tB64, ST, kblocks, out);
            if (N == 256 && !mn) k_probe<256, 0><<<2 * pairs, 128, smem>>>(tA, tB128, ST, kblocks, out);
            if (N == 128 && mn) k_probe<128, 1><<<2 * pairs, 128, smem>>>(tA, tMN, ST, kblocks, out);
            if (N == 256 && mn) k_probe<256, 1><<<2 * pairs, 128, smem>>>(tA, tMN, ST, kblocks, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          }
          cudaMemcpy(h, out, pairs * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
          double clk = 0;
          for (int p = 0; p < pairs; p++) clk += h[p];
          clk /= pairs;
          const double ideal = (double)kblocks * 4 * (N / 2);
          printf("%s  {\"N\": %d, \"b_major\": \"%s\", \"stages\": %d, \"pairs\": %d, \"mma_frac_of_peak\": %.3f, "
                 "\"operand_B_per_clk_per_sm\": %.1f}",
                 first ? "" : ",\n", N, mn ? "MN" : "K", ST, pairs, ideal / clk,
                 (double)kblocks * (128 * 128 + N / 2 * 128) / clk);
          first = false;
        }
  printf("\n]}\n");
  // the backward's operand shapes at S = 1024: dZ rows 5120 elements apart (10 KB), U (MN-major)
  // rows 2048 apart (4 KB); N = 128, 64 pairs
  printf("{\"probe\": \"row strides of the C4 backward (dZ 10 KB, U 4 KB) vs 2 KB\", \"rows\": [\n");
  first = true;
  for (int ac : {1024, 5120})
    for (int bc : {1024, 2048}) {
      CUtensorMap a2, b2;
      mk(&a2, 64, 128, ac);
      mk(&b2, 64, 64, bc);
      for (int rep = 0; rep < 2; rep++) k_probe<128, 1><<<128, 128, smem>>>(a2, b2, 4, kblocks, out, ROWS * COLS / ac, ROWS * COLS / bc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, out, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double clk = 0;
      for (int p = 0; p < 64; p++) clk += h[p];
      clk /= 64;
      printf("%s  {\"a_row_bytes\": %d, \"b_row_bytes\": %d, \"mma_frac_of_peak\": %.3f, \"operand_B_per_clk_per_sm\": %.1f}",
             first ? "" : ",\n", 2 * ac, 2 * bc, (double)kblocks * 4 * 64 / clk, (double)kblocks * (128 * 128 + 64 * 128) / clk);
      first = false;
    }
  printf("\n]}\n");
  {
    // dZ: 3 levels x 1024 rows x 5120 bf16 (30 MB); U: 5120 x 2048 bf16 (21 MB), MN-major
    void *z, *u;
    cudaMalloc(&z, (size_t)64 * 1024 * 5120 * 2);
    cudaMalloc(&u, (size_t)5120 * 2048 * 2);
    cudaMemset(z, 0x3c, (size_t)64 * 1024 * 5120 * 2);
    cudaMemset(u, 0x3c, (size_t)5120 * 2048 * 2);
    auto mk2 = [&](CUtensorMap *m, void *base, int cols, int rows, int bc, int br) {
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
      cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
      cuuint32_t es[2] = {1, 1};
      enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap tz, tu;
    mk2(&tz, z, 5120, 64 * 1024, 64, 128);
    mk2(&tu, u, 2048, 5120, 64, 64);
    cudaFuncSetAttribute(k_c4<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_c4<384>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    {  // random bf16 data in [-1, 1) instead of a constant fill
      const size_t nz = (size_t)3 * 1024 * 5120, nu = (size_t)5120 * 2048;
      unsigned short *hz = (unsigned short *)malloc(nz * 2);
      uint32_t x = 777u;
      for (size_t i = 0; i < nz; i++) { x = x * 1664525u + 1013904223u; hz[i] = (unsigned short)(0x3c00 | ((x >> 16) & 0x80ff)) ; }
      cudaMemcpy(z, hz, nz * 2, cudaMemcpyHostToDevice);
      cudaMemcpy(u, hz, nu * 2, cudaMemcpyHostToDevice);
      free(hz);
    }
    printf("{\"probe\": \"C4 backward access pattern (64 pairs: 4 row tiles x 16 column tiles, N = 128, K = 5120)\", \"rows\": [\n");
    for (int ls : {1, 0, 2, 3, 4}) {
      for (int rep = 0; rep < 2; rep++) {
        if (ls <= 1) k_c4<128><<<128, 128, smem>>>(tz, tu, 64, ls, out, 64);
        else if (ls == 2) k_c4<384><<<128, 384, smem>>>(tz, tu, 64, 1, out, 64);
        else if (ls == 3) k_c4<384><<<148, 384, smem>>>(tz, tu, 64, 1, out, 64);
        else k_c4<384><<<148, 384, smem>>>(tz, tu, 64, 1, out, 64, 64);  // every level's dZ block new (from DRAM)
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, out, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double clk = 0;
      for (int p = 0; p < 64; p++) clk += h[p];
      clk /= 64;
      const double kbt = 64.0 * 80;
      printf("%s  {\"variant\": %d, \"clk_per_kblock\": %.0f, \"mma_frac_of_peak\": %.3f, \"us_per_tile_at_1965MHz\": %.2f}",
             ls ? "" : ",\n", ls, clk / kbt, kbt * 4 * 64 / clk, clk / 64 / 1965.0);
    }
    printf("\n]}\n");
    // 8 levels, 8 distinct dZ blocks (84 MB: L2-resident), written or read by another kernel just before
    printf("{\"probe\": \"C4 pattern, dZ blocks freshly written vs freshly read by a previous kernel (8 levels)\", \"rows\": [\n");
    for (int w : {0, 1, 2, 3, 4, 5}) {
      // 0/1: 8 blocks read/written before, 8 levels; 2/3: 2 blocks read/written before, 2 levels;
      // 4/5: 2 blocks, 8 levels (each block re-read 4 times)
      const int nb = w < 2 ? 8 : 2, lev = w < 4 ? nb : 8;
      k_touch<<<1184, 256>>>((uint4 *)z, (size_t)nb * 1024 * 5120 * 2 / 16, w & 1);
      k_c4<384><<<148, 384, smem>>>(tz, tu, lev, 1, out, 64, nb);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, out, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double clk = 0;
      for (int p = 0; p < 64; p++) clk += h[p];
      clk /= 64;
      printf("  {\"dZ_touched_by\": \"%s\", \"blocks\": %d, \"levels\": %d, \"clk_per_kblock\": %.0f}", (w & 1) ? "write" : "read", nb, lev, clk / (lev * 80.0));
      printf(",\n");
    }
    printf("]}\n");
  }
  return 0;
}

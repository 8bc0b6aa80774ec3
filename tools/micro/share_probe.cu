// Is a 2-CTA tcgen05 mainloop slowed when many CTA pairs stream the SAME A-operand boxes at
// the same time (the backward's latency-bound levels: at C4 B=1024 the 16 column tiles of a
// 256-row tile read one dZ row tile together)? Each pair runs the kernels' pipeline (TMA ring
// of ST stages -> elected-lane MMAs M=256, N in {128, 256}, K=16 x 4 per k-block -> commit to
// both CTAs' empty barriers) over L2-resident bf16 data (32 MB); `share` consecutive pairs
// read identical A boxes (share = 1: every pair its own rows), B boxes are per pair.
// Prints the MMA rate as a fraction of the tensor peak (N/2 cycles per MMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1702_02181_b200/csrc \
//        tools/micro/share_probe.cu -o /tmp/share_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace fold;

constexpr int ROWS = 16384, COLS = 1024;  // 32 MB bf16

__device__ __forceinline__ void tma_pair(const CUtensorMap *m, uint64_t *bar, void *dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar) & ptx::kLeaderMask), "r"(x), "r"(y)
      : "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_share(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int share, int ST,
            int kblocks, unsigned long long *out) {
  constexpr int ABYTES = 128 * 128, BBYTES = (N / 2) * 128, STAGE = ABYTES + BBYTES;
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
    const int grp = pair / share;
    for (int kb = 0; kb < kblocks; kb++) {
      const int tile = kb / 16, kk = kb % 16;
      const int ra = ((grp * 7919 + tile * 13) % (ROWS / 256)) * 256;
      const int rb = ((pair * 104729 + tile * 31) % (ROWS / 256)) * 256;
      const int s = kb % ST;
      ptx::mbar_wait(&empty[s], ((kb / ST) & 1) ^ 1);
      if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * STAGE);
      uint8_t *st = smem + s * STAGE;
      tma_pair(&tmA, &full[s], st, kk * 64, ra + (int)rank * 128);
      tma_pair(&tmB, &full[s], st + ABYTES, kk * 64, rb + (int)rank * (N / 2));
    }
  } else if (warp == 1 && rank == 0) {
    const uint32_t idesc = ptx::idesc_bf16(256, N, 0, 0);
    const unsigned long long c0 = clock64();
    for (int kb = 0; kb < kblocks; kb++) {
      const int s = kb % ST;
      ptx::mbar_wait(&full[s], (kb / ST) & 1);
      __syncwarp();
      ptx::tc_fence_after();
      const uint32_t a0 = ptx::smem_u32(smem + s * STAGE), b0 = a0 + ABYTES;
      const uint64_t da = ptx::sdesc_sw128(a0, 16, 1024), db = ptx::sdesc_sw128(b0, 16, 1024);
      if (ptx::elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; k++)
          ptx::umma_bf16_2cta(tbase, ptx::desc_add(da, 32 * k), ptx::desc_add(db, 32 * k), idesc, (kb % 16) | k);
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
  auto mk = [&](CUtensorMap *m, int box_rows) {
    cuuint64_t dims[2] = {COLS, ROWS};
    cuuint64_t strides[1] = {COLS * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUtensorMap tA, tB64, tB128;
  mk(&tA, 128); mk(&tB64, 64); mk(&tB128, 128);
  const int smem = 8 * 32768 / 8 * 7 + 1024;  // <= 7 stages of 32 KB
  cudaFuncSetAttribute(k_share<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_share<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *out, h[128];
  cudaMalloc(&out, 128 * sizeof(unsigned long long));
  const int kblocks = 4096;
  printf("{\"probe\": \"A-operand sharing across CTA pairs (L2-resident)\", \"rows\": [\n");
  bool first = true;
  for (int N : {128, 256})
    for (int ST : {4, 6})
      for (int share : {1, 2, 8, 16, 37}) {
        for (int rep = 0; rep < 2; rep++) {
          if (N == 128) k_share<128><<<148, 128, smem>>>(tA, tB64, share, ST, kblocks, out);
          else k_share<256><<<148, 128, smem>>>(tA, tB128, share, ST, kblocks, out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        }
        cudaMemcpy(h, out, 74 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double clk = 0;
        for (int p = 0; p < 74; p++) clk += h[p];
        clk /= 74;
        const double ideal = (double)kblocks * 4 * (N / 2);
        printf("%s  {\"N\": %d, \"stages\": %d, \"pairs_sharing_A\": %d, \"mma_frac_of_peak\": %.3f, "
               "\"operand_B_per_clk_per_sm\": %.1f}",
               first ? "" : ",\n", N, ST, share, ideal / clk, (double)kblocks * (128 * 128 + N / 2 * 128) / clk);
        first = false;
      }
  printf("\n]}\n");
  return 0;
}

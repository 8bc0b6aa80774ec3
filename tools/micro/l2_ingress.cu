// L2 -> SM operand delivery on B200: is the wide GEMMs' ceiling a per-SM ingress limit or
// the chip's aggregate L2 (LTS) throughput? (the three pair-tile GEMMs move
// ~7.8 B of L2 operand traffic per kFLOP; k_gemm_dU_tc reaches ~8400 B/clk chip-wide.)
// Each CTA (one per SM: 200 KB of shared memory) streams TMA boxes of an L2-resident bf16
// matrix through a 4-stage x 32 KB ring without consuming them. Variants:
//   unicast, grid = 148 / 74 / 37 CTAs            -> per-SM vs aggregate limit
//   multicast, cluster 2 / 4: each CTA requests 1/cs of a stage and multicasts it to the
//   cluster (every CTA still lands 32 KB per stage) -> does multicast relieve the limit?
// Standalone tool (not part of libfold):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1702_02181_b200/csrc \
//        tools/micro/l2_ingress.cu -o /tmp/l2_ingress -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace fold;

constexpr int NST = 4;
constexpr int STAGE = 32768;  // 256 rows x 64 bf16 (128 B) per stage
constexpr int ROWS = 16384, COLS = 1024;  // 32 MB bf16 source (L2 resident)

__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
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
__device__ __forceinline__ void tma_mc(const CUtensorMap *m, uint64_t *bar, void *dst, int x, int y, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// cs = cluster size (1: unicast); box = 256 / cs rows
__global__ void __launch_bounds__(32, 1) k_ingress(const __grid_constant__ CUtensorMap tm1,
                                                   const __grid_constant__ CUtensorMap tm2,
                                                   const __grid_constant__ CUtensorMap tm4, int cs, int iters,
                                                   unsigned long long *out) {
  extern __shared__ uint8_t raw[];
  uint8_t *smem = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  const uint32_t rank = cs > 1 ? cluster_rank() : 0;
  const CUtensorMap *tm = cs == 1 ? &tm1 : cs == 2 ? &tm2 : &tm4;
  const int brows = 256 / cs;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], cs); }
    ptx::fence_mbar_init();
  }
  if (cs > 1) cluster_sync_all(); else __syncthreads();
  unsigned long long t0 = 0, c0 = 0;
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    c0 = clock64();
    // pseudo-random row block per CTA and iteration (no two CTAs request the same box at once)
    uint32_t seed = blockIdx.x * 2654435761u + 12345u;
    for (int it = 0; it < iters + NST; it++) {
      const int s = it % NST;
      const uint32_t ph = (it / NST) & 1;
      if (it >= NST) {
        ptx::mbar_wait(&full[s], ph ^ 1);  // round it - NST landed here
        // release the stage in every CTA of the cluster (their next multicast writes it)
        for (int c = 0; c < cs; c++) arrive_remote(mapa(ptx::smem_u32(&empty[s]), (uint32_t)c));
      }
      if (it >= iters) continue;
      if (it >= NST) mbar_wait_cluster(&empty[s], ph ^ 1);
      ptx::mbar_arrive_expect_tx(&full[s], STAGE);
      seed = seed * 1664525u + 1013904223u;
      const int rb = (int)((seed >> 8) % (uint32_t)(ROWS / 256));
      const int cb = (int)((seed >> 20) % (uint32_t)(COLS / 64));
      uint8_t *dst = smem + s * STAGE;
      if (cs == 1) {
        ptx::tma_load_2d(tm, &full[s], dst, cb * 64, rb * 256);
      } else {
        // all CTAs of the cluster use the same (rb, cb): rank r requests rows r*brows.. and
        // multicasts them to every CTA (same smem offset, each CTA's own full[s])
        tma_mc(tm, &full[s], dst + rank * brows * 128, cb * 64, rb * 256 + rank * brows, (uint16_t)((1u << cs) - 1));
      }
    }
    unsigned long long t1, c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[3 * blockIdx.x] = t1 - t0;
    out[3 * blockIdx.x + 1] = c1 - c0;
    out[3 * blockIdx.x + 2] = (unsigned long long)iters * STAGE;
  }
  if (cs > 1) cluster_sync_all();
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
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap tm[3];
  for (int i = 0; i < 3; i++) {
    const int cs = 1 << i;
    cuuint64_t dims[2] = {COLS, ROWS};
    cuuint64_t strides[1] = {COLS * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)(256 / cs)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }
  const int smem = NST * STAGE + 2048;  // > half the SM: one CTA per SM
  cudaFuncSetAttribute(k_ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_ingress, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  unsigned long long *out;
  cudaMalloc(&out, 3 * 148 * sizeof(unsigned long long));
  unsigned long long h[3 * 148];
  struct V { int grid, cs; } vs[] = {{148, 1}, {74, 1}, {37, 1}, {148, 2}, {148, 4}, {148, 1}};
  const int iters = 20000;
  printf("{\"rows\": [\n");
  for (size_t v = 0; v < sizeof(vs) / sizeof(vs[0]); v++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(vs[v].grid);
      cfg.blockDim = dim3(32);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = vs[v].cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchKernelEx(&cfg, k_ingress, tm[0], tm[1], tm[2], vs[v].cs, iters, out);
      cudaEventRecord(e1);
      cudaError_t e2 = cudaDeviceSynchronize();
      if (err != cudaSuccess || e2 != cudaSuccess) {
        printf("launch failed: %s / %s\n", cudaGetErrorString(err), cudaGetErrorString(e2));
        return 1;
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, out, 3 * vs[v].grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double bytes = 0, clk = 0, ns = 0;
      for (int b = 0; b < vs[v].grid; b++) { ns += h[3 * b]; clk += h[3 * b + 1]; bytes += h[3 * b + 2]; }
      ns /= vs[v].grid; clk /= vs[v].grid;
      const double per_sm_bpc = bytes / vs[v].grid / clk;
      const double ghz = clk / ns;
      if (rep == 1)
        printf("  {\"grid\": %d, \"cluster\": %d, \"landed_TBps\": %.2f, \"per_sm_B_per_clk\": %.1f, "
               "\"chip_B_per_clk\": %.0f, \"l2_requested_B_per_clk\": %.0f, \"sm_ghz\": %.3f, \"ms\": %.3f}%s\n",
               vs[v].grid, vs[v].cs, bytes / (ms * 1e-3) / 1e12, per_sm_bpc, per_sm_bpc * vs[v].grid,
               per_sm_bpc * vs[v].grid / vs[v].cs, ghz, ms, v + 1 < sizeof(vs) / sizeof(vs[0]) ? "," : "");
    }
  }
  printf("]}\n");
  return 0;
}

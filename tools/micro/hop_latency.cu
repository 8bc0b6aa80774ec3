// Dependency-hop latency floor on B200 ("report µs per level against a
// measured grid-barrier floor"). Two measurements, both with the publication pattern the
// executor uses (stores; __threadfence; atomicAdd on a counter; consumer polls with
// ld.acquire.gpu):
//  1. ping-pong between two CTAs on different SMs: one hop = round trip / 2;
//  2. a software grid barrier over 148 CTAs (the scheduler's gsync pattern), per barrier.
// Standalone tool (not part of libfold): nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void pingpong(int *cnt, int iters, long long *out) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;  // 0 or 1
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < iters; i++) {
    const int target = 2 * i + me;  // block 0 waits for even values, block 1 for odd
    while (ld_acquire(cnt) < target) {
    }
    __threadfence();
    atomicAdd(cnt, 1);
  }
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (me == 0) out[0] = (long long)(g1 - g0);
  (void)t0;
}

__global__ void gridbar(int *bar, int iters, long long *out) {
  __shared__ int dummy;
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < iters; i++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1);
      const int target = (i + 1) * gridDim.x;
      while (ld_acquire(bar) < target) {
      }
    }
    __syncthreads();
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (long long)(g1 - g0);
  dummy = 0;
}

int main() {
  int *cnt;
  long long *out, h[2];
  cudaMalloc(&cnt, 64);
  cudaMalloc(&out, 16);
  const int iters = 20000;
  for (int rep = 0; rep < 3; rep++) {
    cudaMemset(cnt, 0, 64);
    pingpong<<<2, 32>>>(cnt, iters, out);  // blocks land on different SMs
    cudaMemset(cnt + 8, 0, 4);
    gridbar<<<148, 128>>>(cnt + 8, iters / 10, out);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("{\"hop_us\": %.3f, \"grid_barrier_148_us\": %.3f, \"err\": \"%s\"}\n",
         h[0] / 1e3 / (2.0 * iters), h[1] / 1e3 / (iters / 10), cudaGetErrorString(cudaGetLastError()));
  return 0;
}

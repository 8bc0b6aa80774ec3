// common.cuh — shared helpers for the fold kernels (product code; nothing from oracle/).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/fold.h"

namespace fold {

constexpr int kWarp = 32;
constexpr int kNumSMsB200 = 148;

// Per-thread launch counter (instrumentation for bench.py's gpu_launches).
extern thread_local int64_t g_launches;

// Optional per-kernel-class CUDA-event timing (fold_profile_enable / fold_profile_read):
// when enabled, the launchers bracket their kernels with events on the launch stream.
enum KClass {
  K_SCHED = 0, K_EMBED_FWD, K_CELL_FWD, K_BWD_PW, K_GEMM_DA, K_GEMM_DU, K_EMBED_BWD, K_COLSUM,
  K_SGD, K_PREP, K_ROOT, K_NCLASS
};
void prof_mark(int cls, cudaStream_t st, bool begin);
struct ProfScope {
  int cls;
  cudaStream_t st;
  ProfScope(int c, cudaStream_t s) : cls(c), st(s) { prof_mark(cls, st, true); }
  ~ProfScope() { prof_mark(cls, st, false); }
};

// After every launch: count it, surface launch errors; with FOLD_DEBUG_SYNC=1 in the
// environment also synchronize and name the failing launch site on stderr.
fold_status launch_check(const char *file, int line);
#define FOLD_LAUNCH_CHECK()                                          \
  do {                                                               \
    fold_status _s = ::fold::launch_check(__FILE__, __LINE__);       \
    if (_s != FOLD_OK) return _s;                                    \
  } while (0)

#define FOLD_CUDA_TRY(x)                                      \
  do {                                                        \
    cudaError_t _e = (x);                                     \
    if (_e != cudaSuccess) return FOLD_E_CUDA;                \
  } while (0)

#define FOLD_TRY(x)                                           \
  do {                                                        \
    fold_status _s = (x);                                     \
    if (_s != FOLD_OK) return _s;                             \
  } while (0)

// Current device id clamped to [0, kMaxDevices): index of the per-device host caches
// (kernel attributes, occupancy and SM counts are per device).
constexpr int kMaxDevices = 16;
inline int cur_dev() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return cdiv(a, b) * b; }

// Row stride (elements) of H and C: >= S, multiple of 8 so that bf16 rows are
// 16-byte aligned (TMA global strides must be multiples of 16 bytes).
__host__ __device__ inline int ld_of(int S) { return (int)round_up(S, 8); }

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }
__device__ __forceinline__ float tanhf_(float x) { return tanhf(x); }
// BF16-path epilogues: hardware tanh (MUFU.TANH, max rel. error ~2^-11, far below the
// bf16 rounding of the stored states) and sigmoid(x) = 0.5 tanh(x/2) + 0.5.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigmoid_fast(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated atomic increment of a global counter; returns this lane's slot.
__device__ __forceinline__ int warp_push(int *counter, bool active) {
  unsigned mask = __ballot_sync(0xffffffffu, active);
  if (!mask) return -1;
  int leader = __ffs(mask) - 1;
  int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  return active ? base + __popc(mask & lanemask_lt()) : -1;
}

// Binary search: first index i in [0, n) with a[i] >= key (n if none).
__device__ __forceinline__ int lower_bound_dev(const int32_t *a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace fold

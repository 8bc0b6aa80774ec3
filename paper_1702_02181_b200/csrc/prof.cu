// prof.cu — optional CUDA-event timing per kernel class (bench.py's roofline figures are
// measured live inside the timed region with these events on the launch stream).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace fold {

namespace {
struct Rec {
  int cls;
  cudaEvent_t a, b;
};
thread_local bool g_on = false;
thread_local uint32_t g_mask = ~0u;  // classes recorded while on
thread_local std::vector<Rec> g_recs;
thread_local std::vector<cudaEvent_t> g_pool;
thread_local std::vector<std::pair<int, cudaEvent_t>> g_open;  // per-class open begin events

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

fold_status launch_check(const char *file, int line) {
  static const bool dbg = [] {
    const char *e = getenv("FOLD_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  g_launches++;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && dbg) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (dbg) fprintf(stderr, "[fold] CUDA error after launch at %s:%d: %s\n", file, line, cudaGetErrorString(e));
    return FOLD_E_CUDA;
  }
  return FOLD_OK;
}

void prof_mark(int cls, cudaStream_t st, bool begin) {
  if (!g_on || cls >= 32 || !((g_mask >> cls) & 1u)) return;
  cudaEvent_t e = get_event();
  cudaEventRecord(e, st);
  if (begin) {
    g_open.push_back({cls, e});
  } else {
    for (int i = (int)g_open.size() - 1; i >= 0; i--) {
      if (g_open[i].first == cls) {
        g_recs.push_back({cls, g_open[i].second, e});
        g_open.erase(g_open.begin() + i);
        return;
      }
    }
    g_pool.push_back(e);
  }
}

}  // namespace fold

using namespace fold;

extern "C" {

void fold_profile_enable(int32_t on) {
  for (auto &r : g_recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  g_recs.clear();
  for (auto &o : g_open) g_pool.push_back(o.second);
  g_open.clear();
  g_on = on != 0;
  g_mask = ~0u;
}

void fold_profile_enable_classes(uint32_t mask) {
  fold_profile_enable(mask != 0);
  g_mask = mask;
}

fold_status fold_profile_read(int32_t n_classes, double *ms, int64_t *launches) {
  if (!ms || !launches || n_classes < 0) return FOLD_E_INVALID;
  for (int i = 0; i < n_classes; i++) { ms[i] = 0.0; launches[i] = 0; }
  for (auto &r : g_recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return FOLD_E_CUDA;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return FOLD_E_CUDA;
    if (r.cls < n_classes) { ms[r.cls] += t; launches[r.cls] += 1; }
  }
  return FOLD_OK;
}

}  // extern "C"

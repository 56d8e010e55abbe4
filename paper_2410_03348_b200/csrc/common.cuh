// Shared helpers for the sm_100a kernels of the Dolphin hot path.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include "../../include/sgb200.h"

#define SG_RETURN_IF(cond, err) \
  do {                          \
    if (cond) return (int)(err); \
  } while (0)

#define SG_LAUNCH_CHECK()                      \
  do {                                         \
    cudaError_t e__ = cudaGetLastError();      \
    if (e__ != cudaSuccess) return (int)e__;   \
  } while (0)

namespace sg {

constexpr int kWarp = 32;

__device__ __forceinline__ float clamp01(float x) { return fminf(fmaxf(x, 0.0f), 1.0f); }

// A strided (rows, B) fp32 operand: row stride and sample stride (0 = broadcast sample).
struct Rows {
  const float* p;
  int64_t sr;  // stride between rows (symbols)
  int64_t sb;  // stride between samples (0 = broadcast)
  __device__ __forceinline__ float ld(int64_t r, int64_t b) const { return __ldg(p + r * sr + b * sb); }
};

struct WRows {
  float* p;
  int64_t sr;
  int64_t sb;
  __device__ __forceinline__ void st(int64_t r, int64_t b, float v) const { p[r * sr + b * sb] = v; }
};

__host__ __forceinline__ Rows rows_of(const sg_rows& r) { return Rows{r.ptr, r.stride_row, r.stride_b}; }
__host__ __forceinline__ WRows wrows_of(const sg_rows& r) { return WRows{r.ptr, r.stride_row, r.stride_b}; }

// Load one record of RW int32 words (RW in {1,2,4,8}); the address is warp-uniform.
template <int RW>
struct Rec {
  int v[RW];
};

template <int RW>
__device__ __forceinline__ Rec<RW> load_rec(const int32_t* __restrict__ p) {
  Rec<RW> r;
  if constexpr (RW == 1) {
    r.v[0] = __ldg(p);
  } else if constexpr (RW == 2) {
    int2 t = __ldg(reinterpret_cast<const int2*>(p));
    r.v[0] = t.x; r.v[1] = t.y;
  } else if constexpr (RW == 4) {
    int4 t = __ldg(reinterpret_cast<const int4*>(p));
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
  } else {
    int4 t = __ldg(reinterpret_cast<const int4*>(p));
    int4 u = __ldg(reinterpret_cast<const int4*>(p) + 1);
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
    r.v[4] = u.x; r.v[5] = u.y; r.v[6] = u.z; r.v[7] = u.w;
  }
  return r;
}

// Kernels enqueued by this library (every launch site calls count_launch once per
// kernel), exported as sg_launch_count() so callers can report what ran natively.
inline std::atomic<long long> g_launches{0};
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Raise a kernel's dynamic shared-memory limit (to the largest request seen so far) once
// per (device, kernel): repeated cudaFuncSetAttribute calls are avoided so launches stay
// legal inside CUDA-graph capture.
inline cudaError_t ensure_smem(const void* fn, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, fn);
  auto it = done.find(key);
  if (it != done.end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done[key] = smem;
  return e;
}

}  // namespace sg

// common.cuh — shared helpers of the MoEBlaze sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <algorithm>

#include "../../include/moeblaze.h"

namespace moeb {

// ----------------------------------------------------------------- launch accounting
// Every kernel launch of the library goes through MOE_LAUNCH so the bench can
// report how many of OUR kernels ran inside its timed region.
void note_launch();

// Bench instrumentation of the non-GEMM steps (moe_profile_read_named): while
// profiling is on, a scope brackets its launches with two CUDA events on the stream.
struct ProfScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a;
  ProfScope(const char* name, cudaStream_t st);
  ~ProfScope();
};

#define MOE_LAUNCH(kernel, grid, block, smem, stream, ...)                 \
  do {                                                                    \
    kernel<<<(grid), (block), (smem), (cudaStream_t)(stream)>>>(__VA_ARGS__); \
    ::moeb::note_launch();                                                \
  } while (0)

#define MOE_CUDA_CHECK(expr)                                              \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) return MOE_ERR_CUDA;                           \
  } while (0)

// ----------------------------------------------------------------- dtype helpers
__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

__device__ __forceinline__ float sigmoidf_(float a) { return 1.0f / (1.0f + __expf(-a)); }
// ~2-ulp sigmoid (MUFU.EX2 + MUFU.RCP, no IEEE division sequence) for the bf16
// tensor-core epilogues, whose outputs are rounded to bf16 (2^-9) anyway.
__device__ __forceinline__ float sigmoid_fast(float a) { return __fdividef(1.0f, 1.0f + __expf(-a)); }

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Index of the expert segment containing tile `i` given per-expert tile starts
// `start[0..E]` (start[E] = total).  Binary search, E <= 256.
__device__ __forceinline__ int find_segment(const int* start, int E, int i) {
  int lo = 0, hi = E;  // invariant: start[lo] <= i < start[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (start[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// 8 consecutive elements of a row as fp32 (16-byte load for bf16, 2 x 16 for fp32)
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* v) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void load8(const float* p, float* v) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* v) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = q;
}
__device__ __forceinline__ void store8(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

}  // namespace moeb

// common.cuh — shared device helpers for the Evoformer attention kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/evoattn.h"

namespace evo {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <> __device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half from_f<__half>(float x) { return __float2half_rn(x); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Shape/stride bundle shared by every kernel. Canonical row index b in
// [0, B) with B = Bo*N; tensors are (B, L, H, D) row-major.
struct Shape {
  int B, N, L, H, D;
  float scale;        // logit scale
  float scale_log2;   // scale * log2(e)
  const void* bias1;  // (B, L) or null
  const void* bias2;  // (Bo, H, L, L) or null
};

__device__ __forceinline__ size_t row_off(const Shape& s, int b, int i, int h) {
  return (((size_t)b * s.L + i) * s.H + h) * (size_t)s.D;
}

}  // namespace evo

// common.cuh — shared device helpers for the Evoformer attention kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/evoattn.h"

#ifndef EVO_TRACE
#define EVO_TRACE 0  // bring-up timelines (tools/trace_*.py build with -DEVO_TRACE=1); compiled out otherwise
#endif

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

// 2^x for a pair on the FMA pipe (relieves the MUFU pipe in softmax loops, FA4-style): x = n + f with
// n = round(x) by the 1.5*2^23 magic add, f in [-0.5, 0.5]; 2^f by a degree-3 fit (max relative error
// 7.7e-5, far below the bf16 rounding P receives); 2^n inserted into the exponent with one integer add.
// Inputs are clamped at -125 so the exponent add stays in the normal range (2^-125 ~ 2.4e-38 is
// zero for every use here: it rounds to 0 in bf16 P and vanishes in the fp32 row sums).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  const float2 lo = make_float2(-125.f, -125.f);
  x = make_float2(fmaxf(x.x, lo.x), fmaxf(x.y, lo.y));
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);                    // round(x) in the low mantissa bits
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-n.x, -n.y));  // [-0.5, 0.5]
  float2 p = __ffma2_rn(f, make_float2(0.05508868f, 0.05508868f), make_float2(0.24260405f, 0.24260405f));
  p = __ffma2_rn(f, p, make_float2(0.69327623f, 0.69327623f));
  p = __ffma2_rn(f, p, make_float2(0.99992895f, 0.99992895f));
  const int nx = __float_as_int(t.x) - 0x4B400000, ny = __float_as_int(t.y) - 0x4B400000;
  return make_float2(__int_as_float(__float_as_int(p.x) + (nx << 23)),
                     __int_as_float(__float_as_int(p.y) + (ny << 23)));
}

// acc[x] += part[0][x] + part[1][x] + ... + part[np-1][x], added one part at a time in ascending order
// (fp32): the fixed-order reduction of row / head / chunk partials — bit-reproducible.
template <typename F>
__global__ void ordered_sum_kernel(const F* __restrict__ part, int np, size_t stride, F* __restrict__ acc, size_t n) {
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n; x += (size_t)gridDim.x * blockDim.x) {
    F a = acc[x];
    for (int k = 0; k < np; ++k) a += part[(size_t)k * stride + x];
    acc[x] = a;
  }
}

// Shape/stride bundle shared by every kernel. Canonical row index b in
// [0, B) with B = Bo*N; tensors are (B, L, H, D) row-major.
struct Shape {
  int B, N, L, H, D;
  float scale;        // logit scale
  float scale_log2;   // scale * log2(e)
  const void* bias1;  // (B, L) or null
  const void* bias2;  // (Bo, H, L, L) or null
  int swapped;        // 1: q/k/v/o are (L, B, H, D) — the raw msa_col / tri_end layout (Bo == 1)
  int* flag;          // numeric-check word (NaN / non-finite results set it), or null: no checks
  const void* gate;   // output-gate logits G, same layout as O (OpenFold gating: O_g = sigmoid(G) * O), or null
  void* dgate;        // backward with a gate: dG output (layout of O)
  void* dog;          // backward with a gate: workspace for the gated dO = dO_g * sigmoid(G)
};

// sigmoid on the MUFU pipe: 1 / (1 + 2^(-g log2 e)) (0 and 1 at the saturated ends)
__device__ __forceinline__ float sigmoidf_fast(float g) { return __frcp_rn(1.f + ex2(-g * kLog2e)); }

// NumericError detection (attention_tiled.cpp:49-53, 62-65, 125-127, 209): a NaN input or a
// non-finite logit row shows up as a non-finite LSE / delta or a NaN output; the kernels OR a flag
// the C-ABI reads back when the caller asked for numeric checks.
__device__ __forceinline__ void flag_if(int* flag, bool bad) {
  if (flag && bad) atomicOr(flag, 1);
}

__device__ __forceinline__ size_t row_off(const Shape& s, int b, int i, int h) {
  return ((s.swapped ? (size_t)i * s.B + b : (size_t)b * s.L + i) * s.H + h) * (size_t)s.D;
}

}  // namespace evo

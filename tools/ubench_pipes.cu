// Micro-benchmark: per-SM throughput of the instructions the softmax loops are made of, to decide
// which pipe bounds them (MUFU ex2 vs the f32 -> bf16x2 pack vs packed FMA vs integer ops).
// One CTA of 512 threads per SM, 8 independent chains per thread; prints thread-ops / clock / SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pipes tools/ubench_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, float seed, long long* cyc, float* sink) {
  float a[8];
  uint32_t u[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { a[c] = seed * (threadIdx.x + c) * 1e-6f - 0.5f; u[c] = __float_as_uint(a[c]); }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if constexpr (MODE == 0) {  // ex2.approx.ftz.f32
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[c]));
      } else if constexpr (MODE == 1) {  // cvt.rn.bf16x2.f32 (dependent on itself through u)
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(a[c]), "f"(__uint_as_float(u[c])));
      } else if constexpr (MODE == 2) {  // cvt.rn.f16x2.f32
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(a[c]), "f"(__uint_as_float(u[c])));
      } else if constexpr (MODE == 3) {  // ex2 f32 + bf16x2 pack, 1:1
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[c]));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(a[c]), "f"(__uint_as_float(u[c])));
      } else if constexpr (MODE == 4) {  // ex2.approx.ftz.bf16x2
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[c]));
      } else if constexpr (MODE == 5) {  // ex2.approx.f16x2
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[c]));
      } else if constexpr (MODE == 6) {  // prmt
        asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(u[c]) : "r"(u[(c + 1) & 7]));
      } else if constexpr (MODE == 7) {  // fma.rn.f32x2
        asm volatile("{.reg .b64 x; mov.b64 x, {%0, %1}; fma.rn.f32x2 x, x, x, x; mov.b64 {%0, %1}, x;}"
                     : "+f"(a[c]), "+r"(u[c]));
      } else if constexpr (MODE == 8) {  // max.f32 three inputs
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(a[(c + 1) & 7]), "f"(a[(c + 2) & 7]));
      } else if constexpr (MODE == 9) {  // integer add (VIADD/IADD3)
        asm volatile("add.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(u[(c + 3) & 7]));
      } else if constexpr (MODE == 10) {  // f32 -> bf16 pair by integer round-half-up + prmt
        uint32_t x0 = u[c] + 0x8000u, x1 = u[(c + 1) & 7] + 0x8000u;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(u[c]) : "r"(x0), "r"(x1));
      } else if constexpr (MODE == 11) {  // ex2.bf16x2 + pack of its input, 1:1
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(a[c]), "f"(__uint_as_float(u[c])));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[c]));
      } else if constexpr (MODE == 12) {  // cvt.rn.satfinite.e4m3x2? no: f32 -> f16x2 via cvt.rn.f16x2 + ex2.f16x2
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(a[c]), "f"(__uint_as_float(u[c])));
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[c]));
      } else if constexpr (MODE == 13) {  // bf16x2 -> f32 pair unpack (shift + and): what the bias load costs
        const uint32_t lo = u[c] << 16, hi = u[c] & 0xFFFF0000u;
        a[c] += __uint_as_float(lo) + __uint_as_float(hi);
      } else if constexpr (MODE == 14) {  // fma.rn.bf16x2 (packed bf16 FMA)
        asm volatile("fma.rn.bf16x2 %0, %0, %1, %0;" : "+r"(u[c]) : "r"(u[(c + 1) & 7]));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c] + __uint_as_float(u[c]);
  if (s == 1.2345f) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, double ops_per_inner, long long* cyc, float* sink) {
  const int iters = 4096, threads = 512, blocks = 148;
  k<MODE><<<blocks, threads>>>(16, 1.f, cyc, sink);
  k<MODE><<<blocks, threads>>>(iters, 1.f, cyc, sink);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int b = 0; b < blocks; ++b) avg += h[b];
  avg /= blocks;
  const double ops = (double)iters * 8 * threads * ops_per_inner;
  printf("%-44s %8.2f thread-ops/clk/SM\n", name, ops / avg);
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 512 * 4);
  run<0>("ex2.approx.ftz.f32", 1, cyc, sink);
  run<1>("cvt.rn.bf16x2.f32", 1, cyc, sink);
  run<2>("cvt.rn.f16x2.f32", 1, cyc, sink);
  run<3>("ex2.f32 + cvt.bf16x2 (1:1, count both)", 2, cyc, sink);
  run<4>("ex2.approx.ftz.bf16x2 (instr)", 1, cyc, sink);
  run<5>("ex2.approx.f16x2 (instr)", 1, cyc, sink);
  run<6>("prmt", 1, cyc, sink);
  run<7>("fma.rn.f32x2 (instr)", 1, cyc, sink);
  run<8>("max.f32 3-input", 1, cyc, sink);
  run<9>("add.u32", 1, cyc, sink);
  run<10>("round+prmt pack (pairs)", 1, cyc, sink);
  run<11>("cvt.bf16x2 + ex2.bf16x2 (count both)", 2, cyc, sink);
  run<12>("cvt.f16x2 + ex2.f16x2 (count both)", 2, cyc, sink);
  run<13>("bf16x2 unpack + 2 fadd (pairs)", 1, cyc, sink);
  run<14>("fma.rn.bf16x2 (instr)", 1, cyc, sink);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

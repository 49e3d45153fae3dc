// Micro-benchmark: TMEM load/store throughput per SM (tcgen05.ld / st 32x32b) with 4, 8, 16
// warps, and MUFU ex2 throughput alone / mixed with TMEM loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_04610_b200/csrc -o tools/ubench_tmem tools/ubench_tmem.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"
#include "tc_ptx.cuh"

using namespace evo::ptx;

template <int MODE>  // 0: ld x32, 1: st x32, 2: ex2 only, 3: ld + ex2 mixed, 4: ld x16
__global__ void k(float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp / 4) * 32;
  float acc = 0.f;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 3) {
      tmem_ld32(tmem, r);
      tmem_ld_wait();
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
    if (MODE == 4) {
      uint32_t q[16];
      tmem_ld16(tmem, q);
      tmem_ld_wait();
      acc += __uint_as_float(q[0]) + __uint_as_float(q[15]);
    }
    if (MODE == 1) {
      tmem_st32(tmem, r);
      tmem_st_wait();
    }
    if (MODE == 2 || MODE == 3) {
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += evo::ex2(__uint_as_float(r[e]) * 1e-9f + acc * 1e-30f);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x * 2] = (float)(t1 - t0);
  out[blockIdx.x * 2 + 1] += acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int MODE>
void run(const char* name, int warps, float* out) {
  const int iters = 4096;
  k<MODE><<<148, warps * 32>>>(out, iters);
  cudaDeviceSynchronize();
  k<MODE><<<148, warps * 32>>>(out, iters);
  float h[2];
  cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
  const double cyc = h[0];
  const double bytes = (double)warps * 32 * 32 * 4 * iters;  // per SM (x32 of 4B per lane)
  const double ex2 = (double)warps * 32 * 32 * iters;
  printf("%-22s warps=%2d  cycles/iter=%8.1f  TMEM B/clk/SM=%7.1f  ex2/clk/SM=%6.2f  (%s)\n", name, warps,
         cyc / iters, (MODE <= 1 || MODE == 3) ? bytes / cyc : (MODE == 4 ? bytes / 2 / cyc : 0.0),
         (MODE >= 2 && MODE <= 3) ? ex2 / cyc : 0.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 2 * 4);
  cudaMemset(out, 0, 148 * 8);
  for (int w : {4, 8, 16}) run<0>("tcgen05.ld 32x32b.x32", w, out);
  for (int w : {4, 8, 16}) run<4>("tcgen05.ld 32x32b.x16", w, out);
  for (int w : {4, 8, 16}) run<1>("tcgen05.st 32x32b.x32", w, out);
  for (int w : {4, 8, 16}) run<2>("ex2 only", w, out);
  for (int w : {4, 8, 16}) run<3>("ld.x32 + 32 ex2", w, out);
  return 0;
}

// Micro-benchmark: cycles per tcgen05.mma (kind::f16, SS operands) for the shapes the backward uses.
// One CTA per SM, one elected thread issues `n` MMAs back to back into one accumulator, commits,
// waits; reports cycles per MMA (issue + execution, steady state).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_04610_b200/csrc -o tools/ubench_umma tools/ubench_umma.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"
#include "tc_ptx.cuh"

using namespace evo::ptx;

struct Shape {
  int M, N;
  bool a_mn, b_mn;
  uint32_t a_layout, b_layout, a_sbo, b_sbo, a_lbo, b_lbo;
  const char* name;
};

__global__ void k(Shape s, int n, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = instr_desc(s.M, s.N, false, s.a_mn, s.b_mn);
  const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    for (int rep = 0; rep < 2; ++rep) {
      __syncwarp();
      t0 = clock64();
      if (elect_one()) {
        const uint64_t ad = smem_desc(a, s.a_lbo, s.a_sbo, s.a_layout);
        const uint64_t bd = smem_desc(b, s.b_lbo, s.b_sbo, s.b_layout);
        const uint32_t m = (uint32_t)nacc - 1;
        for (int i = 0; i < n; i += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            mma_ss(tmem + ((uint32_t)(u & m) << 7), ad + (uint64_t)(u * 128), bd + (uint64_t)(u * 64), idesc, 1);
        }
        tc_commit(&bar);
      }
      __syncwarp();
      mbar_wait_spin(&bar, rep & 1);
      t1 = clock64();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}


// The backward's per-step MMA sequence: S, dP (M128 N64 K-major, 2 k-steps each), 8 x (dV, dK) M64 N32
// MN-major with dV at TMEM lane offset 16 (interleaved) or at +32 columns, 4 x dQ M128 N32.
__global__ void kstep(int interleave, int steps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idS = instr_desc(128, 64, false, false, false);
  const uint32_t idKV = instr_desc(64, 32, false, true, true);
  const uint32_t idQ = instr_desc(128, 32, false, false, true);
  const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
  if (warp == 0) {
    __syncwarp();
    const long long t0 = clock64();
    if (elect_one()) {
      const uint64_t aK = smem_desc(a, 16, 512, 4), bK = smem_desc(b, 16, 512, 4);
      const uint64_t aMN = smem_desc(a, 1024, 1024, 2), bMN = smem_desc(b, 1024, 512, 4);
      const uint64_t aQ = smem_desc(a, 16, 1024, 2);
      const uint32_t dv = interleave ? tmem + 480 + (16u << 16) : tmem + 448;
      for (int st = 0; st < steps; ++st) {
        const uint32_t sb = (st & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          mma_ss(tmem + sb, aK + kk * 2, bK + kk * 2, idS, kk);
          mma_ss(tmem + sb + 64, aK + 512 + kk * 2, bK + 256 + kk * 2, idS, kk);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_ss(dv, aMN + kk * 128, bMN + kk * 64, idKV, 1);
          mma_ss(tmem + 480, aMN + 1024 + kk * 128, bMN + 512 + kk * 64, idKV, 1);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_ss(tmem + 416, aQ + kk * 2, bK + kk * 64, idQ, kk);
      }
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait_spin(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  Shape shapes[] = {
      {128, 64, false, false, 4, 4, 512, 512, 16, 16, "M128 N64 K-major SW64 (S, dP)"},
      {128, 256, false, false, 4, 4, 512, 512, 16, 16, "M128 N256 K-major SW64"},
      {64, 32, true, true, 2, 4, 1024, 512, 1024, 1024, "M64 N32 A MN SW128, B MN SW64 (dK, dV)"},
      {64, 64, true, true, 2, 4, 1024, 512, 1024, 1024, "M64 N64 A MN SW128, B MN SW64"},
      {128, 32, false, true, 2, 4, 1024, 512, 16, 1024, "M128 N32 A K SW128, B MN SW64 (dQ)"},
      {128, 64, true, true, 2, 4, 1024, 512, 4096, 1024, "M128 N64 A MN SW128 (2 atoms), B MN SW64"},
      {64, 32, false, false, 4, 4, 512, 512, 16, 16, "M64 N32 K-major SW64"},
  };
  for (auto& s : shapes) {
    for (int nacc : {1, 2, 4}) {
      const int n = 256;
      if (s.N > 128 && nacc > 2) continue;
      k<<<148, 128, 70000>>>(s, n, nacc, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%-48s acc=%d  cycles/mma=%7.1f  floor=%5.1f  (%s)\n", s.name, nacc, (double)mx / n,
             (s.M < 128 ? 128.0 : s.M) * s.N / 256.0, cudaGetErrorString(e));
    }
  }
  cudaFuncSetAttribute(kstep, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int il = 0; il < 2; ++il) {
    const int steps = 64;
    kstep<<<148, 128, 70000>>>(il, steps, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("bwd step sequence (24 MMAs), dV %s: cycles/step=%7.1f (%s)\n", il ? "interleaved lane+16" : "separate columns",
           (double)mx / steps, cudaGetErrorString(e));
  }
  return 0;
}

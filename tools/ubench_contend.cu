// Micro-benchmark: does concurrent TMEM ld/st or shared-memory traffic from other warps slow the
// tensor pipe? Warp 0 issues a chain of UMMAs (M64 N32, SS, bf16) while warps 1..8 run
// MODE 0: nothing, 1: tcgen05.ld x16 loops, 2: tcgen05.ld + st loops, 3: LDS.128 loops,
// 4: STS.128 loops. Reports cycles per MMA and per background iteration.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_04610_b200/csrc -o tools/ubench_contend tools/ubench_contend.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"
#include "tc_ptx.cuh"

using namespace evo::ptx;

__global__ void k(int mode, int M, int N, int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool mn = M == 64;
  const uint32_t idesc = instr_desc(M, N, false, mn, mn);
  const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
  if (warp == 0) {
    __syncwarp();
    const long long t0 = clock64();
    if (elect_one()) {
      const uint64_t ad = smem_desc(a, 1024, 1024, 2);
      const uint64_t bd = smem_desc(b, 1024, 512, 4);
      for (int i = 0; i < n; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          mma_ss(tmem + ((uint32_t)(u & 1) << 6), ad + (uint64_t)(u * 128), bd + (uint64_t)(u * 64), idesc, 1);
      }
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait_spin(&bar, 0);
    const long long t1 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      done = 1;
    }
  } else if (warp <= 8 && mode > 0) {
    // background traffic on TMEM columns [256, 512) of this warp's lane quadrant / on smem [64K, 96K)
    const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256 + ((warp - 1) / 4) * 64;
    const uint32_t sa = smem_u32(smem + 65536) + (warp - 1) * 4096 + lane * 16;
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = lane + i;
    long long iters = 0;
    float acc = 0.f;
    while (!done) {
#pragma unroll 1
      for (int j = 0; j < 16; ++j) {
        if (mode == 1 || mode == 2) {
          tmem_ld16(ta + (j & 3) * 16, r);
          tmem_ld_wait();
          acc += __uint_as_float(r[0]);
          if (mode == 2) {
            tmem_st16(ta + (j & 3) * 16, r);
            tmem_st_wait();
          }
        } else if (mode == 3) {
          uint4 v;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(sa + (j & 7) * 512));
          acc += __uint_as_float(v.x);
        } else if (mode == 4) {
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sa + (j & 7) * 512), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
        }
      }
      iters += 16;
    }
    if (lane == 0 && warp == 1) out[blockIdx.x * 2 + 1] = iters;
    if (acc == 12345.f) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  const char* names[] = {"none", "tmem ld x16", "tmem ld+st x16", "LDS.128", "STS.128"};
  int shapes[][2] = {{64, 32}, {128, 64}};
  for (auto& sh : shapes) {
    for (int mode = 0; mode < 5; ++mode) {
      cudaMemset(out, 0, 148 * 16);
      const int n = 4096;
      k<<<148, 288, 100000>>>(mode, sh[0], sh[1], n, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[2];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      printf("M%d N%d  background=%-16s cycles/mma=%6.1f  bg warp iters/kcycle=%6.1f (%s)\n", sh[0], sh[1], names[mode],
             (double)h[0] / n, h[0] ? 1000.0 * h[1] / h[0] : 0.0, cudaGetErrorString(e));
    }
  }
  return 0;
}

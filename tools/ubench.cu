// Micro-benchmarks that decide the backward kernel's reduction strategy:
// how fast can B200 reduce fp32 partials (dQ / dBias) through L2 atomics,
// vector atomics, TMA bulk reductions and DSMEM, and how fast is MUFU ex2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_red_f32(float* buf, size_t n, int iters) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (size_t i = tid; i < n; i += stride)
      asm volatile("red.global.add.f32 [%0], %1;" :: "l"(buf + i), "f"(1.0f) : "memory");
}

__global__ void k_red_v4(float* buf, size_t n, int iters) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (size_t i = tid; i < n / 4; i += stride)
      asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(buf + 4 * i), "f"(1.0f), "f"(1.0f), "f"(1.0f), "f"(1.0f) : "memory");
}

__global__ void k_store(float4* buf, size_t n4, int iters) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (size_t i = tid; i < n4; i += stride) buf[i] = make_float4(it, 1, 2, 3);
}

// each CTA reduces a 16 KB smem tile into its own global slice with one bulk op per chunk
__global__ void k_bulk_red(float* buf, size_t n, int iters) {
  extern __shared__ __align__(128) float sm[];
  const int chunk = 4096;  // floats = 16 KB
  for (int i = threadIdx.x; i < chunk; i += blockDim.x) sm[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    size_t nchunks = n / chunk;
    for (int it = 0; it < iters; ++it) {
      for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                     :: "l"(buf + c * chunk), "r"(s), "r"(chunk * 4) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void k_ex2(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define EX(a) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    EX(a0) EX(a1) EX(a2) EX(a3) EX(a4) EX(a5) EX(a6) EX(a7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_ffma2(float* out, int iters) {
  float2 a = make_float2(threadIdx.x, 1.f), b = make_float2(0.999f, 0.998f), c = make_float2(0.1f, 0.2f);
  float2 d = a, e = a, f = a;
  for (int i = 0; i < iters; ++i) {
    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*(unsigned long long*)&a) : "l"(*(unsigned long long*)&b), "l"(*(unsigned long long*)&c));
    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*(unsigned long long*)&d) : "l"(*(unsigned long long*)&b), "l"(*(unsigned long long*)&c));
    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*(unsigned long long*)&e) : "l"(*(unsigned long long*)&b), "l"(*(unsigned long long*)&c));
    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*(unsigned long long*)&f) : "l"(*(unsigned long long*)&b), "l"(*(unsigned long long*)&c));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a.x + d.x + e.x + f.x + a.y;
}

// DSMEM: every CTA of a cluster of 4 pushes fp32 adds into its right neighbour's smem
__global__ void __cluster_dims__(4, 1, 1) k_dsmem_red(float* out, int iters) {
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 0.f;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  unsigned rank = cl.block_rank();
  float* peer = cl.map_shared_rank(sm, (rank + 1) % 4);
  for (int it = 0; it < iters; ++it)
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) atomicAdd(peer + i, 1.0f);
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

__global__ void __cluster_dims__(4, 1, 1) k_dsmem_st(float* out, int iters) {
  __shared__ float4 sm[2048];
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  unsigned rank = cl.block_rank();
  float4* peer = cl.map_shared_rank(sm, (rank + 1) % 4);
  for (int it = 0; it < iters; ++it)
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) peer[i] = make_float4(it, i, 0, 1);
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[1].x;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  const size_t n = 16u << 20;  // 16M floats = 64 MB (L2 resident)
  float* buf; CK(cudaMalloc(&buf, n * 4)); CK(cudaMemset(buf, 0, n * 4));
  auto timeit = [&](const char* name, auto launch, double bytes) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("%-28s %9.3f ms  %8.1f GB/s %s\n", name, ms, bytes / ms / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  int it = 4;
  timeit("store.v4 (L2 64MB)", [&] { k_store<<<sms * 8, 256>>>((float4*)buf, n / 4, it); }, 4.0 * n * it);
  timeit("red.f32 (64MB)", [&] { k_red_f32<<<sms * 8, 256>>>(buf, n, it); }, 4.0 * n * it);
  timeit("red.v4.f32 (64MB)", [&] { k_red_v4<<<sms * 8, 256>>>(buf, n, it); }, 4.0 * n * it);
  CK(cudaFuncSetAttribute(k_bulk_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  timeit("bulk reduce.add.f32 (64MB)", [&] { k_bulk_red<<<sms, 128, 16384>>>(buf, n, it); }, 4.0 * n * it);
  timeit("bulk reduce x2 CTA/SM", [&] { k_bulk_red<<<sms * 2, 128, 16384>>>(buf, n, it); }, 4.0 * n * it);
  const size_t nb = 256u << 20;  // 1 GB (HBM)
  float* big; CK(cudaMalloc(&big, nb * 4)); CK(cudaMemset(big, 0, nb * 4));
  timeit("store.v4 (HBM 1GB)", [&] { k_store<<<sms * 8, 256>>>((float4*)big, nb / 4, 1); }, 4.0 * nb);
  timeit("red.v4.f32 (HBM 1GB)", [&] { k_red_v4<<<sms * 8, 256>>>(big, nb, 1); }, 4.0 * nb);
  timeit("bulk reduce (HBM 1GB)", [&] { k_bulk_red<<<sms * 2, 128, 16384>>>(big, nb, 1); }, 4.0 * nb);
  float* out; CK(cudaMalloc(&out, sms * 8 * 256 * 4));
  int iters = 4096;
  cudaEventRecord(e0); k_ex2<<<sms * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double ex = (double)sms * 4 * 256 * iters * 8;
  printf("ex2.approx: %.3f ms  %.2f Tex2/s  = %.2f per SM per ns\n", ms, ex / ms / 1e9, ex / ms / 1e6 / sms);
  cudaEventRecord(e0); k_ffma2<<<sms * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fm = (double)sms * 4 * 256 * iters * 4 * 2;
  printf("fma.f32x2: %.3f ms  %.2f Tfma/s = %.2f per SM per ns\n", ms, fm / ms / 1e9, fm / ms / 1e6 / sms);
  int itd = 256;
  timeit("dsmem atomicAdd f32", [&] { k_dsmem_red<<<sms, 256>>>(out, itd); }, 4.0 * 4096 * itd * sms);
  timeit("dsmem st.v4", [&] { k_dsmem_st<<<sms, 256>>>(out, itd); }, 16.0 * 2048 * itd * sms);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sm clock attr %d kHz, SMs %d\n", clk, sms);
  return 0;
}

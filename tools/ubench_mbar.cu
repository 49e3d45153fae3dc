// Micro-benchmark: latency of mbarrier.try_wait on an already-completed phase (one warp), alone and
// while other warps sit in sleeping try_waits on another barrier; and the round trip of an
// arrive -> wake-up handshake between two warps (ping-pong).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_04610_b200/csrc -o tools/ubench_mbar tools/ubench_mbar.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"
#include "tc_ptx.cuh"

using namespace evo::ptx;

__global__ void k(int mode, int iters, long long* out) {
  __shared__ uint64_t done_bar, idle_bar, ping, pong;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&done_bar, 1);
    mbar_init(&idle_bar, 1);
    mbar_init(&ping, 1);
    mbar_init(&pong, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&done_bar);  // phase 0 complete
  __syncthreads();
  if (mode <= 1) {
    if (warp == 0) {
      long long t0 = clock64();
      uint32_t s = 0;
      for (int i = 0; i < iters; ++i) s += mbar_try_wait(&done_bar, 0) ? 1 : 0;
      long long t1 = clock64();
      if (lane == 0) out[blockIdx.x] = (t1 - t0) * 1000 / iters + (s == 12345);
      if (lane == 0) mbar_arrive(&idle_bar);
    } else if (mode == 1) {
      mbar_wait(&idle_bar, 0);  // sleeping waiters
    }
  } else {
    // ping-pong: warp 0 arrives ping, warp 1 waits ping then arrives pong, warp 0 waits pong
    if (warp == 0) {
      long long t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        if (lane == 0) mbar_arrive(&ping);
        if (mode == 2) mbar_wait_spin(&pong, i & 1); else mbar_wait(&pong, i & 1);
      }
      long long t1 = clock64();
      if (lane == 0) out[blockIdx.x] = (t1 - t0) * 1000 / iters;
    } else if (warp == 1) {
      for (int i = 0; i < iters; ++i) {
        if (mode == 2) mbar_wait_spin(&ping, i & 1); else mbar_wait(&ping, i & 1);
        if (lane == 0) mbar_arrive(&pong);
      }
    }
  }
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * 8);
  const char* names[] = {"try_wait on completed phase, alone", "try_wait on completed phase, 8 warps sleeping",
                         "ping-pong round trip, spin waits", "ping-pong round trip, sleep-hint waits"};
  for (int mode = 0; mode < 4; ++mode) {
    k<<<148, 288, 0>>>(mode, 4096, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("%-48s %8.1f cycles (%s)\n", names[mode], h / 1000.0, cudaGetErrorString(e));
  }
  return 0;
}

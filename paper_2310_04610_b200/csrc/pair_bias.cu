// pair_bias.cu — the pair-bias projection that feeds the attention's bias2:
//
//   bias2[b, h, i, j] = sum_c LN(z[b, i, j, :])_c * W[c, h],   LN(x) = (x - mean) * rstd * gamma + beta
//
// (OpenFold's MSARowAttentionWithPairBias: layer_norm_z then linear_z without bias; the reference has
// no counterpart, SPEC.md:153 lists projections as non-goals). The forward writes straight into the
// [Bo, 1, H, L, L] layout K1 / K3 read (no permute / contiguous pass over the bias); the backward
// consumes K3's dBias2 in that same layout (fp32, or the 16-bit type) — no transpose, no rounding of
// dBias2 on the way. Both passes are HBM-bound over z (c_z channels per (i, j)): one warp per (i, j)
// row, c_z / 32 channels per lane, LayerNorm statistics by warp shuffles; a CTA owns 32 consecutive j
// of one (b, i) so the per-head bias rows it writes (or dBias2 rows it reads) are contiguous.
// The weight gradients are per-CTA partial sums reduced in a fixed order (deterministic).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "evoattn.h"
#include "tc_ptx.cuh"

namespace evo {
void set_last_error(const char* msg);  // evoattn_capi.cu
}

namespace {

constexpr int kWarps = 8, kRowsPerWarp = 4, kTileJ = kWarps * kRowsPerWarp;  // 32 j per CTA

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CPL consecutive 16-bit values of one lane (2 * CPL bytes, naturally aligned): one vector access
template <int CPL> struct Vec { using type = unsigned short; };
template <> struct Vec<2> { using type = uint32_t; };
template <> struct Vec<4> { using type = uint2; };
template <> struct Vec<8> { using type = uint4; };

template <typename T, int CPL>
__device__ __forceinline__ void load_row(const T* p, float* x) {
  union { typename Vec<CPL>::type v; T e[CPL]; } u;
  u.v = *(const typename Vec<CPL>::type*)p;
#pragma unroll
  for (int k = 0; k < CPL; ++k) x[k] = evo::to_f(u.e[k]);
}

template <typename T, int CPL>
__device__ __forceinline__ void store_row(T* p, const float* x) {
  union { typename Vec<CPL>::type v; T e[CPL]; } u;
#pragma unroll
  for (int k = 0; k < CPL; ++k) u.e[k] = evo::from_f<T>(x[k]);
  *(typename Vec<CPL>::type*)p = u.v;
}

// LayerNorm statistics of one row held CPL channels per lane (two-pass, fp32)
template <int CPL>
__device__ __forceinline__ void ln_stats(const float* x, int C, float eps, float& mean, float& rstd) {
  const float invC = 1.f / (float)C;
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < CPL; ++k) s += x[k];
  mean = warp_sum(s) * invC;
  float v = 0.f;
#pragma unroll
  for (int k = 0; k < CPL; ++k) v += (x[k] - mean) * (x[k] - mean);
  rstd = rsqrtf(warp_sum(v) * invC + eps);
}

// Sum of v[0..HM) over the warp, scattered: afterwards lane l holds the total of head
// h = scatter_head<HM>(l) (halving exchanges, then plain butterflies: HM - 1 + 5 - log2 HM shuffles
// instead of 5 HM)
template <int HM>
__device__ __forceinline__ float warp_sum_scatter(float* v, int lane) {
  int n = HM;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (n > 1) {
      const bool up = lane & off;
#pragma unroll
      for (int k = 0; k < HM / 2; ++k)
        if (k < n / 2) {
          const float mine = up ? v[k + n / 2] : v[k], other = up ? v[k] : v[k + n / 2];
          v[k] = mine + __shfl_xor_sync(0xffffffffu, other, off);
        }
      n >>= 1;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}
template <int HM>
__device__ __forceinline__ int scatter_head(int lane) {  // the head warp_sum_scatter leaves in `lane`
  int h = 0, n = HM;
#pragma unroll
  for (int off = 16; off >= 1 && n > 1; off >>= 1, n >>= 1)
    if (lane & off) h += n / 2;
  return h;
}

// W [C][H] fp32 into shared memory as ws[(k * HM + h) * 32 + lane] = W[lane * CPL + k][h] (0 past H):
// lane-contiguous, conflict-free reads
template <int CPL, int HM>
__device__ __forceinline__ void stage_w(const float* __restrict__ w, float* ws, int H) {
  for (int t = threadIdx.x; t < CPL * HM * 32; t += blockDim.x) {
    const int ln = t % 32, h = (t / 32) % HM, k = t / (32 * HM);
    ws[t] = h < H ? w[(size_t)(ln * CPL + k) * H + h] : 0.f;
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   evo::ptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(evo::ptx::smem_u32(bar))
               : "memory");
}

// Forward, persistent (one wave): a CTA walks (b, i, 8*FR-wide j) tiles; the tile's z rows are one
// contiguous block, bulk-copied (TMA engine, no registers) into a double-buffered shared stage while
// the previous tile is reduced — the HBM stream never waits on the shuffles.
template <typename T, int CPL, int HM, int FR>
__global__ void __launch_bounds__(kWarps * 32) pair_bias_fwd_kernel(const T* __restrict__ z, const float* __restrict__ gam,
                                                                    const float* __restrict__ bet,
                                                                    const float* __restrict__ w, T* __restrict__ out,
                                                                    int Bo, int L, int C, int H, float eps) {
  constexpr int TJ = kWarps * FR;
  __shared__ float tile[HM][TJ];
  __shared__ alignas(8) uint64_t full[2];
  extern __shared__ __align__(128) unsigned char dsm[];
  float* ws = (float*)dsm;                                     // CPL * HM * 32
  T* stage = (T*)(dsm + (size_t)CPL * HM * 32 * 4);           // [2][TJ][C]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nj = (L + TJ - 1) / TJ;
  const int ntiles = Bo * L * nj;
  const int c0 = lane * CPL;
  const float invC = 1.f / (float)C;
  auto issue = [&](int tix, int st) {  // one thread: the tile's rows j0 .. min(j0 + TJ, L) - 1
    const int jt = tix % nj, i = (tix / nj) % L, b = tix / (nj * L), j0 = jt * TJ;
    const uint32_t bytes = (uint32_t)(min(TJ, L - j0) * C * (int)sizeof(T));
    evo::ptx::mbar_expect_tx(&full[st], bytes);
    bulk_g2s(stage + (size_t)st * TJ * C, z + (((size_t)b * L + i) * L + j0) * C, bytes, &full[st]);
  };
  if (threadIdx.x == 0) {
    evo::ptx::mbar_init(&full[0], 1);
    evo::ptx::mbar_init(&full[1], 1);
    evo::ptx::fence_barrier_init();
  }
  stage_w<CPL, HM>(w, ws, H);
  __syncthreads();
  if (threadIdx.x == 0) {
    if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  float g[CPL], be[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    g[k] = gam[c0 + k];
    be[k] = bet[c0 + k];
  }
  const int hl = scatter_head<HM>(lane);
  int n = 0;
  for (int tix = blockIdx.x; tix < ntiles; tix += gridDim.x, ++n) {
    const int st = n & 1;
    const int jt = tix % nj, i = (tix / nj) % L, b = tix / (nj * L);
    const int nval = min(TJ, L - jt * TJ);
    evo::ptx::mbar_wait(&full[st], (n >> 1) & 1);
    float x[FR][CPL];
#pragma unroll
    for (int r = 0; r < FR; ++r)  // rows past L read the last valid row (not stored)
      load_row<T, CPL>(stage + ((size_t)st * TJ + min(warp * FR + r, nval - 1)) * C + c0, x[r]);
    __syncthreads();  // stage st read by every warp; the previous tile's outputs written
    if (threadIdx.x == 0 && tix + 2 * (int)gridDim.x < ntiles) issue(tix + 2 * gridDim.x, st);
    float mean[FR], rstd[FR];
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      float sm = 0.f;
#pragma unroll
      for (int k = 0; k < CPL; ++k) sm += x[r][k];
      mean[r] = sm;
    }
#pragma unroll
    for (int r = 0; r < FR; ++r) mean[r] = warp_sum(mean[r]) * invC;
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      float v = 0.f;
#pragma unroll
      for (int k = 0; k < CPL; ++k) v += (x[r][k] - mean[r]) * (x[r][k] - mean[r]);
      rstd[r] = v;
    }
#pragma unroll
    for (int r = 0; r < FR; ++r) rstd[r] = rsqrtf(warp_sum(rstd[r]) * invC + eps);
#pragma unroll
    for (int r = 0; r < FR; ++r)
#pragma unroll
      for (int k = 0; k < CPL; ++k) x[r][k] = (x[r][k] - mean[r]) * rstd[r] * g[k] + be[k];  // y
    float acc[FR][HM];
#pragma unroll
    for (int r = 0; r < FR; ++r)
#pragma unroll
      for (int h = 0; h < HM; ++h) acc[r][h] = 0.f;
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
      for (int h = 0; h < HM; ++h) {
        const float wv = ws[(k * HM + h) * 32 + lane];
#pragma unroll
        for (int r = 0; r < FR; ++r) acc[r][h] = fmaf(x[r][k], wv, acc[r][h]);
      }
#pragma unroll
    for (int r = 0; r < FR; ++r) {
      const float t = warp_sum_scatter<HM>(acc[r], lane);
      if ((lane & (32 / HM - 1)) == 0) tile[hl][warp * FR + r] = t;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < H * TJ; t += blockDim.x) {
      const int h = t / TJ, jj = t % TJ, j = jt * TJ + jj;
      if (j < L) out[(((size_t)b * H + h) * L + i) * L + j] = evo::from_f<T>(tile[h][jj]);
    }
  }
}

// Forward on the tensor pipe (mma.sync m16n8k16, fp32 accumulate): with W' = diag(gamma) W rounded to
// the 16-bit type, s1[h] = sum_c W'[c][h] and s2[h] = sum_c beta_c W[c][h],
//   bias[row][h] = rstd_row * (z_row . W'[:, h] - mean_row * s1[h]) + s2[h]
// — the LayerNorm folded into an epilogue, the c_z x H contraction a 64-row x C x H MMA per warp tile
// on the raw z values (exact 16-bit inputs). The rows land in a double-buffered shared stage by bulk
// copies, one per row at a padded pitch (C * 2 + 16 bytes: conflict-free fragment loads); the per-row
// statistics (sum, sum of squares in fp32) come from two lanes per row.
template <typename T, int HM>
__global__ void __launch_bounds__(128) pair_bias_fwd_mma_kernel(const T* __restrict__ z, const float* __restrict__ gam,
                                                              const float* __restrict__ bet,
                                                              const float* __restrict__ w, T* __restrict__ out,
                                                              int Bo, int L, int C, int H, float eps) {
  constexpr int TJ = 64;           // rows per tile: 4 warps x 16
  constexpr int NT = HM / 8;       // n tiles of 8 heads
  constexpr int KMAX = 256 / 16;   // k steps at the largest c_z
  __shared__ float tile[HM][TJ];
  __shared__ float s1s[HM], s2s[HM];
  __shared__ alignas(8) uint64_t full[2];
  extern __shared__ __align__(128) unsigned char dsm[];
  const int pitch = C * 2 + 16;    // bytes per staged row
  unsigned char* stage = dsm;      // [2][TJ][pitch]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nj = (L + TJ - 1) / TJ;
  const int ntiles = Bo * L * nj;
  const int KS = C / 16;
  const float invC = 1.f / (float)C;
  // B fragments (W' = gamma * W in the 16-bit type), per k step and n tile: b0 = (k 2q, 2q+1; n g),
  // b1 = (k 8 + 2q, 9 + 2q; n g) with g = lane / 4, q = lane % 4
  uint32_t bf[KMAX][NT][2];
  {
    const int g = lane / 4, q = lane % 4;
#pragma unroll
    for (int ks = 0; ks < KMAX; ++ks)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t v = 0u;
          const int h = nt * 8 + g, k0 = ks * 16 + hf * 8 + 2 * q;
          if (ks < KS && h < H) {
            T e[2];
            e[0] = evo::from_f<T>(gam[k0] * w[(size_t)k0 * H + h]);
            e[1] = evo::from_f<T>(gam[k0 + 1] * w[(size_t)(k0 + 1) * H + h]);
            v = *(const uint32_t*)e;
          }
          bf[ks][nt][hf] = v;
        }
  }
  {  // s1 from the rounded W' (consistent with the MMA), s2 in fp32: channels over the threads, then a
     // fixed-order reduction (warp shuffles, then the 4 warps in order)
    __shared__ float red1[4][HM], red2[4][HM];
    float v1[HM], v2[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) v1[h] = v2[h] = 0.f;
    for (int c = threadIdx.x; c < C; c += blockDim.x)
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < H) {
          const float wv = w[(size_t)c * H + h];
          v1[h] += evo::to_f(evo::from_f<T>(gam[c] * wv));
          v2[h] += bet[c] * wv;
        }
#pragma unroll
    for (int h = 0; h < HM; ++h) {
      const float a = warp_sum(v1[h]), c2 = warp_sum(v2[h]);
      if (lane == 0) { red1[warp][h] = a; red2[warp][h] = c2; }
    }
    __syncthreads();
    if (threadIdx.x < HM) {
      float a = 0.f, c2 = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) { a += red1[q][threadIdx.x]; c2 += red2[q][threadIdx.x]; }
      s1s[threadIdx.x] = a;
      s2s[threadIdx.x] = c2;
    }
  }
  auto issue = [&](int tix, int st) {  // warp 0: a bulk copy per row (padded pitch), rows over the lanes
    const int jt = tix % nj, i = (tix / nj) % L, b = tix / (nj * L), j0 = jt * TJ;
    const int nr = min(TJ, L - j0);
    if (lane == 0) evo::ptx::mbar_expect_tx(&full[st], (uint32_t)(nr * C * 2));
    __syncwarp();
    const T* src = z + (((size_t)b * L + i) * L + j0) * C;
    for (int r = lane; r < nr; r += 32)
      bulk_g2s(stage + ((size_t)st * TJ + r) * pitch, src + (size_t)r * C, (uint32_t)(C * 2), &full[st]);
  };
  if (threadIdx.x == 0) {
    evo::ptx::mbar_init(&full[0], 1);
    evo::ptx::mbar_init(&full[1], 1);
    evo::ptx::fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) {
    if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  int n = 0;
  for (int tix = blockIdx.x; tix < ntiles; tix += gridDim.x, ++n) {
    const int st = n & 1;
    const int jt = tix % nj, i = (tix / nj) % L, b = tix / (nj * L);
    evo::ptx::mbar_wait(&full[st], (n >> 1) & 1);
    const unsigned char* rows = stage + ((size_t)st * TJ + warp * 16) * pitch;  // this warp's 16 rows
    // statistics: lanes 2r, 2r+1 sum the two halves of row r
    float sx = 0.f, sxx = 0.f;
    {
      const int r = lane / 2, half = lane % 2;
      const uint4* p = (const uint4*)(rows + (size_t)r * pitch + half * C);
      for (int c8 = 0; c8 < C / 16; ++c8) {
        const uint4 u = p[c8];
        const T* e = (const T*)&u;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float x = evo::to_f(e[k]);
          sx += x;
          sxx = fmaf(x, x, sxx);
        }
      }
      sx += __shfl_xor_sync(0xffffffffu, sx, 1);
      sxx += __shfl_xor_sync(0xffffffffu, sxx, 1);
    }
    // the MMA: A fragments straight from the staged rows (a0: row g, k 2q..; a1: row g + 8; a2, a3: k + 8)
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
    {
      const int g = lane / 4, q = lane % 4;
      const unsigned char* r0 = rows + (size_t)g * pitch + 4 * q;
      const unsigned char* r8 = rows + (size_t)(g + 8) * pitch + 4 * q;
#pragma unroll
      for (int ks = 0; ks < KMAX; ++ks) {
        if (ks < KS) {
          const uint32_t a0 = *(const uint32_t*)(r0 + ks * 32), a1 = *(const uint32_t*)(r8 + ks * 32);
          const uint32_t a2 = *(const uint32_t*)(r0 + ks * 32 + 16), a3 = *(const uint32_t*)(r8 + ks * 32 + 16);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (std::is_same<T, __half>::value)
              asm volatile(
                  "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                  "{%0,%1,%2,%3};"
                  : "+f"(acc[nt][0]), "+f"(acc[nt][1]), "+f"(acc[nt][2]), "+f"(acc[nt][3])
                  : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bf[ks][nt][0]), "r"(bf[ks][nt][1]));
            else
              asm volatile(
                  "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                  "{%0,%1,%2,%3};"
                  : "+f"(acc[nt][0]), "+f"(acc[nt][1]), "+f"(acc[nt][2]), "+f"(acc[nt][3])
                  : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bf[ks][nt][0]), "r"(bf[ks][nt][1]));
          }
        }
      }
    }
    __syncthreads();  // stage st read by every warp; the previous tile's outputs written
    if (warp == 0 && tix + 2 * (int)gridDim.x < ntiles) issue(tix + 2 * gridDim.x, st);
    // epilogue: rows g and g + 8 of the warp's 16, heads nt * 8 + 2q, + 1
    {
      const int g = lane / 4, q = lane % 4;
      const float sx0 = __shfl_sync(0xffffffffu, sx, 2 * g), sxx0 = __shfl_sync(0xffffffffu, sxx, 2 * g);
      const float sx8 = __shfl_sync(0xffffffffu, sx, 2 * (g + 8)), sxx8 = __shfl_sync(0xffffffffu, sxx, 2 * (g + 8));
      const float m0 = sx0 * invC, m8 = sx8 * invC;
      const float rs0 = rsqrtf(fmaxf(sxx0 * invC - m0 * m0, 0.f) + eps);
      const float rs8 = rsqrtf(fmaxf(sxx8 * invC - m8 * m8, 0.f) + eps);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int h = nt * 8 + 2 * q + e;
          tile[h][warp * 16 + g] = rs0 * (acc[nt][e] - m0 * s1s[h]) + s2s[h];
          tile[h][warp * 16 + g + 8] = rs8 * (acc[nt][2 + e] - m8 * s1s[h]) + s2s[h];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < H * TJ; t += blockDim.x) {
      const int h = t / TJ, jo = t % TJ, j = jt * TJ + jo;
      if (j < L) out[(((size_t)b * H + h) * L + i) * L + j] = evo::from_f<T>(tile[h][jo]);
    }
  }
}

// Per CTA (grid-stride over the (b, i, j-tile) tiles): dz rows, and this CTA's partial sums of
// dW[c][h] = sum y_c g_h, dgamma_c = sum dy_c xhat_c, dbeta_c = sum dy_c into part[blockIdx.x].
template <typename T, typename G, int CPL, int HM>
__global__ void __launch_bounds__(kWarps * 32, 2) pair_bias_bwd_kernel(const G* __restrict__ dbias, const T* __restrict__ z,
                                                                    const float* __restrict__ gam,
                                                                    const float* __restrict__ bet,
                                                                    const float* __restrict__ w, T* __restrict__ dz,
                                                                    float* __restrict__ part, int Bo, int L, int C,
                                                                    int H, float eps) {
  __shared__ float gt[HM][kTileJ];
  extern __shared__ float dyn[];
  float* ws = dyn;                      // CPL * HM * 32: W, lane-contiguous
  float* red = dyn + CPL * HM * 32;     // CPL * (HM + 2) * 32: the CTA's partial sums, warps added in order
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c0 = lane * CPL;
  const float invC = 1.f / (float)C;
  const int nj = (L + kTileJ - 1) / kTileJ;
  const long long ntiles = (long long)Bo * L * nj;
  stage_w<CPL, HM>(w, ws, H);
  float g[CPL], be[CPL], dw[CPL][HM], dg[CPL], db[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    g[k] = gam[c0 + k];
    be[k] = bet[c0 + k];
    dg[k] = db[k] = 0.f;
#pragma unroll
    for (int h = 0; h < HM; ++h) dw[k][h] = 0.f;
  }
  // the warp's rows of z: the next tile's loaded while this one is processed
  auto load_tile = [&](long long tx, float (*xr)[CPL]) {
    const int jt = (int)(tx % nj), i = (int)((tx / nj) % L), b = (int)(tx / ((long long)nj * L));
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      const int j = min(jt * kTileJ + warp * kRowsPerWarp + r, L - 1);
      load_row<T, CPL>(z + (((size_t)b * L + i) * L + j) * C + c0, xr[r]);
    }
  };
  float xn[kRowsPerWarp][CPL];
  if (blockIdx.x < ntiles) load_tile(blockIdx.x, xn);
  for (long long tix = blockIdx.x; tix < ntiles; tix += gridDim.x) {
    const int t32 = (int)tix, jt = t32 % nj, i = (t32 / nj) % L, b = t32 / (nj * L);
    float x[kRowsPerWarp][CPL];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r)
#pragma unroll
      for (int k = 0; k < CPL; ++k) x[r][k] = xn[r][k];
    if (tix + gridDim.x < ntiles) load_tile(tix + gridDim.x, xn);
    __syncthreads();  // the previous tile's gradient rows were read (and W staged)
    for (int t = threadIdx.x; t < H * kTileJ; t += blockDim.x) {
      const int h = t / kTileJ, jj = t % kTileJ, j = jt * kTileJ + jj;
      gt[h][jj] = j < L ? evo::to_f(dbias[(((size_t)b * H + h) * L + i) * L + j]) : 0.f;
    }
    float mean[kRowsPerWarp], rstd[kRowsPerWarp], dxs[kRowsPerWarp][CPL];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      float sm = 0.f;
#pragma unroll
      for (int k = 0; k < CPL; ++k) sm += x[r][k];
      mean[r] = sm;
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) mean[r] = warp_sum(mean[r]) * invC;
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      float v = 0.f;
#pragma unroll
      for (int k = 0; k < CPL; ++k) v += (x[r][k] - mean[r]) * (x[r][k] - mean[r]);
      rstd[r] = v;
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) rstd[r] = rsqrtf(warp_sum(rstd[r]) * invC + eps);
    __syncthreads();  // dBias2 rows staged
    float gh[kRowsPerWarp][HM], s1[kRowsPerWarp], s2[kRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      const int jj = warp * kRowsPerWarp + r;
      const bool valid = jt * kTileJ + jj < L;  // rows past L (clamped loads) contribute nothing
#pragma unroll
      for (int h = 0; h < HM; ++h) gh[r][h] = h < H && valid ? gt[h][jj] : 0.f;
#pragma unroll
      for (int k = 0; k < CPL; ++k) x[r][k] = (x[r][k] - mean[r]) * rstd[r];  // xhat
      s1[r] = s2[r] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      float dy[kRowsPerWarp];
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) dy[r] = 0.f;
#pragma unroll
      for (int h = 0; h < HM; ++h) {
        const float wv = ws[(k * HM + h) * 32 + lane];
        float dwa = dw[k][h];
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r) {
          dy[r] = fmaf(wv, gh[r][h], dy[r]);
          dwa = fmaf(x[r][k] * g[k] + be[k], gh[r][h], dwa);
        }
        dw[k][h] = dwa;
      }
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) {
        const float xh = x[r][k];
        dg[k] = fmaf(dy[r], xh, dg[k]);
        db[k] += dy[r];
        const float dxh = dy[r] * g[k];
        s1[r] += dxh;
        s2[r] += dxh * xh;
        dy[r] = dxh;
      }
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) dxs[r][k] = dy[r];
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      s1[r] = warp_sum(s1[r]) * invC;
      s2[r] = warp_sum(s2[r]) * invC;
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      const int j = jt * kTileJ + warp * kRowsPerWarp + r;
      if (j < L) {
        // dz = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat))
        float dzr[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) dzr[k] = rstd[r] * (dxs[r][k] - s1[r] - x[r][k] * s2[r]);
        store_row<T, CPL>(dz + (((size_t)b * L + i) * L + j) * C + c0, dzr);
      }
    }
  }
  // the CTA's partial sums: warps add their values in order (deterministic) into a lane-contiguous
  // (conflict-free) layout red[(k * (HM + 2) + e) * 32 + lane], e < HM: dW, HM: dgamma, HM + 1: dbeta;
  // then one row of `part` in the (dW[c][h], dgamma[c], dbeta[c]) order
  const int nv = C * H + 2 * C;
  for (int t = threadIdx.x; t < CPL * (HM + 2) * 32; t += blockDim.x) red[t] = 0.f;
  for (int wv = 0; wv < kWarps; ++wv) {
    __syncthreads();
    if (warp == wv) {
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
#pragma unroll
        for (int h = 0; h < HM; ++h) red[(k * (HM + 2) + h) * 32 + lane] += dw[k][h];
        red[(k * (HM + 2) + HM) * 32 + lane] += dg[k];
        red[(k * (HM + 2) + HM + 1) * 32 + lane] += db[k];
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nv; t += blockDim.x) {
    int c, e;
    if (t < C * H) { c = t / H; e = t % H; }
    else if (t < C * H + C) { c = t - C * H; e = HM; }
    else { c = t - C * H - C; e = HM + 1; }
    part[(size_t)blockIdx.x * nv + t] = red[((c % CPL) * (HM + 2) + e) * 32 + c / CPL];
  }
}

// out[v] = sum of the np CTA partials of value v (v < C*H: dW, then dgamma, dbeta) in a fixed order:
// a CTA owns 32 values; its 8 warps sum partials k = w, w + 8, ... (coalesced rows of 32 values), then
// warp 0 adds the 8 warp sums in order — deterministic, and every partial row is read once
__global__ void pair_bias_reduce_kernel(const float* __restrict__ part, int np, int nv, int CH, int C,
                                        float* __restrict__ dw, float* __restrict__ dg, float* __restrict__ db) {
  __shared__ float ws8[8][32];
  const int lane = threadIdx.x % 32, wv = threadIdx.x / 32, v = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (v < nv)
    for (int k = wv; k < np; k += 8) s += part[(size_t)k * nv + v];
  ws8[wv][lane] = s;
  __syncthreads();
  if (wv == 0 && v < nv) {
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += ws8[q][lane];
    if (v < CH) dw[v] = t;
    else if (v < CH + C) dg[v - CH] = t;
    else db[v - CH - C] = t;
  }
}

evo_status check(const evo_pair_bias_desc* d) {
  if (!d) {
    evo::set_last_error("null descriptor");
    return EVO_ERR_USAGE;
  }
  if (d->Bo < 1 || d->L < 1 || d->C < 1 || d->H < 1) {
    evo::set_last_error("extents must be >= 1 (Bo, L, C, H)");
    return EVO_ERR_VALIDATION;
  }
  if (d->dtype != EVO_BF16 && d->dtype != EVO_F16) {
    evo::set_last_error("z must be bf16 or f16");
    return EVO_ERR_VALIDATION;
  }
  if (d->dbias_dtype != EVO_F32 && d->dbias_dtype != d->dtype) {
    evo::set_last_error("dbias_dtype must be EVO_F32 or equal to dtype");
    return EVO_ERR_VALIDATION;
  }
  if (!(d->eps > 0.f) || !std::isfinite(d->eps)) {
    evo::set_last_error("eps must be finite and > 0");
    return EVO_ERR_NUMERIC;
  }
  if (d->Bo * d->L * d->L >= (1LL << 31)) {  // 32-bit tile / row indices
    evo::set_last_error("pair-bias projection: Bo * L * L must be < 2^31");
    return EVO_ERR_UNSUPPORTED;
  }
  if (d->C % 32 != 0 || d->C > 256 || d->H > 16) {
    evo::set_last_error("pair-bias projection supports c_z in {32, 64, ..., 256} and H <= 16");
    return EVO_ERR_UNSUPPORTED;
  }
  return EVO_OK;
}

// persistent grids: up to 8 CTAs per SM walk the (b, i, j-tile) tiles
unsigned grid_of(const evo_pair_bias_desc* d) {
  const long long nj = (d->L + kTileJ - 1) / kTileJ, ntiles = d->Bo * d->L * nj;
  return (unsigned)std::min<long long>(ntiles, 148LL * 8);
}
unsigned bwd_grid(const evo_pair_bias_desc* d) {  // one wave at the backward's 2 CTAs per SM: fewer partials
  const long long nj = (d->L + kTileJ - 1) / kTileJ, ntiles = d->Bo * d->L * nj;
  return (unsigned)std::min<long long>(ntiles, 148LL * 2);
}

#ifndef EVO_PB_FR
#define EVO_PB_FR 4  // forward rows per warp (a CTA covers 8 * EVO_PB_FR consecutive j)
#endif
#ifndef EVO_PB_MMA_CTAS
#define EVO_PB_MMA_CTAS 8  // resident CTAs per SM of the tensor-pipe forward, at most (persistent)
#endif
#ifndef EVO_PB_MMA
#define EVO_PB_MMA 1  // forward on the tensor pipe (mma.sync), else the shuffle-reduction kernel
#endif
template <typename T, int CPL, int HM>
void launch_fwd(const evo_pair_bias_desc* d, const void* z, const float* g, const float* b, const float* w, void* out,
                cudaStream_t st) {
  if (EVO_PB_MMA) {
    auto kern = pair_bias_fwd_mma_kernel<T, HM>;
    const size_t shm = 2 * 64 * ((size_t)d->C * 2 + 16);
    static int set = 0;
    if ((int)shm > set) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
      set = (int)shm;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, shm);
    const long long ntiles = d->Bo * d->L * ((d->L + 63) / 64);
    // resident CTAs per SM: up to the occupancy limit, but >= ~4 tiles per CTA (the prologue builds the
    // weight fragments) and <= EVO_PB_MMA_CTAS
    const long long want = std::max<long long>(2, std::min<long long>(EVO_PB_MMA_CTAS, ntiles / (148LL * 4)));
    const unsigned grid = (unsigned)std::min<long long>(ntiles, 148LL * std::min<long long>(std::max(per_sm, 1), want));
    kern<<<grid, 128, shm, st>>>((const T*)z, g, b, w, (T*)out, (int)d->Bo, (int)d->L, (int)d->C, (int)d->H, d->eps);
    return;
  }
  constexpr int FR = EVO_PB_FR;
  auto kern = pair_bias_fwd_kernel<T, CPL, HM, FR>;
  const size_t shm = (size_t)CPL * HM * 32 * 4 + 2 * (size_t)kWarps * FR * d->C * sizeof(T);
  static int shm_set = 0;  // dynamic + static shared memory past 48 KB needs the opt-in
  if ((int)shm > shm_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    shm_set = (int)shm;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, shm);
  const long long nj = (d->L + kWarps * FR - 1) / (kWarps * FR), ntiles = d->Bo * d->L * nj;
  const unsigned grid = (unsigned)std::min<long long>(ntiles, 148LL * std::max(per_sm, 1));  // one wave
  kern<<<grid, kWarps * 32, shm, st>>>((const T*)z, g, b, w, (T*)out, (int)d->Bo, (int)d->L, (int)d->C, (int)d->H,
                                       d->eps);
}

template <typename T, int CPL, int HM>
void launch_bwd(const evo_pair_bias_desc* d, const void* dbias, const void* z, const float* g, const float* b,
                const float* w, void* dz, float* part, cudaStream_t st) {
  const size_t shm = ((size_t)CPL * HM * 32 + (size_t)CPL * (HM + 2) * 32) * 4;
  if (d->dbias_dtype == EVO_F32)
    pair_bias_bwd_kernel<T, float, CPL, HM><<<bwd_grid(d), kWarps * 32, shm, st>>>(
        (const float*)dbias, (const T*)z, g, b, w, (T*)dz, part, (int)d->Bo, (int)d->L, (int)d->C, (int)d->H, d->eps);
  else
    pair_bias_bwd_kernel<T, T, CPL, HM><<<bwd_grid(d), kWarps * 32, shm, st>>>(
        (const T*)dbias, (const T*)z, g, b, w, (T*)dz, part, (int)d->Bo, (int)d->L, (int)d->C, (int)d->H, d->eps);
}

// dispatch over (dtype, channels per lane, head bound)
template <template <typename, int, int> class F, typename... A>
void dispatch(const evo_pair_bias_desc* d, A... a) {
  const int cpl = (int)(d->C / 32);
  auto by_h = [&](auto t, auto c) {
    using T = decltype(t);
    constexpr int CPL = decltype(c)::value;
    if (d->H <= 8) F<T, CPL, 8>::run(d, a...);
    else F<T, CPL, 16>::run(d, a...);
  };
  auto by_c = [&](auto t) {
    switch (cpl) {
      case 1: by_h(t, std::integral_constant<int, 1>{}); break;
      case 2: by_h(t, std::integral_constant<int, 2>{}); break;
      case 4: by_h(t, std::integral_constant<int, 4>{}); break;
      case 8: by_h(t, std::integral_constant<int, 8>{}); break;
      default: break;
    }
  };
  if (d->dtype == EVO_BF16) by_c(__nv_bfloat16{});
  else by_c(__half{});
}

template <typename T, int CPL, int HM>
struct FwdOp {
  static void run(const evo_pair_bias_desc* d, const void* z, const float* g, const float* b, const float* w,
                  void* out, cudaStream_t st) {
    launch_fwd<T, CPL, HM>(d, z, g, b, w, out, st);
  }
};
template <typename T, int CPL, int HM>
struct BwdOp {
  static void run(const evo_pair_bias_desc* d, const void* dbias, const void* z, const float* g, const float* b,
                  const float* w, void* dz, float* part, cudaStream_t st) {
    launch_bwd<T, CPL, HM>(d, dbias, z, g, b, w, dz, part, st);
  }
};

evo_status cuda_status() {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return EVO_OK;
  evo::set_last_error(cudaGetErrorString(e));
  return EVO_ERR_CUDA;
}

}  // namespace

extern "C" evo_status evo_pair_bias_fwd(const evo_pair_bias_desc* d, const void* z, const float* ln_w,
                                        const float* ln_b, const float* w, void* bias2, evo_stream_t stream) {
  if (evo_status st = check(d)) return st;
  if (!z || !ln_w || !ln_b || !w || !bias2) {
    evo::set_last_error("null tensor pointer");
    return EVO_ERR_VALIDATION;
  }
  dispatch<FwdOp>(d, z, ln_w, ln_b, w, bias2, (cudaStream_t)stream);
  return cuda_status();
}

extern "C" size_t evo_pair_bias_bwd_workspace_size(const evo_pair_bias_desc* d) {
  if (check(d) != EVO_OK) return 0;
  return (size_t)bwd_grid(d) * (size_t)(d->C * d->H + 2 * d->C) * 4;
}

extern "C" evo_status evo_pair_bias_bwd(const evo_pair_bias_desc* d, const void* dbias2, const void* z,
                                        const float* ln_w, const float* ln_b, const float* w, void* dz,
                                        float* dln_w, float* dln_b, float* dw, void* workspace, size_t ws_bytes,
                                        evo_stream_t stream) {
  if (evo_status st = check(d)) return st;
  if (!dbias2 || !z || !ln_w || !ln_b || !w || !dz || !dln_w || !dln_b || !dw) {
    evo::set_last_error("null tensor pointer");
    return EVO_ERR_VALIDATION;
  }
  if (!workspace || ws_bytes < evo_pair_bias_bwd_workspace_size(d)) {
    evo::set_last_error("workspace smaller than evo_pair_bias_bwd_workspace_size");
    return EVO_ERR_VALIDATION;
  }
  cudaStream_t st = (cudaStream_t)stream;
  float* part = (float*)workspace;
  dispatch<BwdOp>(d, dbias2, z, ln_w, ln_b, w, dz, part, st);
  const int nv = (int)(d->C * d->H + 2 * d->C);
  pair_bias_reduce_kernel<<<(nv + 31) / 32, 256, 0, st>>>(part, (int)bwd_grid(d), nv, (int)(d->C * d->H),
                                                            (int)d->C, dw, dln_w, dln_b);
  return cuda_status();
}

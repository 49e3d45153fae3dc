// simt_kernels.cuh — K5: FFMA (CUDA-core) forward/backward Evoformer attention.
//
// The fp32 path (TF32 would miss the 1e-4 parity bar) and the
// envelope outside the tcgen05 kernels (D not a multiple of 16, D < 16).
// Semantics: /root/reference/proj/core/src/attention_tiled.cpp
//   forward  :57-180  online softmax over key tiles, O = acc / l, LSE = m + ln l
//   backward :182-340 P recomputed from LSE, delta = rowsum(dO*O),
//                     dS = P (dP - delta), dQ/dK scaled once, dBias = sum_b dS
// plus the bias1 (mask) term of DS4Sci_EvoformerAttention. Softmax runs in the
// log2 domain (ex2.approx) with fp32 accumulation everywhere.
#pragma once
#include "common.cuh"

namespace evo {
namespace simt {

// Rows per CTA (one per thread) and staged key tile; halved for D = 64 so the fp32 staging
// buffers stay inside 48 KB of static shared memory.
template <int DP>
struct Tiles {
  static constexpr int kRows = DP <= 32 ? 64 : 32;  // query (fwd, dQ) or key (dK/dV) rows per CTA
  static constexpr int kKeyTile = DP <= 32 ? 64 : 32;
};
constexpr int kQTile = 32;

// ---------------------------------------------------------------- forward
template <typename T, int DP>
__global__ void __launch_bounds__(Tiles<DP>::kRows) fwd_kernel(Shape s, const T* __restrict__ q,
                                                    const T* __restrict__ k,
                                                    const T* __restrict__ v, T* __restrict__ o,
                                                    float* __restrict__ lse) {
  constexpr int kRows = Tiles<DP>::kRows, kKeyTile = Tiles<DP>::kKeyTile;
  __shared__ float ks[kKeyTile][DP + 1];
  __shared__ float vs[kKeyTile][DP + 1];
  __shared__ float b1s[kKeyTile];
  const int tid = threadIdx.x;
  const int i = blockIdx.x * kRows + tid;
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const bool valid = i < s.L;
  const int ob = b / s.N;
  const T* b1 = static_cast<const T*>(s.bias1);
  const T* b2row = (s.bias2 && valid)
                       ? static_cast<const T*>(s.bias2) + (((size_t)ob * s.H + h) * s.L + i) * s.L
                       : nullptr;

  float qr[DP], acc[DP];
#pragma unroll
  for (int d = 0; d < DP; ++d) {
    qr[d] = (valid && d < s.D) ? to_f(q[row_off(s, b, i, h) + d]) : 0.f;
    acc[d] = 0.f;
  }
  float m = -INFINITY, l = 0.f;

  for (int j0 = 0; j0 < s.L; j0 += kKeyTile) {
    __syncthreads();
    for (int x = tid; x < kKeyTile * DP; x += kRows) {
      const int jj = x / DP, d = x % DP, j = j0 + jj;
      const bool in = j < s.L && d < s.D;
      ks[jj][d] = in ? to_f(k[row_off(s, b, j, h) + d]) : 0.f;
      vs[jj][d] = in ? to_f(v[row_off(s, b, j, h) + d]) : 0.f;
    }
    for (int jj = tid; jj < kKeyTile; jj += kRows) {
      const int j = j0 + jj;
      b1s[jj] = (b1 && j < s.L) ? to_f(b1[(size_t)b * s.L + j]) * kLog2e : 0.f;
    }
    __syncthreads();
    if (!valid) continue;
    const int jn = min(kKeyTile, s.L - j0);
    for (int c0 = 0; c0 < jn; c0 += 16) {
      float x[16];
      float mx = m;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int jj = c0 + t;
        float val = -INFINITY;
        if (jj < jn) {
          float dot = 0.f;
#pragma unroll
          for (int d = 0; d < DP; ++d) dot = fmaf(qr[d], ks[jj][d], dot);
          val = fmaf(dot, s.scale_log2, b1s[jj]);
          if (b2row) val = fmaf(to_f(b2row[j0 + jj]), kLog2e, val);
        }
        x[t] = val;
        mx = fmaxf(mx, val);
      }
      const float base = mx == -INFINITY ? 0.f : mx;
      const float alpha = ex2(m - base);
      l *= alpha;
#pragma unroll
      for (int d = 0; d < DP; ++d) acc[d] *= alpha;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float p = ex2(x[t] - base);
        l += p;
        const int jj = c0 + t < kKeyTile ? c0 + t : kKeyTile - 1;
#pragma unroll
        for (int d = 0; d < DP; ++d) acc[d] = fmaf(p, vs[jj][d], acc[d]);
      }
      m = mx;
    }
  }
  if (!valid) return;
  const float inv = l > 0.f ? 1.f / l : 0.f;
  T* orow = o + row_off(s, b, i, h);
  const T* grow = s.gate ? static_cast<const T*>(s.gate) + row_off(s, b, i, h) : nullptr;
  bool nan = false;
#pragma unroll
  for (int d = 0; d < DP; ++d)
    if (d < s.D) {
      // fused output gate (OpenFold): o = sigmoid(G) * O
      orow[d] = from_f<T>(acc[d] * inv * (grow ? sigmoidf_fast(to_f(grow[d])) : 1.f));
      nan |= isnan(acc[d]);
    }
  const float lv = l > 0.f ? (m + __log2f(l)) * kLn2 : -INFINITY;
  lse[((size_t)b * s.H + h) * s.L + i] = lv;
  flag_if(s.flag, nan || !isfinite(lv));
}

// ------------------------------------------------------- backward: delta
// delta[b,h,i] = sum_d dO*O (attention_tiled.cpp:227-241), fp32.
template <typename T>
__global__ void delta_kernel(Shape s, const T* __restrict__ dout, const T* __restrict__ o,
                             float* __restrict__ delta) {
  const size_t rows = (size_t)s.B * s.L * s.H;
  for (size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x; r < rows;
       r += (size_t)gridDim.x * blockDim.x) {
    // r enumerates (b, i, h); delta is stored (b, h, i)
    const int h = (int)(r % s.H);
    const size_t bi = r / s.H;
    const int i = (int)(bi % s.L);
    const size_t b = bi / s.L;
    const T* a = dout + row_off(s, (int)b, i, h);
    const T* c = o + row_off(s, (int)b, i, h);
    float acc = 0.f;
    for (int d = 0; d < s.D; ++d) acc = fmaf(to_f(a[d]), to_f(c[d]), acc);
    delta[(b * s.H + h) * s.L + i] = acc;
    flag_if(s.flag, !isfinite(acc));  // NaN in dO (attention_tiled.cpp:209) or O
  }
}

// ------------------------------------------- backward of the fused output gate
// With o = sigmoid(G) * O saved by the forward and dout the gradient of o: the attention backward
// takes dO = dout * sigmoid(G) (written to dog), dG = dout * o * (1 - sigmoid(G)), and
// delta = sum_d dO * O = sum_d dout * o (the gate cancels), so no ungated O is ever needed.
template <typename T>
__global__ void gate_bwd_kernel(size_t n, const T* __restrict__ dout, const T* __restrict__ o,
                                const T* __restrict__ gate, T* __restrict__ dog, T* __restrict__ dgate) {
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n; x += (size_t)gridDim.x * blockDim.x) {
    const float sg = sigmoidf_fast(to_f(gate[x])), g = to_f(dout[x]);
    dog[x] = from_f<T>(g * sg);
    dgate[x] = from_f<T>(g * to_f(o[x]) * (1.f - sg));
  }
}

// ------------------------------------------- backward: dK, dV, dBias (key side)
template <typename T, int DP>
__global__ void __launch_bounds__(Tiles<DP>::kRows) dkdv_kernel(
    Shape s, const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
    const T* __restrict__ dout, const float* __restrict__ lse, const float* __restrict__ delta,
    T* __restrict__ dk, T* __restrict__ dv, int b0, float* __restrict__ db1_part, float* __restrict__ db2_part) {
  // Rows [b0, b0 + gridDim.z) of one outer batch. dBias2 is not added with atomics: every (row, i, j)
  // term dS is stored once into the row's partial plane db2_part[b - b0][h] (rows of a launch are
  // never reduced concurrently), and ordered_sum_kernel adds the planes in ascending row order into
  // the fp32 accumulator — attention_tiled.cpp:246-252, 318-323 with the deterministic (ascending b)
  // policy. dBias1 partials per head: db1_part[h][b - b0][j], summed over h in order.
  constexpr int kRows = Tiles<DP>::kRows;
  __shared__ float kv[2][kRows][DP + 1];
  __shared__ float qs[kQTile][DP];
  __shared__ float dos[kQTile][DP];
  __shared__ float ls[kQTile], dls[kQTile];
  const int tid = threadIdx.x;
  const int j = blockIdx.x * kRows + tid;
  const int h = blockIdx.y;
  const int b = b0 + blockIdx.z;
  const bool valid = j < s.L;
  const int ob = b / s.N;
  for (int x = tid; x < kRows * DP; x += kRows) {
    const int jj = x / DP, d = x % DP, jr = blockIdx.x * kRows + jj;
    const bool in = jr < s.L && d < s.D;
    kv[0][jj][d] = in ? to_f(k[row_off(s, b, jr, h) + d]) : 0.f;
    kv[1][jj][d] = in ? to_f(v[row_off(s, b, jr, h) + d]) : 0.f;
  }
  const float b1j = (s.bias1 && valid) ? to_f(static_cast<const T*>(s.bias1)[(size_t)b * s.L + j]) * kLog2e : 0.f;
  const T* b2 = s.bias2 ? static_cast<const T*>(s.bias2) + ((size_t)ob * s.H + h) * s.L * s.L : nullptr;
  float* db2 = db2_part ? db2_part + ((size_t)blockIdx.z * s.H + h) * s.L * s.L : nullptr;
  float dka[DP], dva[DP];
#pragma unroll
  for (int d = 0; d < DP; ++d) dka[d] = dva[d] = 0.f;
  float db1 = 0.f;

  for (int i0 = 0; i0 < s.L; i0 += kQTile) {
    __syncthreads();
    for (int x = tid; x < kQTile * DP; x += kRows) {
      const int ii = x / DP, d = x % DP, i = i0 + ii;
      const bool in = i < s.L && d < s.D;
      qs[ii][d] = in ? to_f(q[row_off(s, b, i, h) + d]) : 0.f;
      dos[ii][d] = in ? to_f(dout[row_off(s, b, i, h) + d]) : 0.f;
    }
    for (int ii = tid; ii < kQTile; ii += kRows) {
      const int i = i0 + ii;
      const float lv = i < s.L ? lse[((size_t)b * s.H + h) * s.L + i] : -INFINITY;
      ls[ii] = lv * kLog2e;
      dls[ii] = i < s.L ? delta[((size_t)b * s.H + h) * s.L + i] : 0.f;
    }
    __syncthreads();
    if (!valid) continue;
    const int in_ = min(kQTile, s.L - i0);
    for (int ii = 0; ii < in_; ++ii) {
      const int i = i0 + ii;
      float dot = 0.f, dp = 0.f;
#pragma unroll
      for (int d = 0; d < DP; ++d) {
        dot = fmaf(qs[ii][d], kv[0][tid][d], dot);
        dp = fmaf(dos[ii][d], kv[1][tid][d], dp);
      }
      float x = fmaf(dot, s.scale_log2, b1j);
      if (b2) x = fmaf(to_f(b2[(size_t)i * s.L + j]), kLog2e, x);
      const float p = ls[ii] == -INFINITY ? 0.f : ex2(x - ls[ii]);
      const float ds = p * (dp - dls[ii]);
#pragma unroll
      for (int d = 0; d < DP; ++d) {
        dva[d] = fmaf(p, dos[ii][d], dva[d]);
        dka[d] = fmaf(ds, qs[ii][d], dka[d]);
      }
      db1 += ds;
      if (db2) db2[(size_t)i * s.L + j] = ds;
    }
  }
  if (!valid) return;
  T* dkr = dk + row_off(s, b, j, h);
  T* dvr = dv + row_off(s, b, j, h);
  bool nan = false;
#pragma unroll
  for (int d = 0; d < DP; ++d)
    if (d < s.D) {
      dkr[d] = from_f<T>(dka[d] * s.scale);
      dvr[d] = from_f<T>(dva[d]);
      nan |= isnan(dka[d]) || isnan(dva[d]);
    }
  flag_if(s.flag, nan);
  if (db1_part) db1_part[((size_t)h * gridDim.z + blockIdx.z) * s.L + j] = db1;
}

// ------------------------------------------------- backward: dQ (query side)
template <typename T, int DP>
__global__ void __launch_bounds__(Tiles<DP>::kRows) dq_kernel(
    Shape s, const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
    const T* __restrict__ dout, const float* __restrict__ lse, const float* __restrict__ delta,
    T* __restrict__ dq, int b0) {
  constexpr int kRows = Tiles<DP>::kRows, kKeyTile = Tiles<DP>::kKeyTile;
  __shared__ float ks[kKeyTile][DP];
  __shared__ float vs[kKeyTile][DP];
  __shared__ float b1s[kKeyTile];
  __shared__ float own[2][kRows][DP + 1];
  const int tid = threadIdx.x;
  const int i = blockIdx.x * kRows + tid;
  const int h = blockIdx.y;
  const int b = b0 + blockIdx.z;
  const bool valid = i < s.L;
  const int ob = b / s.N;
  for (int x = tid; x < kRows * DP; x += kRows) {
    const int ii = x / DP, d = x % DP, ir = blockIdx.x * kRows + ii;
    const bool in = ir < s.L && d < s.D;
    own[0][ii][d] = in ? to_f(q[row_off(s, b, ir, h) + d]) : 0.f;
    own[1][ii][d] = in ? to_f(dout[row_off(s, b, ir, h) + d]) : 0.f;
  }
  const float l2 = valid ? lse[((size_t)b * s.H + h) * s.L + i] * kLog2e : -INFINITY;
  const float dl = valid ? delta[((size_t)b * s.H + h) * s.L + i] : 0.f;
  const T* b2row = (s.bias2 && valid)
                       ? static_cast<const T*>(s.bias2) + (((size_t)ob * s.H + h) * s.L + i) * s.L
                       : nullptr;
  const T* b1 = static_cast<const T*>(s.bias1);
  float dqa[DP];
#pragma unroll
  for (int d = 0; d < DP; ++d) dqa[d] = 0.f;
  for (int j0 = 0; j0 < s.L; j0 += kKeyTile) {
    __syncthreads();
    for (int x = tid; x < kKeyTile * DP; x += kRows) {
      const int jj = x / DP, d = x % DP, j = j0 + jj;
      const bool in = j < s.L && d < s.D;
      ks[jj][d] = in ? to_f(k[row_off(s, b, j, h) + d]) : 0.f;
      vs[jj][d] = in ? to_f(v[row_off(s, b, j, h) + d]) : 0.f;
    }
    for (int jj = tid; jj < kKeyTile; jj += kRows) {
      const int j = j0 + jj;
      b1s[jj] = (b1 && j < s.L) ? to_f(b1[(size_t)b * s.L + j]) * kLog2e : 0.f;
    }
    __syncthreads();
    if (!valid || l2 == -INFINITY) continue;
    const int jn = min(kKeyTile, s.L - j0);
    for (int jj = 0; jj < jn; ++jj) {
      float dot = 0.f, dp = 0.f;
#pragma unroll
      for (int d = 0; d < DP; ++d) {
        dot = fmaf(own[0][tid][d], ks[jj][d], dot);
        dp = fmaf(own[1][tid][d], vs[jj][d], dp);
      }
      float x = fmaf(dot, s.scale_log2, b1s[jj]);
      if (b2row) x = fmaf(to_f(b2row[j0 + jj]), kLog2e, x);
      const float ds = ex2(x - l2) * (dp - dl);
#pragma unroll
      for (int d = 0; d < DP; ++d) dqa[d] = fmaf(ds, ks[jj][d], dqa[d]);
    }
  }
  if (!valid) return;
  T* r = dq + row_off(s, b, i, h);
  bool nan = false;
#pragma unroll
  for (int d = 0; d < DP; ++d)
    if (d < s.D) {
      r[d] = from_f<T>(dqa[d] * s.scale);
      nan |= isnan(dqa[d]);
    }
  flag_if(s.flag, nan);
}

}  // namespace simt

// fp32 -> T conversion of the reduced bias gradients (the paper's separate
// convert-back kernel), optionally accumulating.
template <typename T>
__global__ void convert_kernel(const float* __restrict__ src, T* __restrict__ dst, size_t n) {
  for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n;
       x += (size_t)gridDim.x * blockDim.x)
    dst[x] = from_f<T>(src[x]);
}

}  // namespace evo

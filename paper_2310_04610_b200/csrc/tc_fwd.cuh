// tc_fwd.cuh — K1: fused Evoformer attention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Reference semantics: attn_forward_tiled, /root/reference/proj/core/src/attention_tiled.cpp:57-180
// (S = scale*QK^T + bias, online softmax over key tiles, O = acc/l, LSE = m + ln l), plus the
// DS4Sci mask bias1[b, j]. Layout and schedule are B200-first:
//
//  * persistent CTAs (one per SM) walk a contiguous range of (ob, h, q-tile, row) work items,
//    rows innermost, so one CTA keeps the pair-bias row block bias2[ob, h, q-tile, :] resident in
//    shared memory (TMA, 128B swizzle) and reuses it for every MSA row it processes — the bias is
//    read from L2 once per CTA instead of once per row (the paper's on-the-fly broadcast).
//  * warp 0: TMA producer (Q per row, K/V per key tile through a 3-stage ring).
//    warp 1: single-thread tcgen05.mma issuer: S = Q K^T (SS, K-major) into a double-buffered
//            128x128 fp32 TMEM tile; O_j = P_j V_j (TS: P read from TMEM, V MN-major) into a
//            double-buffered 128xD fp32 TMEM tile.
//    warps 2-5: softmax warpgroup, one thread per query row (TMEM lane): S -> registers,
//            bias1/bias2 add, online max/sum in the log2 domain (ex2.approx), P (bf16) written
//            back into the S columns (FA4-style aliasing), per-tile O_j folded into a register
//            accumulator with the running rescale factor; epilogue writes O and LSE.
#pragma once
#include "common.cuh"
#include "tc_ptx.cuh"

namespace evo {
namespace tc {

constexpr int kBM = 128;   // query rows per tile (UMMA M, TMEM lanes)
constexpr int kBN = 128;   // keys per tile (UMMA N of S)
constexpr int kFwdThreads = 192;

// bias2 delivery
enum BiasMode : int { kBiasNone = 0, kBiasResident = 1, kBiasStreamed = 2, kBiasGlobal = 3 };

struct FwdParams {
  int B, N, L, H, Bo;
  int nQT, nKT;
  long long total;   // work items = Bo*H*nQT*N
  float scale_log2;
  int bias_mode;
  int nbias_slots;   // resident: nKT; streamed: 2
  const void* bias1;  // [B, L] or null
  const void* bias2;  // [Bo, H, L, L] (used directly in kBiasGlobal mode)
  void* o;           // [B, L, H, D]
  float* lse;        // [B, H, L]
};

template <int D>
struct FwdSmem {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTileBytes = kBM * kRowBytes;      // Q/K/V tile
  static constexpr int kStages = D == 64 ? 2 : 3;
  static constexpr int kBiasTileBytes = kBM * kBN * 2;    // 32 KB
};

__device__ __forceinline__ void decode_item(long long t, int N, int nQT, int H, int& ob, int& h, int& qt,
                                            int& n) {
  n = (int)(t % N);
  long long u = t / N;
  qt = (int)(u % nQT);
  u /= nQT;
  h = (int)(u % H);
  ob = (int)(u / H);
}

template <bool F16>
__device__ __forceinline__ float load_half(const void* base, size_t idx) {
  const unsigned short u = ((const unsigned short*)base)[idx];
  return F16 ? __half2float(__ushort_as_half(u)) : __uint_as_float((uint32_t)u << 16);
}

template <int D, bool F16>
__global__ void __launch_bounds__(kFwdThreads, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmB2,
               const FwdParams p) {
  using S = FwdSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem;                                        // 2 x tile
  uint8_t* sK = sQ + 2 * S::kTileBytes;                      // stages x tile
  uint8_t* sV = sK + S::kStages * S::kTileBytes;             // stages x tile
  uint8_t* sBias = sV + S::kStages * S::kTileBytes;          // nbias_slots x 32 KB
  float* sB1 = (float*)(sBias + (size_t)p.nbias_slots * S::kBiasTileBytes);  // nKT*128 floats
  uint64_t* bars = (uint64_t*)(sB1 + p.nKT * kBN);
  uint64_t* q_full = bars;                 // 2
  uint64_t* q_empty = bars + 2;            // 2
  uint64_t* kv_full = bars + 4;            // stages
  uint64_t* kv_empty = kv_full + S::kStages;
  uint64_t* s_full = kv_empty + S::kStages;  // 2
  uint64_t* s_free = s_full + 2;             // 2
  uint64_t* p_full = s_free + 2;             // 2
  uint64_t* o_full = p_full + 2;             // 2
  uint64_t* o_free = o_full + 2;             // 2
  uint64_t* bias_full = o_free + 2;          // nbias_slots
  uint64_t* bias_empty = bias_full + p.nbias_slots;
  uint32_t* tmem_slot = (uint32_t*)(bias_empty + p.nbias_slots);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  // contiguous slice of the work list for this CTA
  const long long t0 = p.total * blockIdx.x / gridDim.x;
  const long long t1 = p.total * (blockIdx.x + 1) / gridDim.x;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&q_full[0], 1); ptx::mbar_init(&q_full[1], 1);
    ptx::mbar_init(&q_empty[0], 1); ptx::mbar_init(&q_empty[1], 1);
    for (int s = 0; s < S::kStages; ++s) { ptx::mbar_init(&kv_full[s], 1); ptx::mbar_init(&kv_empty[s], 1); }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_free[s], 1);
      ptx::mbar_init(&p_full[s], 128);
      ptx::mbar_init(&o_full[s], 1);
      ptx::mbar_init(&o_free[s], 128);
    }
    for (int s = 0; s < p.nbias_slots; ++s) { ptx::mbar_init(&bias_full[s], 1); ptx::mbar_init(&bias_empty[s], 128); }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const uint32_t idS = ptx::instr_desc(kBM, kBN, F16, false, false);
  const uint32_t idO = ptx::instr_desc(kBM, D, F16, false, true);
  constexpr uint32_t kSw = ptx::swizzle_code(S::kRowBytes);
  const bool streamed = p.bias_mode == kBiasStreamed;
  const bool resident = p.bias_mode == kBiasResident;

  if (warp == 0) {
    // ===================================================== TMA producer
    if (lane == 0) {
      ptx::tma_prefetch(&tmQ); ptx::tma_prefetch(&tmK); ptx::tma_prefetch(&tmV);
      if (resident || streamed) ptx::tma_prefetch(&tmB2);
      int qs = 0; uint32_t qph = 0;
      int ks = 0; uint32_t kph = 0;
      int bslot = 0; uint32_t bph = 0;
      long long cur_unit = -1;
      for (long long t = t0; t < t1; ++t) {
        int ob, h, qt, n;
        decode_item(t, p.N, p.nQT, p.H, ob, h, qt, n);
        const int b = ob * p.N + n;
        const long long unit = t / p.N;
        if (resident && unit != cur_unit) {
          cur_unit = unit;
          for (int j = 0; j < p.nKT; ++j) {
            ptx::mbar_wait(&bias_empty[j], bph ^ 1);
            ptx::mbar_expect_tx(&bias_full[j], S::kBiasTileBytes);
            uint8_t* dst = sBias + (size_t)j * S::kBiasTileBytes;
            ptx::tma_load_3d(dst, &tmB2, &bias_full[j], j * kBN, qt * kBM, ob * p.H + h);
            ptx::tma_load_3d(dst + 16384, &tmB2, &bias_full[j], j * kBN + 64, qt * kBM, ob * p.H + h);
          }
          bph ^= 1;
        }
        ptx::mbar_wait(&q_empty[qs], qph ^ 1);
        ptx::mbar_expect_tx(&q_full[qs], S::kTileBytes);
        ptx::tma_load_4d(sQ + qs * S::kTileBytes, &tmQ, &q_full[qs], 0, h, qt * kBM, b);
        if (++qs == 2) { qs = 0; qph ^= 1; }
        for (int j = 0; j < p.nKT; ++j) {
          ptx::mbar_wait(&kv_empty[ks], kph ^ 1);
          ptx::mbar_expect_tx(&kv_full[ks], 2 * S::kTileBytes);
          ptx::tma_load_4d(sK + ks * S::kTileBytes, &tmK, &kv_full[ks], 0, h, j * kBN, b);
          ptx::tma_load_4d(sV + ks * S::kTileBytes, &tmV, &kv_full[ks], 0, h, j * kBN, b);
          if (++ks == S::kStages) { ks = 0; kph ^= 1; }
          if (streamed) {
            ptx::mbar_wait(&bias_empty[bslot], bph ^ 1);
            ptx::mbar_expect_tx(&bias_full[bslot], S::kBiasTileBytes);
            uint8_t* dst = sBias + (size_t)bslot * S::kBiasTileBytes;
            ptx::tma_load_3d(dst, &tmB2, &bias_full[bslot], j * kBN, qt * kBM, ob * p.H + h);
            ptx::tma_load_3d(dst + 16384, &tmB2, &bias_full[bslot], j * kBN + 64, qt * kBM, ob * p.H + h);
            if (++bslot == p.nbias_slots) { bslot = 0; bph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer
    if (lane == 0) {
      int qs = 0; uint32_t qph = 0;
      int ks = 0; uint32_t kph = 0;
      long long tt = 0;  // global tile counter
      bool pend = false; long long pt = 0; int pks = 0;
      auto issue_pv = [&](long long tp, int ksp) {
        const int sb = (int)(tp & 1);
        const uint32_t ph = (uint32_t)((tp >> 1) & 1);
        ptx::mbar_wait(&p_full[sb], ph);
        ptx::mbar_wait(&o_free[sb], ph ^ 1);
        ptx::tc_fence_after();
        const uint32_t vbase = ptx::smem_u32(sV + ksp * S::kTileBytes);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          // V is MN-major: 16 keys = 2 x 8-row swizzle atoms, SBO = 8 rows
          const uint64_t bd = ptx::smem_desc(vbase + kk * 16 * S::kRowBytes, 16 * S::kRowBytes,
                                             8 * S::kRowBytes, kSw);
          ptx::mma_ts(tmem + 256 + sb * D, tmem + sb * 128 + kk * 8, bd, idO, kk > 0);
        }
        ptx::tc_commit(&o_full[sb]);
        ptx::tc_commit(&s_free[sb]);
        ptx::tc_commit(&kv_empty[ksp]);
      };
      for (long long t = t0; t < t1; ++t) {
        ptx::mbar_wait(&q_full[qs], qph);
        const uint32_t qbase = ptx::smem_u32(sQ + qs * S::kTileBytes);
        for (int j = 0; j < p.nKT; ++j) {
          const int sb = (int)(tt & 1);
          ptx::mbar_wait(&kv_full[ks], kph);
          ptx::mbar_wait(&s_free[sb], (uint32_t)(((tt >> 1) & 1) ^ 1));
          ptx::tc_fence_after();
          const uint32_t kbase = ptx::smem_u32(sK + ks * S::kTileBytes);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t ad = ptx::smem_desc(qbase + kk * 32, 16, 8 * S::kRowBytes, kSw);
            const uint64_t bd = ptx::smem_desc(kbase + kk * 32, 16, 8 * S::kRowBytes, kSw);
            ptx::mma_ss(tmem + sb * 128, ad, bd, idS, kk > 0);
          }
          ptx::tc_commit(&s_full[sb]);
          if (j == p.nKT - 1) ptx::tc_commit(&q_empty[qs]);
          if (pend) issue_pv(pt, pks);
          pend = true; pt = tt; pks = ks;
          if (++ks == S::kStages) { ks = 0; kph ^= 1; }
          ++tt;
        }
        if (++qs == 2) { qs = 0; qph ^= 1; }
      }
      if (pend) issue_pv(pt, pks);
    }
  } else {
    // ===================================================== softmax warpgroup
    const int q4 = warp & 3;                 // TMEM lane quadrant of this warp
    const int r = q4 * 32 + lane;            // query row within the tile / TMEM lane
    const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16);
    const int tid_sm = (warp - 2) * 32 + lane;  // 0..127 for cooperative smem fills
    long long tt = 0;
    int bslot = 0; uint32_t bph = 0;
    for (long long t = t0; t < t1; ++t) {
      int ob, h, qt, n;
      decode_item(t, p.N, p.nQT, p.H, ob, h, qt, n);
      const int b = ob * p.N + n;
      const int i = qt * kBM + r;
      // stage bias1[b, :] * log2e in shared memory (fp32), keys >= L masked to -inf
      ptx::named_bar_sync(1, 128);
      for (int j = tid_sm; j < p.nKT * kBN; j += 128) {
        float v = -INFINITY;
        if (j < p.L) v = p.bias1 ? load_half<F16>(p.bias1, (size_t)b * p.L + j) * kLog2e : 0.f;
        sB1[j] = v;
      }
      ptx::named_bar_sync(1, 128);
      const uint16_t* b2row = nullptr;
      if (p.bias_mode == kBiasGlobal)
        b2row = (const uint16_t*)p.bias2 + (((size_t)ob * p.H + h) * p.L + min(i, p.L - 1)) * (size_t)p.L;

      float m_run = -INFINITY, l_run = 0.f, alpha_prev = 0.f;
      float acc[D];
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] = 0.f;

      auto fold_o = [&](long long tp, float alpha) {
        const int sb = (int)(tp & 1);
        ptx::mbar_wait(&o_full[sb], (uint32_t)((tp >> 1) & 1));
        ptx::tc_fence_after();
        constexpr int kChunk = D < 32 ? D : 32;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += kChunk) {
          uint32_t ov[32];
          if constexpr (kChunk == 16) {
            ptx::tmem_ld16(lane_base + 256 + sb * D + c0, *(uint32_t(*)[16])ov);
          } else {
            ptx::tmem_ld32(lane_base + 256 + sb * D + c0, ov);
          }
          ptx::tmem_ld_wait();
#pragma unroll
          for (int d = 0; d < kChunk; ++d) acc[c0 + d] = fmaf(acc[c0 + d], alpha, __uint_as_float(ov[d]));
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&o_free[sb]);
      };

      for (int j = 0; j < p.nKT; ++j) {
        const int sb = (int)(tt & 1);
        ptx::mbar_wait(&s_full[sb], (uint32_t)((tt >> 1) & 1));
        ptx::tc_fence_after();
        // ---- S chunk by chunk (32 columns), each finished with its bias terms before the
        //      next TMEM load is waited on:  x = S*scale*log2e + bias2*log2e + bias1*log2e
        const int j0 = j * kBN;
        int slot = 0;
        if (resident) { slot = j; ptx::mbar_wait(&bias_full[slot], bph); }
        if (streamed) { slot = bslot; ptx::mbar_wait(&bias_full[slot], bph); }
        const uint8_t* bt = sBias + (size_t)slot * S::kBiasTileBytes;
        const bool smem_bias = resident || streamed;
        float x[kBN];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t rr[32];
          ptx::tmem_ld32(lane_base + sb * 128 + c * 32, rr);
          ptx::tmem_ld_wait();
          const float4* b1v = (const float4*)(sB1 + j0 + c * 32);
          if (smem_bias) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int cc = c * 4 + q;  // 16-byte chunk (8 keys) within the 128-key row
              const uint8_t* rowp = bt + (cc >> 3) * 16384 + r * 128;
              const uint4 raw = *(const uint4*)(rowp + (((cc & 7) ^ (r & 7)) << 4));
              const float4 bb0 = b1v[q * 2], bb1 = b1v[q * 2 + 1];
              const float b1f[8] = {bb0.x, bb0.y, bb0.z, bb0.w, bb1.x, bb1.y, bb1.z, bb1.w};
              const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const uint32_t hv = (w[e >> 1] >> ((e & 1) * 16)) & 0xFFFF;
                const float bv = F16 ? __half2float(__ushort_as_half((unsigned short)hv)) : __uint_as_float(hv << 16);
                x[c * 32 + q * 8 + e] = fmaf(__uint_as_float(rr[q * 8 + e]), p.scale_log2, fmaf(bv, kLog2e, b1f[e]));
              }
            }
          } else if (b2row) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const int jj = min(j0 + c * 32 + k, p.L - 1);
              const uint32_t hv = b2row[jj];
              const float bv = F16 ? __half2float(__ushort_as_half((unsigned short)hv)) : __uint_as_float(hv << 16);
              x[c * 32 + k] = fmaf(__uint_as_float(rr[k]), p.scale_log2, fmaf(bv, kLog2e, sB1[j0 + c * 32 + k]));
            }
          } else {
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
              const float4 bb = b1v[k / 4];
              x[c * 32 + k] = fmaf(__uint_as_float(rr[k]), p.scale_log2, bb.x);
              x[c * 32 + k + 1] = fmaf(__uint_as_float(rr[k + 1]), p.scale_log2, bb.y);
              x[c * 32 + k + 2] = fmaf(__uint_as_float(rr[k + 2]), p.scale_log2, bb.z);
              x[c * 32 + k + 3] = fmaf(__uint_as_float(rr[k + 3]), p.scale_log2, bb.w);
            }
          }
        }
        if (streamed) {
          ptx::mbar_arrive(&bias_empty[slot]);
          if (++bslot == p.nbias_slots) { bslot = 0; bph ^= 1; }
        }
        // resident bias: release all tiles right after the last use of this unit (before the
        // O fold, which waits on an MMA that is only issued once the next unit is loading)
        if (resident && j == p.nKT - 1 && (t + 1 == t1 || (t + 1) / p.N != t / p.N)) {
          for (int s2 = 0; s2 < p.nKT; ++s2) ptx::mbar_arrive(&bias_empty[s2]);
          bph ^= 1;
        }
        // ---- online max / exp / sum
        float mt = x[0];
#pragma unroll
        for (int c = 1; c < kBN; ++c) mt = fmaxf(mt, x[c]);
        const float m_new = fmaxf(m_run, mt);
        const float base = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = ex2(m_run - base);
        float sum = 0.f;
        uint32_t pk0[32], pk1[32];
#pragma unroll
        for (int c = 0; c < kBN / 2; c += 2) {
          const float p0 = ex2(x[c] - base), p1 = ex2(x[c + 1] - base);
          sum += p0 + p1;
          pk0[c / 2] = F16 ? ptx::pack_f16(p0, p1) : ptx::pack_bf16(p0, p1);
        }
        ptx::tmem_st32(lane_base + sb * 128, pk0);
#pragma unroll
        for (int c = kBN / 2; c < kBN; c += 2) {
          const float p0 = ex2(x[c] - base), p1 = ex2(x[c + 1] - base);
          sum += p0 + p1;
          pk1[c / 2 - 32] = F16 ? ptx::pack_f16(p0, p1) : ptx::pack_bf16(p0, p1);
        }
        ptx::tmem_st32(lane_base + sb * 128 + 32, pk1);
        l_run = l_run * alpha + sum;
        m_run = m_new;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[sb]);
        // ---- fold the previous tile's O_j into the register accumulator
        if (j > 0) fold_o(tt - 1, alpha_prev);
        alpha_prev = alpha;
        if (j == p.nKT - 1) fold_o(tt, alpha);
        ++tt;
      }
      // ---- epilogue: O = acc / l, LSE = (m + log2 l) * ln 2
      if (i < p.L) {
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        uint32_t ow[D / 2];
#pragma unroll
        for (int d = 0; d < D; d += 2)
          ow[d / 2] = F16 ? ptx::pack_f16(acc[d] * inv, acc[d + 1] * inv) : ptx::pack_bf16(acc[d] * inv, acc[d + 1] * inv);
        uint4* dst = (uint4*)((uint16_t*)p.o + (((size_t)b * p.L + i) * p.H + h) * D);
#pragma unroll
        for (int v = 0; v < D / 8; ++v) dst[v] = make_uint4(ow[4 * v], ow[4 * v + 1], ow[4 * v + 2], ow[4 * v + 3]);
        p.lse[((size_t)b * p.H + h) * p.L + i] = l_run > 0.f ? (m_run + __log2f(l_run)) * kLn2 : -INFINITY;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace tc
}  // namespace evo

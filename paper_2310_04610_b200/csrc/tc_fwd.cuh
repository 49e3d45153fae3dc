// tc_fwd.cuh — K1: fused Evoformer attention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Reference semantics: attn_forward_tiled, /root/reference/proj/core/src/attention_tiled.cpp:57-180
// (S = scale*QK^T + bias, online softmax over key tiles, O = acc/l, LSE = m + ln l), plus the
// DS4Sci mask bias1[b, j]. Layout and schedule are B200-first:
//
//  * Persistent CTAs walk work items (ob, h, q-tile, row) with rows innermost. A run of items with
//    the same (ob, h, q-tile) is a "segment": its pair-bias row block bias2[ob, h, q-tile rows, :]
//    is loaded into shared memory once by TMA (128B swizzle, one 16 KB box per 64 keys) and
//    reused for every MSA row of the segment — the paper's on-the-fly broadcast, read from L2
//    once per CTA instead of once per row. L too long for residency: bias tiles stream per key
//    tile and are shared by the rows in flight. When the grid splits evenly, CTAs get aligned
//    row ranges so the q-tiles of one (row, head) run concurrently and share K/V through L2.
//  * warp 0: TMA producer. warp 1: single-thread tcgen05.mma issuer.
//    NWG independent softmax warpgroups (3 for D <= 32), each owning whole MSA rows: rows of a
//    segment are dealt round-robin, so warpgroups sit at different phases (bias math, MUFU, TMEM
//    traffic) and overlap instead of contending. Per warpgroup: a double-buffered 128x64 fp32 S
//    tile in TMEM (S = Q K^T, SS-MMA) -> registers (one thread = one query row = one TMEM lane),
//    bias1 + bias2 add and online max/sum in the log2 domain with packed f32x2 math, P (bf16)
//    written back over S and consumed by a K=64 TS-MMA that accumulates O in TMEM. The running max
//    only moves (rescaling O in TMEM) when it grows by more than 2^8 (FA4's lazy rescale), so the
//    steady state has no per-tile O traffic; O is read once per row.
//  * TMEM per warpgroup w: S buffers [W*w, W*w+64) [W*w+64, W*w+128), O [W*w+128, W*w+128+D),
//    W = 128 + D.
#pragma once
#include "common.cuh"
#include "tc_ptx.cuh"

namespace evo {
namespace tc {

constexpr int kBM = 128;                 // query rows per tile (UMMA M, TMEM lanes)
constexpr int kBN = 64;                  // keys per tile (UMMA N of S)
#ifndef EVO_FWD_RESCALE_LOG2
#define EVO_FWD_RESCALE_LOG2 8  // lazy rescale once the running max grew by more than this (log2 units)
#endif
constexpr float kRescaleThreshold = (float)EVO_FWD_RESCALE_LOG2;
#ifndef EVO_FWD_POLY_EVERY
#define EVO_FWD_POLY_EVERY 4
#endif
constexpr int kPolyEvery = EVO_FWD_POLY_EVERY;  // 1 pair in kPolyEvery exponentiated by polynomial (0: none)
#ifndef EVO_FWD_SELF_PV
#define EVO_FWD_SELF_PV 0  // 1: the softmax warpgroup's last thread to finish P issues the PV UMMA itself
#endif

template <int D>
struct FwdCfg {
  static constexpr int NWG = D <= 32 ? 3 : 2;          // softmax warpgroups
  static constexpr int kThreads = 32 + 160 * NWG;        // TMA warp + per warpgroup: UMMA warp, 4 softmax warps
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTileQ = kBM * kRowBytes;       // Q tile
  static constexpr int kTileKV = kBN * kRowBytes;      // K or V tile
  static constexpr int kStages = 2 * NWG;              // K/V ring depth
  static constexpr int kBiasTile = kBM * kBN * 2;      // 16 KB
  static constexpr int kWGcols = 128 + D;              // TMEM columns per warpgroup
};

enum BiasMode : int { kBiasNone = 0, kBiasResident = 1, kBiasStreamed = 2, kBiasGlobal = 3 };

struct FwdParams {
  int B, N, L, H, Bo;
  int swapped;       // 1: o is [L, B, H, D] (raw msa_col / tri_end layout)
  int nQT, nKT;
  long long total;   // work items = Bo*H*nQT*N
  int aligned;       // 1: CTA c owns part c%split of unit c/split; 0: flat contiguous split
  int split;
  float scale_log2;
  int dreal;         // head dim in memory (D = 16 kernels serve D = 8: TMA zero-fills the padded columns)
  int nbias_slots;   // resident: nKT; streamed: 3
  int b1_tma;        // bias1 rows fetched by TMA bulk copy (L % 8 == 0)
  int aug;           // bias1 / key mask enter S as one extra K=16 MMA step (bias1 present or L % 64 != 0)
  uint32_t aug_c;    // (c_lo << 16) | c_hi: 16-bit two-term split of 1/scale
  int b1_rows;       // bias1 rows staged in shared memory per Q slot (b1_tma and the budget allows)
  int* flag;         // numeric-check flag (non-finite LSE / NaN O) or null
  const void* bias1;  // [B, L] or null
  const void* bias2;  // [Bo, H, L, L] (read directly in kBiasGlobal mode)
  void* o;           // [B, L, H, D]
  float* lse;        // [B, H, L]
  // The parameter block keeps the layout the hot kernel variants were tuned with (extra fields measurably
  // changed their code generation): the gate pointer shares the slot of the bring-up trace buffer
  union {
    unsigned long long* trace;  // bring-up timeline of CTA 0 (EVO_TRACE builds only)
    const void* gate;           // output-gate logits (layout of o) or null: o = sigmoid(gate) * attention
  };
};

enum TraceEv { kTrKV = 0, kTrS = 1, kTrSseen = 2, kTrP0 = 3, kTrP1 = 4, kTrPV = 5, kTrRowEnd = 6, kTrRowStart = 7 };
__device__ __forceinline__ void trace(const FwdParams& p, int ev, uint32_t tile) {
  if constexpr (EVO_TRACE) {
    if (p.trace && blockIdx.x == 0 && tile < 64) p.trace[ev * 64 + tile] = clock64();
  }
}

template <bool F16>
__device__ __forceinline__ float load_half(const void* base, size_t idx) {
  const unsigned short u = ((const unsigned short*)base)[idx];
  return F16 ? __half2float(__ushort_as_half(u)) : __uint_as_float((uint32_t)u << 16);
}
template <bool F16>
__device__ __forceinline__ float2 unpack2(uint32_t w) {  // two packed 16-bit floats, low first
  if constexpr (F16) {
    __half2 hh = *reinterpret_cast<__half2*>(&w);
    return __half22float2(hh);
  } else {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  }
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(ptx::smem_u32(a)), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

// One CTA's item range, cut into segments at (ob, h, q-tile) boundaries. Inside a segment the
#ifndef EVO_FWD_PREFETCH
#define EVO_FWD_PREFETCH 0  // L2 prefetch distance of K/V tiles; 0 = off (measured 5 % faster at C4:
#endif                      // the extra TMA requests delayed the real loads)
constexpr int kPrefetchAhead = EVO_FWD_PREFETCH;
constexpr int kAugA = kBM * 32, kAugB = kBN * 32;  // bias1 augmentation tiles (16 bf16 per row)  // K/V tiles pulled into L2 ahead of their shared-memory load

// rows go out in groups of NWG (row s0 + g*NWG + w -> warpgroup w).
struct Walker {
  long long t0, t1, N;
  __device__ long long seg_end(long long s) const {
    const long long e = (s / N + 1) * N;
    return e < t1 ? e : t1;
  }
};
__device__ __forceinline__ Walker make_walker(const FwdParams& p) {
  if (p.aligned) {
    const long long unit = blockIdx.x / p.split, part = blockIdx.x % p.split;
    const long long base = unit * p.N;
    return Walker{base + p.N * part / p.split, base + p.N * (part + 1) / p.split, p.N};
  }
  return Walker{p.total * blockIdx.x / gridDim.x, p.total * (blockIdx.x + 1) / gridDim.x, p.N};
}
struct SegInfo {
  int ob, h, qt, n0;  // n0 = row index (within N) of the segment's first item
};
__device__ __forceinline__ SegInfo seg_info(long long s0, const FwdParams& p) {
  SegInfo si;
  long long u = s0 / p.N;
  si.n0 = (int)(s0 - u * p.N);
  si.qt = (int)(u % p.nQT);
  u /= p.nQT;
  si.h = (int)(u % p.H);
  si.ob = (int)(u / p.H);
  return si;
}

template <int D, bool F16, int BM, bool SAFE>  // SAFE: numeric checks, output gate, padded head dim compiled in
__global__ void __launch_bounds__(FwdCfg<D>::kThreads, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmB2,
               const FwdParams p) {
  using C = FwdCfg<D>;
  constexpr int NWG = C::NWG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int LP = p.nKT * kBN;                               // padded key count
  uint8_t* sQ = smem;                                       // [NWG][2] Q tiles
  uint8_t* sK = sQ + NWG * 2 * C::kTileQ;                   // [stages]
  uint8_t* sV = sK + C::kStages * C::kTileKV;               // [stages]
  uint8_t* sBias = sV + C::kStages * C::kTileKV;            // [nbias_slots] x 16 KB
  uint8_t* sAaug = sBias + (size_t)p.nbias_slots * C::kBiasTile;  // 128 x 16: (c_hi, c_lo, 0..), SW32
  uint8_t* sBaug = sAaug + kAugA;                            // [stages] 64 x 16: (bias1, bias1, 0..), SW32
  uint16_t* sB1raw = (uint16_t*)(sBaug + C::kStages * kAugB);  // [NWG][2][LP] bias1 rows (raw), when b1_rows
  uint64_t* bars = (uint64_t*)(sB1raw + (p.b1_rows ? NWG * 2 * LP : 0));
  uint64_t* q_full = bars;                       // [NWG][2] Q (+ bias1 row) landed
  uint64_t* q_empty = q_full + 2 * NWG;          // [NWG][2] last S of the row done
  uint64_t* s_full = q_empty + 2 * NWG;          // [NWG][2]
  uint64_t* s_free = s_full + 2 * NWG;           // [NWG][2] PV reading that buffer done
  uint64_t* p_full = s_free + 2 * NWG;           // [NWG][2]
  uint64_t* o_free = p_full + 2 * NWG;           // [NWG] O read out at row end
  uint64_t* kv_full = o_free + NWG;              // [stages] K tile landed
  uint64_t* kv_empty = kv_full + C::kStages;     // [stages] S of that K tile done
  uint64_t* v_full = kv_empty + C::kStages;      // [stages] V tile landed
  uint64_t* v_empty = v_full + C::kStages;       // [stages] PV of that V tile done
  uint64_t* bias_full = v_empty + C::kStages;    // [nbias_slots]
  uint64_t* bias_empty = bias_full + p.nbias_slots;
  uint32_t* tmem_slot = (uint32_t*)(bias_empty + p.nbias_slots);
  // [NWG][2] threads done writing P into S buffer sb (self-issued PV: the 128th issues it). Per buffer: a
  // thread can run one tile ahead of its warpgroup (the other S buffer), never two (that buffer's S
  // waits for this PV)
  uint32_t* p_count = tmem_slot + 1;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const Walker W = make_walker(p);

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2 * NWG; ++s) {
      ptx::mbar_init(&q_full[s], 1);
      ptx::mbar_init(&q_empty[s], 1);
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_free[s], 1);
      ptx::mbar_init(&p_full[s], 128);
    }
    for (int w = 0; w < NWG; ++w) {
      ptx::mbar_init(&o_free[w], 128);
      p_count[2 * w] = p_count[2 * w + 1] = 0;
    }
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < p.nbias_slots; ++s) { ptx::mbar_init(&bias_full[s], 1); ptx::mbar_init(&bias_empty[s], NWG); }
    ptx::fence_barrier_init();
  }
  // A_aug: row i = (c_hi, c_lo, 0, ...); with B_aug row j = (bias1[j], bias1[j], 0, ...) one extra K=16
  // step of S = Q K^T adds bias1[j] / scale exactly to ~2^-16 (16B chunk 0 of a 32B row sits at chunk
  // (row >> 2) & 1 under the 32B swizzle).
  for (int i = threadIdx.x; i < kBM; i += blockDim.x) {
    const uint32_t c = (uint32_t)((i >> 2) & 1);
    uint4* row = (uint4*)(sAaug + i * 32);
    row[c] = make_uint4(p.aug_c, 0u, 0u, 0u);
    row[c ^ 1] = make_uint4(0u, 0u, 0u, 0u);
  }
  ptx::fence_proxy_async_smem();
  if (warp == 0) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  constexpr uint32_t kSw = ptx::swizzle_code(C::kRowBytes);
  constexpr bool streamed = BM == kBiasStreamed;
  constexpr bool resident = BM == kBiasResident;

  if (warp == 0) {
    if (lane == 0) {
      // ===================================================== TMA producer (polling)
      // Each warpgroup owns Q slots {2w, 2w+1} and K/V stages {2w, 2w+1}; K frees when its S
      // completed, V when its PV completed. Within a group of rows the producer serves whichever
      // warpgroup has a free slot, so a slow warpgroup never blocks the loads of the others.
      ptx::tma_prefetch(&tmQ); ptx::tma_prefetch(&tmK); ptx::tma_prefetch(&tmV);
      if (resident || streamed) ptx::tma_prefetch(&tmB2);
      uint32_t qc[NWG], tk[NWG];  // per warpgroup: Q loads, K/V tiles of finished groups
#pragma unroll
      for (int w = 0; w < NWG; ++w) qc[w] = tk[w] = 0;
      int bslot = 0; uint32_t bph = 0;
      const uint32_t b1_bytes = (uint32_t)p.L * 2;
      const bool b1t = p.bias1 && p.b1_rows;
      for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
        const long long s1 = W.seg_end(s0);
        const SegInfo si = seg_info(s0, p);
        const int plane = si.ob * p.H + si.h;
        const int row_end = si.ob * p.N + si.n0 + (int)(s1 - s0);
        if (resident) {
          for (int j = 0; j < p.nKT; ++j) {
            ptx::mbar_wait(&bias_empty[j], bph ^ 1);
            ptx::mbar_expect_tx(&bias_full[j], C::kBiasTile);
            ptx::tma_load_3d(sBias + (size_t)j * C::kBiasTile, &tmB2, &bias_full[j], j * kBN, si.qt * kBM, plane);
          }
          bph ^= 1;
        }
        int n = si.n0;
        for (long long a = s0; a < s1; a += NWG, n += NWG) {
          const int np = (int)min((long long)NWG, s1 - a);
          uint32_t qdone = 0;
          int jn[NWG], jv[NWG], jb = streamed ? 0 : p.nKT;
#pragma unroll
          for (int w = 0; w < NWG; ++w) jn[w] = jv[w] = w < np ? 0 : p.nKT;
          for (;;) {
            bool progress = false, done = jb >= p.nKT;
#pragma unroll
            for (int w = 0; w < NWG; ++w) {
              if (w >= np) continue;
              const int b = si.ob * p.N + n + w;
              if (!((qdone >> w) & 1)) {
                const uint32_t slot = qc[w] & 1, ph = (qc[w] >> 1) & 1;
                if (ptx::mbar_test(&q_empty[w * 2 + slot], ph ^ 1)) {
                  ptx::mbar_expect_tx(&q_full[w * 2 + slot], C::kTileQ + (b1t ? b1_bytes : 0));
                  ptx::tma_load_4d(sQ + (w * 2 + slot) * C::kTileQ, &tmQ, &q_full[w * 2 + slot], 0, si.h,
                                   si.qt * kBM, b);
                  if (b1t)
                    bulk_g2s(sB1raw + (w * 2 + slot) * LP, (const uint16_t*)p.bias1 + (size_t)b * p.L, b1_bytes,
                             &q_full[w * 2 + slot]);
                  ++qc[w];
                  qdone |= 1u << w;
                  progress = true;
                }
              }
              if (jn[w] < p.nKT) {
                const uint32_t t = tk[w] + jn[w];
                const int ks = w * 2 + (int)(t & 1);
                if (ptx::mbar_test(&kv_empty[ks], ((t >> 1) & 1) ^ 1)) {
                  ptx::mbar_expect_tx(&kv_full[ks], C::kTileKV);
                  ptx::tma_load_4d(sK + ks * C::kTileKV, &tmK, &kv_full[ks], 0, si.h, jn[w] * kBN, b);
                  if (w == 0) trace(p, 10, t);
                  // K/V tiles come from HBM with ~2 us latency under load: pull the ones
                  // kPrefetchAhead further (or this warpgroup's next row's first ones) into L2
                  const int ja = jn[w] + kPrefetchAhead;
                  const int pb = ja < p.nKT ? b : b + NWG;
                  if (kPrefetchAhead > 0 && pb < row_end) {
                    const int pj = ja < p.nKT ? ja : ja - p.nKT;
                    ptx::tma_prefetch_4d(&tmK, 0, si.h, pj * kBN, pb);
                    ptx::tma_prefetch_4d(&tmV, 0, si.h, pj * kBN, pb);
                  }
                  ++jn[w];
                  progress = true;
                }
              }
              if (jv[w] < p.nKT) {
                const uint32_t t = tk[w] + jv[w];
                const int ks = w * 2 + (int)(t & 1);
                if (ptx::mbar_test(&v_empty[ks], ((t >> 1) & 1) ^ 1)) {
                  ptx::mbar_expect_tx(&v_full[ks], C::kTileKV);
                  ptx::tma_load_4d(sV + ks * C::kTileKV, &tmV, &v_full[ks], 0, si.h, jv[w] * kBN, b);
                  if (w == 0) trace(p, kTrKV, t);
                  ++jv[w];
                  progress = true;
                }
              }
              done = done && ((qdone >> w) & 1) && jn[w] >= p.nKT && jv[w] >= p.nKT;
            }
            if (jb < p.nKT && ptx::mbar_test(&bias_empty[bslot], bph ^ 1)) {  // streamed pair-bias ring
              ptx::mbar_expect_tx(&bias_full[bslot], C::kBiasTile);
              ptx::tma_load_3d(sBias + (size_t)bslot * C::kBiasTile, &tmB2, &bias_full[bslot], jb * kBN,
                               si.qt * kBM, plane);
              if (++bslot == p.nbias_slots) { bslot = 0; bph ^= 1; }
              ++jb;
              progress = true;
            }
            if (done) break;
            if (!progress) __nanosleep(64);  // yield issue slots to the softmax warps
          }
#pragma unroll
          for (int w = 0; w < NWG; ++w)
            if (w < np) tk[w] += p.nKT;
        }
      }
    }
  } else if (warp <= NWG) {
    // ===================================================== UMMA issuer of warpgroup w = warp - 1
    // Waits only on this warpgroup's barriers: S(t) = Q K_t^T once K(t) landed and PV(t-2) released
    // the S buffer; PV(t) = P(t) V_t (TS, P from TMEM) once the softmax wrote P(t) and V(t) landed.
    const int w = warp - 1;
    {
      const uint32_t idS = ptx::instr_desc(kBM, kBN, F16, false, false);
      const uint32_t idO = ptx::instr_desc(kBM, D, F16, false, true);
      constexpr uint32_t kHiAug = ptx::desc_hi(256, 6);  // 32-byte rows, SW32
      const uint64_t aAug = ptx::desc_make(ptx::desc_lo(ptx::smem_u32(sAaug), 16), kHiAug);
      const uint32_t wbase = tmem + w * C::kWGcols;
      uint32_t qc = 0, t = 0, rc = 0;
      auto do_pv = [&](uint32_t T, bool first) {
        const uint32_t sb = T & 1;
        const int ks = w * 2 + (int)(T & 1);
        ptx::mbar_wait_spin(&p_full[w * 2 + sb], (T >> 1) & 1);
        if (w == 0 && lane == 0) trace(p, 8, T);
        ptx::mbar_wait_spin(&v_full[ks], (T >> 1) & 1);
        if (w == 0 && lane == 0) trace(p, 9, T);
        if (first) {  // first tile of a row overwrites O: the previous row must be read out
          ptx::mbar_wait_spin(&o_free[w], (rc & 1) ^ 1);
          ++rc;
        }
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t vbase = ptx::smem_u32(sV + ks * C::kTileKV);
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk) {
            // V is MN-major: 16 keys = two 8-row swizzle atoms (SBO = 8 rows)
            const uint64_t bd =
                ptx::smem_desc(vbase + kk * 16 * C::kRowBytes, 16 * C::kRowBytes, 8 * C::kRowBytes, kSw);
            ptx::mma_ts(wbase + 128, wbase + sb * 64 + kk * 8, bd, idO, (!first || kk > 0) ? 1u : 0u);
          }
          ptx::tc_commit(&s_free[w * 2 + sb]);
          ptx::tc_commit(&v_empty[ks]);
          if (w == 0) trace(p, kTrPV, T);
        }
        __syncwarp();
      };
      for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
        const long long s1 = W.seg_end(s0);
        const SegInfo si = seg_info(s0, p);
        for (long long a = s0 + w; a < s1; a += NWG) {
          const uint32_t qs = qc & 1;
          const int b = si.ob * p.N + si.n0 + (int)(a - s0);
          for (int j = 0; j < p.nKT; ++j, ++t) {
            const uint32_t sb = t & 1;
            const int ks = w * 2 + (int)(t & 1);
            if (j == 0) ptx::mbar_wait_spin(&q_full[w * 2 + qs], (qc >> 1) & 1);
            ptx::mbar_wait_spin(&kv_full[ks], (t >> 1) & 1);  // K(t) landed; B_aug slot ks is free
            if (w == 0 && lane == 0) trace(p, 11, t);
            if (p.aug) {
              // B_aug row jj = (bias1[j0 + jj], same or 0 if non-finite) for keys < L, (-inf, 0) past L
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const int jj = lane + 32 * h2, key = j * kBN + jj;
                uint32_t v0 = 0u, v1 = 0u;
                if (key >= p.L) {
                  v0 = F16 ? 0xFC00u : 0xFF80u;
                } else if (p.bias1) {
                  v0 = p.b1_rows ? (uint32_t)sB1raw[(w * 2 + qs) * LP + key]
                                : (uint32_t)((const uint16_t*)p.bias1)[(size_t)b * p.L + key];
                  const bool fin = F16 ? (v0 & 0x7C00u) != 0x7C00u : (v0 & 0x7F80u) != 0x7F80u;
                  v1 = fin ? v0 : 0u;
                }
                const uint32_t c = (uint32_t)((jj >> 2) & 1);
                uint4* row = (uint4*)(sBaug + ks * kAugB + jj * 32);
                row[c] = make_uint4(v0 | (v1 << 16), 0u, 0u, 0u);
                row[c ^ 1] = make_uint4(0u, 0u, 0u, 0u);
              }
              ptx::fence_proxy_async_smem();
              __syncwarp();
            }
            ptx::mbar_wait_spin(&s_free[w * 2 + sb], ((t >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
              const uint32_t qbase = ptx::smem_u32(sQ + (w * 2 + qs) * C::kTileQ);
              const uint32_t kbase = ptx::smem_u32(sK + ks * C::kTileKV);
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint64_t ad = ptx::smem_desc(qbase + kk * 32, 16, 8 * C::kRowBytes, kSw);
                const uint64_t bd = ptx::smem_desc(kbase + kk * 32, 16, 8 * C::kRowBytes, kSw);
                ptx::mma_ss(wbase + sb * 64, ad, bd, idS, kk > 0);
              }
              if (p.aug)
                ptx::mma_ss(wbase + sb * 64, aAug,
                            ptx::desc_make(ptx::desc_lo(ptx::smem_u32(sBaug + ks * kAugB), 16), kHiAug), idS, 1u);
              ptx::tc_commit(&s_full[w * 2 + sb]);
              ptx::tc_commit(&kv_empty[ks]);  // the K stage (and its B_aug rows) may be refilled once S completed
              if (w == 0) trace(p, kTrS, t);
              if (j == p.nKT - 1) ptx::tc_commit(&q_empty[w * 2 + qs]);
            }
            __syncwarp();
            if (!EVO_FWD_SELF_PV && j > 0) do_pv(t - 1, j == 1);
          }
          if (!EVO_FWD_SELF_PV) do_pv(t - 1, p.nKT == 1);
          ++qc;
        }
      }
    }
  } else {
    // ===================================================== softmax warpgroups
    const int wg = (warp - 1 - NWG) / 4;
    const int q4 = warp & 3;                  // TMEM lane quadrant
    const int r = q4 * 32 + lane;             // query row in tile == TMEM lane
    const int tid_wg = (warp - 1 - NWG - 4 * wg) * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t tbase = tmem + lane_off + wg * C::kWGcols;
    const uint32_t o_tmem = tbase + 128;
    const uint32_t bias_addr = ptx::smem_u32(sBias) + r * 128;
    const uint32_t r7 = (uint32_t)(r & 7) << 4;  // 128B swizzle: chunk c of row r -> (c ^ (r & 7))
    const float2 scl2 = make_float2(p.scale_log2, p.scale_log2);
    const float2 lg2 = make_float2(kLog2e, kLog2e);
    uint32_t tcount = 0;
    int bslot = 0; uint32_t bph = 0;

    for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
      const long long s1 = W.seg_end(s0);
      const SegInfo si = seg_info(s0, p);
      const int i = si.qt * kBM + r;
      const uint16_t* b2row = nullptr;
      if constexpr (BM == kBiasGlobal)
        b2row = (const uint16_t*)p.bias2 + (((size_t)si.ob * p.H + si.h) * p.L + min(i, p.L - 1)) * (size_t)p.L;
      bool released = false;
      int n = si.n0;
      for (long long a = s0; a < s1; a += NWG, n += NWG) {
        const int np = (int)min((long long)NWG, s1 - a);
        if (wg >= np) {
          // no row for this warpgroup in the segment's last group: keep the shared streamed-bias
          // ring in step (wait each fill, then release it). All four warps must have seen the fill
          // before the release: the producer may refill the slot right away, and a warp still waiting
          // for the old phase would then see the parity flip twice and wait forever.
          if (streamed) {
            for (int j = 0; j < p.nKT; ++j) {
              ptx::mbar_wait(&bias_full[bslot], bph);
              ptx::named_bar_sync(1 + wg, 128);
              if (tid_wg == 0) ptx::mbar_arrive(&bias_empty[bslot]);
              if (++bslot == p.nbias_slots) { bslot = 0; bph ^= 1; }
            }
          }
          continue;
        }
        const int b = si.ob * p.N + n + wg;
        const bool last_row = a + NWG >= s1;
        // bias1 and the key mask past L are already inside S (the UMMA warp's augmentation step)
        if (tid_wg == 0 && wg == 0) trace(p, kTrRowStart, tcount);

        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < p.nKT; ++j) {
          const uint32_t sb = tcount & 1;
          const uint32_t s_tmem = tbase + sb * 64;
          ptx::mbar_wait(&s_full[wg * 2 + sb], (tcount >> 1) & 1);
          if (tid_wg == 0 && wg == 0) trace(p, kTrSseen, tcount);
          ptx::tc_fence_after();
          uint32_t ra[32], rb[32];
          ptx::tmem_ld32(s_tmem, ra);
          ptx::tmem_ld32(s_tmem + 32, rb);
          const int j0 = j * kBN;
          int slot = 0;
          if (resident) { slot = j; ptx::mbar_wait(&bias_full[slot], bph); }
          if (streamed) { slot = bslot; ptx::mbar_wait(&bias_full[slot], bph); }
          ptx::tmem_ld_wait();
          auto sv = [&](int k) { return __uint_as_float(k < 32 ? ra[k & 31] : rb[k & 31]); };
          // ---- x = (S + bias1/scale) * scale * log2e + bias2 * log2e - m   (log2 domain), relative to the
          // running max m (0 before the first finite logit): one ffma2 per pair (bias path: two), and the
          // exponent argument is final unless the max grows past the lazy-rescale threshold
          const float base0 = m_run == -INFINITY ? 0.f : m_run;
          const float2 nb0 = make_float2(-base0, -base0);
          float2 x[32];
          if constexpr (resident || streamed) {
            // 128B-swizzled bias tile: 8-key chunk c of row r sits at chunk c ^ (r & 7)
            const uint32_t bt = bias_addr + slot * C::kBiasTile;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint4 raw = lds128(bt + ((uint32_t)(c << 4) ^ r7));
              const uint32_t wv[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                x[c * 4 + e] = __ffma2_rn(make_float2(sv(c * 8 + 2 * e), sv(c * 8 + 2 * e + 1)), scl2,
                                          __ffma2_rn(unpack2<F16>(wv[e]), lg2, nb0));
            }
          } else if constexpr (BM == kBiasGlobal) {
#pragma unroll
            for (int k = 0; k < kBN; k += 2) {
              const int ja = min(j0 + k, p.L - 1), jb = min(j0 + k + 1, p.L - 1);
              const float2 bv = make_float2(load_half<F16>(b2row, ja), load_half<F16>(b2row, jb));
              x[k / 2] = __ffma2_rn(make_float2(sv(k), sv(k + 1)), scl2, __ffma2_rn(bv, lg2, nb0));
            }
          } else {
#pragma unroll
            for (int k = 0; k < kBN; k += 2) x[k / 2] = __ffma2_rn(make_float2(sv(k), sv(k + 1)), scl2, nb0);
          }
          // ---- bias release: streamed tiles per use; the resident block after the segment's last use
          if (streamed || (resident && last_row && j == p.nKT - 1)) {
            ptx::named_bar_sync(1 + wg, 128);
            if (tid_wg == 0) {
              if (streamed) ptx::mbar_arrive(&bias_empty[slot]);
              else for (int s2 = 0; s2 < p.nKT; ++s2) ptx::mbar_arrive(&bias_empty[s2]);
            }
            released = true;
          }
          if (streamed && ++bslot == p.nbias_slots) { bslot = 0; bph ^= 1; }
          // ---- tile max; lazy rescale of the running max and O
          float mx[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) mx[k] = fmaxf(x[k].x, x[k].y);
#pragma unroll
          for (int k = 4; k < 32; ++k) mx[k & 3] = fmax3(mx[k & 3], x[k].x, x[k].y);
          const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));  // tile max minus base0
          // grow: the first tile with a finite logit, or the max rose by more than the threshold
          const bool grow = m_run == -INFINITY ? mt != -INFINITY : mt > kRescaleThreshold;
          float dl = 0.f;  // re-bases the exponent arguments on a grown max (0 in the steady state)
          if (__any_sync(0xffffffffu, grow)) {
            const float m_new = grow ? base0 + mt : m_run;
            const float alpha = ex2(m_run - (m_new == -INFINITY ? 0.f : m_new));  // 0 when m_run=-inf
            l_run *= alpha;
            dl = grow ? mt : 0.f;
            if (j > 0) {
              // O holds the PVs of earlier tiles: wait for the last one, scale these rows in TMEM
              const uint32_t tp = tcount - 1;
              ptx::mbar_wait(&s_free[wg * 2 + (tp & 1)], (tp >> 1) & 1);
              ptx::tc_fence_after();
#pragma unroll
              for (int c0 = 0; c0 < D; c0 += 16) {
                uint32_t ov[16];
                ptx::tmem_ld16(o_tmem + c0, ov);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int d = 0; d < 16; ++d) ov[d] = __float_as_uint(__uint_as_float(ov[d]) * alpha);
                ptx::tmem_st16(o_tmem + c0, ov);
              }
            }
            m_run = m_new;
          }
          float2 sum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          uint32_t pk[32];
          const float2 nd = make_float2(-dl, -dl);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            float2 t = __fadd2_rn(x[k], nd);
            if (kPolyEvery > 0 && k % kPolyEvery == kPolyEvery - 1) {
              t = ex2_poly2(t);  // every kPolyEvery-th pair on the FMA pipe, the rest on MUFU
            } else {
              t.x = ex2(t.x);
              t.y = ex2(t.y);
            }
            sum[k & 1] = __fadd2_rn(sum[k & 1], t);
            pk[k] = F16 ? ptx::pack_f16(t.x, t.y) : ptx::pack_bf16(t.x, t.y);
          }
          ptx::tmem_st32(s_tmem, pk);  // P (bf16) over the first 32 columns of this S buffer
          const float2 s01 = __fadd2_rn(sum[0], sum[1]);
          l_run += s01.x + s01.y;
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          if (EVO_FWD_SELF_PV) {
            // PV(t) = P(t) V_t issued by the warpgroup's last thread to finish writing P (acq_rel
            // counter: every thread's TMEM stores are ordered before it) — no round trip through the
            // UMMA warp, which shares its SMSP with three busy softmax warps
            if ((atom_add_acq_rel(&p_count[wg * 2 + sb], 1u) & 127u) == 127u) {
              ptx::tc_fence_after();
              const int ks = wg * 2 + (int)(tcount & 1);
              ptx::mbar_wait(&v_full[ks], (tcount >> 1) & 1);
              const uint32_t vbase = ptx::smem_u32(sV + ks * C::kTileKV);
              const uint32_t idO = ptx::instr_desc(kBM, D, F16, false, true);
              const uint32_t wbase = tmem + wg * C::kWGcols;
#pragma unroll
              for (int kk = 0; kk < kBN / 16; ++kk) {
                const uint64_t bd =
                    ptx::smem_desc(vbase + kk * 16 * C::kRowBytes, 16 * C::kRowBytes, 8 * C::kRowBytes, kSw);
                ptx::mma_ts(wbase + 128, wbase + sb * 64 + kk * 8, bd, idO, (j > 0 || kk > 0) ? 1u : 0u);
              }
              ptx::tc_commit(&s_free[wg * 2 + sb]);
              ptx::tc_commit(&v_empty[ks]);
            }
            __syncwarp();  // reconverge before the next .sync.aligned tcgen05 load
          } else {
            ptx::mbar_arrive(&p_full[wg * 2 + sb]);
          }
          if (tid_wg == 0) trace(p, wg == 0 ? kTrP0 : kTrP1, tcount);
          ++tcount;
        }
        // ---- row end: O = O / l, LSE = (m + log2 l) * ln 2
        const uint32_t tl = tcount - 1;
        ptx::mbar_wait(&s_free[wg * 2 + (tl & 1)], (tl >> 1) & 1);  // last PV of the row done
        ptx::tc_fence_after();
        uint32_t ov[D];
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 16) ptx::tmem_ld16(o_tmem + c0, *(uint32_t(*)[16])(&ov[c0]));
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        if (!EVO_FWD_SELF_PV) ptx::mbar_arrive(&o_free[wg]);
        if (tid_wg == 0 && wg == 0) trace(p, kTrRowEnd, tl);
        if (i < p.L) {
          const float inv = l_run > 0.f ? __frcp_rn(l_run) : 0.f;
          if constexpr (SAFE) {  // special cases (gate, padded D) live in the SAFE variant only
            const int dreal = p.dreal;
            const size_t orow = ((p.swapped ? (size_t)i * p.B + b : (size_t)b * p.L + i) * p.H + si.h) * dreal;
            uint32_t ow[D / 2];
            if (p.gate) {  // fused output gate (OpenFold): o = sigmoid(G) * O, G read in the row's layout
              const uint4* g4 = (const uint4*)((const uint16_t*)p.gate + orow);
#pragma unroll
              for (int c = 0; c < D / 8; ++c) {
                if (c * 8 >= dreal) break;
                const uint4 gr = __ldg(g4 + c);
                const uint32_t gw[4] = {gr.x, gr.y, gr.z, gr.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int d = c * 8 + 2 * e;
                  const float2 g = unpack2<F16>(gw[e]);
                  const float o0 = __uint_as_float(ov[d]) * inv * sigmoidf_fast(g.x);
                  const float o1 = __uint_as_float(ov[d + 1]) * inv * sigmoidf_fast(g.y);
                  ow[d / 2] = F16 ? ptx::pack_f16(o0, o1) : ptx::pack_bf16(o0, o1);
                }
              }
            } else {
#pragma unroll
              for (int d = 0; d < D; d += 2) {
                const float o0 = __uint_as_float(ov[d]) * inv, o1 = __uint_as_float(ov[d + 1]) * inv;
                ow[d / 2] = F16 ? ptx::pack_f16(o0, o1) : ptx::pack_bf16(o0, o1);
              }
            }
            ptx::st_row16<D>((uint16_t*)p.o + orow, ow, dreal);
          } else {
            uint32_t ow[D / 2];
#pragma unroll
            for (int d = 0; d < D; d += 2) {
              const float o0 = __uint_as_float(ov[d]) * inv, o1 = __uint_as_float(ov[d + 1]) * inv;
              ow[d / 2] = F16 ? ptx::pack_f16(o0, o1) : ptx::pack_bf16(o0, o1);
            }
            ptx::st_row16<D>((uint16_t*)p.o + ((p.swapped ? (size_t)i * p.B + b : (size_t)b * p.L + i) * p.H + si.h) * D,
                             ow, D);
          }
          const float lv = l_run > 0.f ? (m_run + __log2f(l_run)) * kLn2 : -INFINITY;
          p.lse[((size_t)b * p.H + si.h) * p.L + i] = lv;
          if (SAFE && p.flag) {  // NumericError: a NaN input or no finite logit in the row
            bool nan = !isfinite(lv);
#pragma unroll
            for (int d = 0; d < D; ++d) nan |= isnan(__uint_as_float(ov[d]));
            flag_if(p.flag, nan);
          }
        }
      }
      if (resident) {
        // a warpgroup with no row in this segment still owes its release: wait for the fill first
        if (!released) {
          for (int s2 = 0; s2 < p.nKT; ++s2) ptx::mbar_wait(&bias_full[s2], bph);
          ptx::named_bar_sync(1 + wg, 128);  // every warp saw the fills before they are released
          if (tid_wg == 0)
            for (int s2 = 0; s2 < p.nKT; ++s2) ptx::mbar_arrive(&bias_empty[s2]);
        }
        bph ^= 1;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace tc
}  // namespace evo

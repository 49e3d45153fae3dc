// tc_bwd.cuh — K3: fused Evoformer attention backward on tcgen05 / TMEM / TMA (sm_100a).
//
// Reference semantics: attn_backward_tiled, /root/reference/proj/core/src/attention_tiled.cpp:182-340:
// P = exp(S - LSE) recomputed per tile, dV += P^T dO, dP = dO V^T, dS = P (dP - delta),
// dQ += dS K, dK += dS^T Q (dQ, dK scaled once), dBias[h] += sum_b dS (F32 accumulator).
//
// B200 layout. A CTA owns one (ob, h, 64-key tile) "unit" and a range of its MSA rows b; for each
// row it walks the query tiles (128 rows each):
//  * the pair-bias strip bias2[ob, h, :, keys] (all queries x 64 keys, bf16) is TMA-loaded once per
//    unit and stays in shared memory;
//  * the dBias2 strip (all queries x 64 keys, fp32) stays in TMEM for the whole unit: every row's
//    dS is reduced into it on chip (the broadcast-reverse sum of attention_tiled.cpp:318-323 done
//    in the kernel), and it leaves the SM once, as a fp32 red.add per unit — not once per row;
//  * S = Q K^T + bias1 and dP = dO V^T (M=128 queries, N=64 keys) land in double-buffered TMEM tiles
//    (bias1 rides along as one extra K=16 step: ones-column x bias1 row, see A_aug/B_aug);
//    four softmax warpgroups (16 keys each) rebuild P from LSE in the log2 domain, form
//    dS = P (dP - delta), add dS into the strip, and write P and dS as bf16 into 128B-swizzled
//    shared tiles that serve both as MN-major (P^T, dS^T) and K-major (dS) UMMA operands;
//  * dV += P^T dO and dK += dS^T Q accumulate over the query tiles in two M=64 TMEM accumulators
//    that share 32 columns (lanes 0-15 / 16-31 of each quadrant); dK/dV are stored once per row;
//  * dQ_partial = dS K (M=128) is drained by an epilogue warpgroup and added into an fp32 dQ
//    accumulator with TMA bulk reduce-add (one partial per 64-key tile), converted afterwards.
//  TMEM: S/dP buffers [0,256), dBias strip [256, 256+64*nQT), dQ at 448, dK|dV at 480 (nQT <= 3).
#pragma once
#include <type_traits>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace evo {
namespace tc {
namespace bk {

#ifndef EVO_BWD_ALT
#define EVO_BWD_ALT 1  // softmax warpgroups take turns on the steps: 0 all 4 on every step, 1 two groups of 2, 2 one at a time
#endif
constexpr int kBM = 128;   // queries per tile
constexpr int kBN = 64;    // keys per tile
// warps: 0 TMA producer, 1 gradient MMAs, 2 S/dP MMAs, 3..3+4*kSoftWG softmax warpgroups, then the epilogue WG
#ifndef EVO_BWD_KSTAGES
#define EVO_BWD_KSTAGES 2  // (K, V, bias1 chunk) ring depth
#endif
#ifndef EVO_BWD_QSTAGES
#define EVO_BWD_QSTAGES 4  // (Q, dO, lse, delta) ring depth of the unchunked variants
#endif
#ifndef EVO_BWD_PREFETCH
#define EVO_BWD_PREFETCH 0  // L2 prefetch of the next row's K / V / Q / dO / lse / delta by the producer
#endif
#ifndef EVO_BWD_SOFTWG
#define EVO_BWD_SOFTWG 4  // softmax warpgroups (fewer warpgroups: more registers per thread)
#endif
#ifndef EVO_BWD_UNROLL
#define EVO_BWD_UNROLL 1  // 1: a warpgroup's 16-key blocks of a step fully unrolled (loads of all blocks in flight)
#endif
constexpr int kSoftWG = EVO_BWD_SOFTWG;
constexpr int kKeysPerThread = 64 / kSoftWG;
// kGroups groups of softmax warpgroups take turns on the steps (step % kGroups): a group's warpgroup
// covers kGroups 16-key blocks of its step, so one group's TMEM / shared-memory phases overlap the
// other's exponentials instead of all warpgroups running the same phase at once
constexpr int kGroups = EVO_BWD_ALT == 2 ? 4 : EVO_BWD_ALT ? 2 : 1;
constexpr int kGroupThreads = 128 * kSoftWG / kGroups;
constexpr int kBlocksPerWG = 4 * kGroups / kSoftWG;  // 16-key blocks a warpgroup covers in each of its steps
constexpr int kCbUnroll = EVO_BWD_UNROLL ? kBlocksPerWG : 1;
static_assert(kBlocksPerWG >= 1 && kBlocksPerWG * kSoftWG == 4 * kGroups, "softmax warpgroup / group split");
constexpr int kSoftWarp0 = 3;
constexpr int kEpiWarp0 = kSoftWarp0 + 4 * kSoftWG;
constexpr int kThreads = (kEpiWarp0 + 4) * 32;
constexpr int kSoftThreads = 128 * kSoftWG;
constexpr uint32_t kEpiBar = 1 + kSoftWG;               // named barrier of the epilogue WG
constexpr int kAugA = kBM * 32, kAugB = 64 * 32;        // bias1 augmentation tiles (16 bf16 per row)
constexpr int kOnes = 16 * 32;                           // 16 x 16 bf16 ones: the dBias1 column-sum operand
constexpr int kIdent = 16 * 32;                          // 16 x 16 identity: dBias2 strip += dS I on the tensor pipe
constexpr uint32_t kStripCol = 256, kDqCol = 448, kDkvCol = 480;
constexpr uint32_t kDb1Col = 384;
#ifndef EVO_BWD_LATE_PDS
#define EVO_BWD_LATE_PDS 1  // softmax waits for its P/dS buffer only before the first store
#endif
#ifndef EVO_BWD_DS_TMEM
#define EVO_BWD_DS_TMEM 0  // 1: dS also written (bf16) into TMEM over its S columns: dQ and the dBias2 strip become
#endif                     // TS-MMAs (A from TMEM), 32 KB less shared-memory operand traffic per step
#ifndef EVO_BWD_POLY
#define EVO_BWD_POLY 0
#endif
#ifndef EVO_BWD_EXP
#define EVO_BWD_EXP 0  // timing experiments only (wrong results), bit mask: 1 no dK/dV MMAs, 2 no dQ MMA, 4 no bias LDS,
                       // 8 no P/dS stores, 16 no exponentials, 32 no dQ staging/reduce, 64 no dBias2 strip MMAs,
                       // 128 every row loads the Q / dO / lse / delta of row 0 (L2-resident), 256 no bias1 UMMA step
#endif  // dBias1 column sums (M=64, 16 columns) when requested: chunks of <= 2 q-tiles

template <int D, bool CH>
struct Cfg {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kTileQ = kBM * kRowBytes;    // Q or dO tile
  static constexpr int kTileK = kBN * kRowBytes;    // K or V tile
  // (Q, dO, lse, delta) ring: a slot refills only once the gradient MMAs of its step completed, so its
  // depth is the TMA slack. 4 deep with one fp32 dQ staging tile (C4: 574 vs 651 us at 3 deep); the
  // chunked variant stages dK/dV partials through the same tiles, and there two staging tiles with a
  // 3-deep ring win (C5: 44.8 vs 57.6 ms)
  static constexpr int kQStages = CH ? 3 : EVO_BWD_QSTAGES;
  static constexpr int kDqBufs = (EVO_BWD_EXP & 32) && !CH ? 0 : kQStages > 3 ? 1 : 2;  // fp32 dQ staging tiles
  static constexpr int kKStages = EVO_BWD_KSTAGES;  // (K, V, bias1 chunk) ring
  static constexpr int kBiasTile = kBM * kBN * 2;   // 16 KB
  static constexpr int kPdsTile = kBM * kBN * 2;    // 16 KB (P or dS, bf16)
  static constexpr int kDqStage = kBM * D * 4;      // fp32 dQ staging
};

struct Params {
  int B, N, L, H, Bo;
  int nQT, nKT;
  int nQC, nIC;      // query tiles per chunk (<= 3: the dBias2 strip of a chunk fits TMEM), chunks
  int nBT;           // pair-bias tiles resident in shared memory (nQC, or 0 without bias2)
  long long total;   // items = Bo*H*nKT*nIC*N
  int aligned, split;
  float scale, scale_log2;
  const void* bias1;    // [B, L] or null
  const float* lse2;    // [B, H, nQT*128] lse * log2e, +inf past L
  const float* delta;   // [B, H, nQT*128] rowsum(dO * O), 0 past L
  void* dk;             // [B, L, H, D] (nIC == 1: written directly)
  void* dv;
  int dkv_reduce;       // nIC > 1: dK/dV partials of each query chunk reduce-add into fp32 accumulators
  float* dbias2;        // [Bo, H, L, L] fp32 accumulator or null (a multicast address when dbias2_mc)
  float* dbias1;        // [B, L] fp32 accumulator or null: dBias1[b, j] = sum_{h,i} dS (the mask-bias gradient)
  int dbias2_mc;        // flush the dBias2 strip with multimem.red into every rank's replica
  int has_bias2;
  int aug;             // extra K-step adding bias1 / scale (bias1 present or L % 64 != 0)
  uint32_t aug_c;      // (c_lo << 16) | c_hi: 16-bit split of 1/scale
  unsigned long long* trace;  // bring-up timeline of CTA 0 (null in production)
  int swapped;  // 1: q/k/v/o/dO/dQ/dK/dV are [L, B, H, D] (raw msa_col / tri_end layout)
};

// Fields only the SAFE kernel variants read. They extend the parameter block of those variants alone:
// the hot variants keep the block they were tuned with (extra fields measurably changed their code
// generation).
struct Extra {
  // Row window of this launch: rows n in [n0w, n0w + nw) of every outer batch (items walk the window;
  // the deterministic mode bounds its partial buffers by launching window after window)
  int n0w, nw;
  // Deterministic mode (AccumPolicy::deterministic, attention_tiled.cpp:246-252): dQ partials of each
  // key tile and the chunked dK/dV partials are TMA-STORED to per-tile / per-chunk slots (window rows
  // jt*Bw + wrow) and summed in order after the kernel; dBias1 partials go to db1_part; the dBias2
  // strip flushes of the CTAs sharing a unit are serialised by part through `tickets`.
  int det;
  int win;          // windowed accumulators (not det): the fp32 dQ (dK, dV) accumulators hold one row window
  int* tickets;     // [units of the window]: strip flushes done (kSoftWG per part), zeroed by the preamble
  float* db1_part;  // [H * nIC][Bw][L] when det and dbias1
  int* flag;        // numeric-check flag (NaN dK / dV) or null
  int dreal;        // head dim in memory (D = 16 kernels serve D = 8 with zero-padded TMA boxes)
};
struct ParamsSafe : Params {
  Extra x;
};
template <bool SAFE>
using ParamsT = typename std::conditional<SAFE, ParamsSafe, Params>::type;
// The extension as the kernel sees it: the launch's values (SAFE) or the constants of a plain launch
template <bool SAFE, int D>
__device__ __forceinline__ Extra extra_of(const ParamsT<SAFE>& p) {
  if constexpr (SAFE) {
    return p.x;
  } else {
    return Extra{0, p.N, 0, 0, nullptr, nullptr, nullptr, D};
  }
}

// CTA-0 timeline of steps [kTrFirst, kTrFirst + 64): 8 events x 64 steps (bring-up aid)
constexpr uint32_t kTrFirst = 100;
enum BwdTrace { kTbSIssue = 0, kTbSSeen = 1, kTbPds0 = 2, kTbPds1 = 3, kTbGrads = 4, kTbDqSeen = 5, kTbDqOut = 6,
                kTbQFull = 7, kTbProdQ = 8, kTbKFull = 9, kTbGradsStart = 10, kTbLoopTop = 11 };
__device__ __forceinline__ void trace(const Params& p, int ev, uint32_t step) {
  if constexpr (EVO_TRACE) {
    if (p.trace && blockIdx.x == 0 && step - kTrFirst < 64u) p.trace[ev * 64 + (step - kTrFirst)] = clock64();
  }
}

struct Walker {
  long long t0, t1, N;
  __device__ long long seg_end(long long s) const {
    const long long e = (s / N + 1) * N;
    return e < t1 ? e : t1;
  }
};
// nw: rows walked per unit — the launch's row window (SAFE variants) or all N rows
__device__ __forceinline__ Walker make_walker(const Params& p, int nw) {
  if (p.aligned) {
    const long long unit = blockIdx.x / p.split, part = blockIdx.x % p.split;
    const long long base = unit * nw;
    return Walker{base + nw * part / p.split, base + nw * (part + 1) / p.split, nw};
  }
  return Walker{p.total * blockIdx.x / gridDim.x, p.total * (blockIdx.x + 1) / gridDim.x, nw};
}
struct Unit {
  int ob, h, jt, ic, it0, it1, n0;  // query tiles [it0, it1) of chunk ic
};
__device__ __forceinline__ Unit unit_of(long long s0, const Params& p, int nw) {
  Unit u;
  long long x = s0 / nw;
  u.n0 = (int)(s0 - x * nw);  // window-local row
  u.ic = (int)(x % p.nIC);
  x /= p.nIC;
  u.jt = (int)(x % p.nKT);
  x /= p.nKT;
  u.h = (int)(x % p.H);
  u.ob = (int)(x / p.H);
  u.it0 = u.ic * p.nQC;
  u.it1 = min(u.it0 + p.nQC, p.nQT);
  return u;
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Index of this CTA among the CTAs whose item ranges intersect `unit` (0 = the first): the flush
// order of the deterministic dBias2 reduction.
__device__ __forceinline__ int unit_part(const Params& p, long long unit, int nw) {
  if (p.aligned) return (int)(blockIdx.x % p.split);
  const long long first = unit * nw;  // first item of the unit; CTA c covers [total*c/G, total*(c+1)/G)
  long long c = first * gridDim.x / p.total;
  while (c > 0 && p.total * c / gridDim.x > first) --c;
  while (p.total * (c + 1) / gridDim.x <= first) ++c;
  return (int)(blockIdx.x - c);
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}
template <bool F16>
__device__ __forceinline__ float2 unpack2(uint32_t w) {
  if constexpr (F16) {
    __half2 hh = *reinterpret_cast<__half2*>(&w);
    return __half22float2(hh);
  } else {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  }
}
__device__ __forceinline__ void red_v4(float* gaddr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(gaddr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
// NVLS: one add through an NVSwitch multicast address lands in every GPU's replica (the cross-GPU
// dBias2 reduction fused into the kernel's strip flush — no separate all-reduce)
__device__ __forceinline__ void red_v4_multimem(float* mc_addr, float a, float b, float c, float d) {
  asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc_addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

// CH: the query axis is split into chunks (L > 384); SW: raw [L, B, H, D] layout; SAFE: the deterministic
// and numeric-check code paths are compiled in (selected at run time by p.det / p.flag)
template <int D, bool F16, bool CH, bool SW, bool SAFE>
__global__ void __launch_bounds__(kThreads, 1)
    bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
               const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmdQ,
               const __grid_constant__ CUtensorMap tmdK, const __grid_constant__ CUtensorMap tmdV,
               const ParamsT<SAFE> p) {
  using C = Cfg<D, CH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // ---- shared memory carve-up (all operand tiles 1024-aligned)
  uint8_t* sQ = smem;                                          // [QS] Q tiles
  uint8_t* sdO = sQ + C::kQStages * C::kTileQ;                 // [QS] dO tiles
  uint8_t* sK = sdO + C::kQStages * C::kTileQ;                 // [KS] K tiles
  uint8_t* sV = sK + C::kKStages * C::kTileK;                  // [KS] V tiles
  uint8_t* sP = sV + C::kKStages * C::kTileK;                  // [2] P tiles (bf16, SW128)
  uint8_t* sdS = sP + 2 * C::kPdsTile;                         // [2] dS tiles
  uint8_t* sBias = sdS + 2 * C::kPdsTile;                      // [nQT] bias strip tiles
  float* sDq = (float*)(sBias + (size_t)p.nBT * C::kBiasTile);  // dQ staging (fp32 128 x D)
  uint8_t* sAaug = (uint8_t*)(sDq + C::kDqBufs * kBM * D);     // 128 x 16 (1/scale split), SW32
  uint8_t* sBaug = sAaug + kAugA;                              // [KS] 64 x 16 (bias1 per key), SW32
  uint8_t* sOnes = sBaug + C::kKStages * kAugB;                // 16 x 16 ones (dBias1 = dS^T 1), SW32
  uint8_t* sIdent = sOnes + kOnes;                             // 16 x 16 identity (strip += dS I), SW32
  float* sLse = (float*)(sIdent + kIdent);                     // [QS][128] lse * log2e
  float* sDel = sLse + C::kQStages * kBM;                      // [QS][128] delta
  uint16_t* sB1 = (uint16_t*)(sDel + C::kQStages * kBM);       // [KS][64] bias1 chunk (raw)
  uint64_t* bars = (uint64_t*)(sB1 + C::kKStages * 64);
  uint64_t* q_full = bars;                          // [QS]
  uint64_t* q_empty = q_full + C::kQStages;         // [QS]
  uint64_t* k_full = q_empty + C::kQStages;         // [KS]
  uint64_t* k_empty = k_full + C::kKStages;         // [KS]
  uint64_t* s_full = k_empty + C::kKStages;         // [2] S and dP of a step computed
  uint64_t* s_free = s_full + 2;                    // [2] softmax done reading S/dP of a buffer
  uint64_t* pds_full = s_free + 2;                  // [2] P/dS of a step written
  uint64_t* pds_free = pds_full + 2;                // [2] MMAs reading that P/dS buffer done
  uint64_t* dq_full = pds_free + 2;                 // [1] dQ partial computed
  uint64_t* dq_free = dq_full + 1;                  // [1] dQ drained from TMEM
  uint64_t* kv_done = dq_free + 1;                  // [1] dK/dV of a row complete
  uint64_t* kv_free = kv_done + 1;                  // [1] dK/dV read out
  uint64_t* bias_full = kv_free + 1;                // [1] bias strip of the unit landed
  uint64_t* bias_empty = bias_full + 1;             // [1] strip readers done (one arrival per WG)
  uint64_t* strip_full = bias_empty + 1;            // [1] last dBias2 strip MMA of a unit completed
  uint32_t* tmem_slot = (uint32_t*)(strip_full + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const Extra X = extra_of<SAFE, D>(p);  // compile-time constants in the plain variants
  const Walker W = make_walker(p, X.nw);
  constexpr uint32_t kSw = ptx::swizzle_code(C::kRowBytes);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kQStages; ++s) { ptx::mbar_init(&q_full[s], 1); ptx::mbar_init(&q_empty[s], 1); }
    for (int s = 0; s < C::kKStages; ++s) { ptx::mbar_init(&k_full[s], 1); ptx::mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      // buffer s serves the group of steps s (mod 2); with dS in TMEM it frees when the gradient MMAs
      // reading dS from it completed, else when the softmax threads loaded S and dP
      ptx::mbar_init(&s_free[s], EVO_BWD_DS_TMEM ? 1 : kGroupThreads);
      ptx::mbar_init(&pds_full[s], kGroupThreads);
      ptx::mbar_init(&pds_free[s], 1);
    }
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_free, 128);
    ptx::mbar_init(kv_done, 1);
    ptx::mbar_init(kv_free, 128);
    ptx::mbar_init(bias_full, 1);
    ptx::mbar_init(bias_empty, kSoftWG);
    ptx::mbar_init(strip_full, 1);
    ptx::fence_barrier_init();
  }
  // A_aug: row i = (c_hi, c_lo, 0, ...): one extra K=16 step of S = Q K^T adds (c_hi + c_lo) * B_aug[j][0..1]
  // = bias1[j] / scale (two-term split of 1/scale, exact to ~2^-16). 16B chunk 0 of a 32B row sits at
  // chunk position (i >> 2) & 1 under the 32B swizzle.
  for (int i = threadIdx.x; i < 16 * 2; i += blockDim.x) {  // ones (1.0 in bf16 / f16), layout-agnostic
    const uint32_t one = F16 ? 0x3C003C00u : 0x3F803F80u;
    ((uint4*)sOnes)[i] = make_uint4(one, one, one, one);
  }
  for (int i = threadIdx.x; i < 16; i += blockDim.x) {  // identity row i: element i = 1 in chunk (i >> 3) ^ ((i >> 2) & 1)
    const uint32_t one = F16 ? 0x3C00u : 0x3F80u;
    uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    w[(i & 7) >> 1] = (i & 1) ? (one << 16) : one;
    uint4* row = (uint4*)(sIdent + i * 32);
    const uint32_t c = (uint32_t)(i >> 3) ^ (uint32_t)((i >> 2) & 1);
    row[c] = make_uint4(w[0], w[1], w[2], w[3]);
    row[c ^ 1] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int i = threadIdx.x; i < kBM; i += blockDim.x) {
    const uint32_t c = (uint32_t)((i >> 2) & 1);
    uint4* row = (uint4*)(sAaug + i * 32);
    row[c] = make_uint4(p.aug_c, 0u, 0u, 0u);
    row[c ^ 1] = make_uint4(0u, 0u, 0u, 0u);
  }
  ptx::fence_proxy_async_smem();
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // launched as a programmatic dependent of the preamble: the prologue above overlapped its tail;
  // lse2 / delta / the zeroed accumulators are read below
  ptx::pdl_wait();
  ptx::pdl_launch_dependents();

  if (warp == 0) {
    if (ptx::elect_one()) {
      // ===================================================== TMA producer
      ptx::tma_prefetch(&tmQ); ptx::tma_prefetch(&tmK); ptx::tma_prefetch(&tmV); ptx::tma_prefetch(&tmdO);
      if (p.has_bias2) ptx::tma_prefetch(&tmB2);
      int qs = 0; uint32_t qph = 0;
      int ks = 0; uint32_t kph = 0;
      uint32_t bph = 0, pstep = 0;
      for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
        const int cnt = (int)(W.seg_end(s0) - s0);
        const Unit u = unit_of(s0, p, X.nw);
        const int plane = u.ob * p.H + u.h;
        if (p.has_bias2) {
          ptx::mbar_wait(bias_empty, bph ^ 1);
          ptx::mbar_expect_tx(bias_full, ((CH ? u.it1 : p.nQT) - (CH ? u.it0 : 0)) * C::kBiasTile);
          for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it)
            ptx::tma_load_3d(sBias + (size_t)(it - (CH ? u.it0 : 0)) * C::kBiasTile, &tmB2, bias_full, u.jt * kBN, it * kBM, plane);
          bph ^= 1;
        }
        int n = u.n0;
        for (int a = 0; a < cnt; ++a, ++n) {
          const int b = u.ob * p.N + X.n0w + n;
          if (EVO_BWD_PREFETCH && a + 1 < cnt) {
            // the next row's operands into L2 one row (nQT steps) ahead: its Q-stage loads are issued
            // only when the gradient MMAs of step - kQStages complete, and then sit on the S -> softmax
            // chain; from L2 they land in about half the HBM latency
            ptx::tma_prefetch_4d(&tmK, 0, u.h, u.jt * kBN, b + 1);
            ptx::tma_prefetch_4d(&tmV, 0, u.h, u.jt * kBN, b + 1);
            for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it) {
              ptx::tma_prefetch_4d(&tmQ, 0, u.h, it * kBM, b + 1);
              ptx::tma_prefetch_4d(&tmdO, 0, u.h, it * kBM, b + 1);
            }
            const size_t r1 = ((size_t)(b + 1) * p.H + u.h) * (p.nQT * kBM) + (size_t)(CH ? u.it0 : 0) * kBM;
            const uint32_t nb = (uint32_t)((CH ? u.it1 - u.it0 : p.nQT) * kBM * 4);
            ptx::bulk_prefetch_l2(p.lse2 + r1, nb);
            ptx::bulk_prefetch_l2(p.delta + r1, nb);
          }
          // K, V (and the bias1 chunk) of this row's key tile
          ptx::mbar_wait(&k_empty[ks], kph ^ 1);
          const int nk = min(kBN, p.L - u.jt * kBN);  // keys of this tile (multiple of 8)
          const uint32_t b1bytes = p.bias1 ? (uint32_t)nk * 2 : 0u;
          ptx::mbar_expect_tx(&k_full[ks], 2 * C::kTileK + b1bytes);
          ptx::tma_load_4d(sK + ks * C::kTileK, &tmK, &k_full[ks], 0, u.h, u.jt * kBN, b);
          ptx::tma_load_4d(sV + ks * C::kTileK, &tmV, &k_full[ks], 0, u.h, u.jt * kBN, b);
          if (b1bytes)
            bulk_g2s(ptx::smem_u32(sB1 + ks * 64), (const uint16_t*)p.bias1 + (size_t)b * p.L + u.jt * kBN, b1bytes,
                     &k_full[ks]);
          if (++ks == C::kKStages) { ks = 0; kph ^= 1; }
          for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it) {
            ptx::mbar_wait(&q_empty[qs], qph ^ 1);
            trace(p, kTbProdQ, pstep++);
            ptx::mbar_expect_tx(&q_full[qs], 2 * C::kTileQ + 2 * kBM * 4);
            const int bq = (EVO_BWD_EXP & 128) ? 0 : b;
            ptx::tma_load_4d(sQ + qs * C::kTileQ, &tmQ, &q_full[qs], 0, u.h, it * kBM, bq);
            ptx::tma_load_4d(sdO + qs * C::kTileQ, &tmdO, &q_full[qs], 0, u.h, it * kBM, bq);
            const size_t row0 = ((size_t)bq * p.H + u.h) * (p.nQT * kBM) + (size_t)it * kBM;
            bulk_g2s(ptx::smem_u32(sLse + qs * kBM), p.lse2 + row0, kBM * 4, &q_full[qs]);
            bulk_g2s(ptx::smem_u32(sDel + qs * kBM), p.delta + row0, kBM * 4, &q_full[qs]);
            if (++qs == C::kQStages) { qs = 0; qph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================================================== gradient MMA issuer (converged warp, one elected
    // lane issues; descriptors stay in uniform registers). For every (row, q-tile) step t, once P/dS(t)
    // are in shared memory: dV += P^T dO, dK += dS^T Q (M=64 accumulators), dQ_t = dS K.
    const uint32_t idKV = ptx::instr_desc(64, D, F16, true, true);       // dV, dK: MN-major A and B
    const uint32_t idQ = ptx::instr_desc(kBM, D, F16, false, true);      // dQ: K-major A, MN-major B
    // descriptor low words (start >> 4 | LBO >> 4 << 16) of stage 0; stages and K-steps are added
    constexpr uint32_t kHiMN = ptx::desc_hi(8 * C::kRowBytes, kSw);   // MN-major dO/Q/K as B
    constexpr uint32_t kHiP = ptx::desc_hi(1024, 2);                  // P, dS tiles (SW128, both majors)
    constexpr uint32_t kRow16 = C::kRowBytes;                         // 16 rows of 2*D bytes, >> 4
    const uint32_t q0n = ptx::desc_lo(ptx::smem_u32(sQ), 16 * C::kRowBytes);
    const uint32_t do0n = ptx::desc_lo(ptx::smem_u32(sdO), 16 * C::kRowBytes);
    const uint32_t k0n = ptx::desc_lo(ptx::smem_u32(sK), 16 * C::kRowBytes);
    const uint32_t p0mn = ptx::desc_lo(ptx::smem_u32(sP), 1024), ds0mn = ptx::desc_lo(ptx::smem_u32(sdS), 1024);
    const uint32_t ds0k = ptx::desc_lo(ptx::smem_u32(sdS), 16);
    const uint32_t tdKV = tmem + kDkvCol, tdQ = tmem + kDqCol;
    const uint32_t idB1 = ptx::instr_desc(64, 16, F16, true, false);  // dBias1: MN-major dS^T, K-major ones
    const uint64_t bOnes = ptx::desc_make(ptx::desc_lo(ptx::smem_u32(sOnes), 16), ptx::desc_hi(256, 6));
    const uint32_t idStrip = ptx::instr_desc(kBM, 16, F16, false, false);  // strip block += dS block x I16
    const uint64_t bIdent = ptx::desc_make(ptx::desc_lo(ptx::smem_u32(sIdent), 16), ptx::desc_hi(256, 6));
    int qs = 0, ks = 0;
    uint32_t step = 0, rows = 0;
    for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
      const int cnt = (int)(W.seg_end(s0) - s0);
      const Unit u = unit_of(s0, p, X.nw);
      for (int a = 0; a < cnt; ++a) {
        for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it) {
          const uint32_t sb = step & 1, ph = (step >> 1) & 1;
          const bool first = it == (CH ? u.it0 : 0), last = it == (CH ? u.it1 : p.nQT) - 1;
          ptx::mbar_wait_spin(&pds_full[sb], ph);
          if (first) {  // first q-tile of a row overwrites dK/dV: previous row must be read out
            ptx::mbar_wait_spin(kv_free, (rows & 1) ^ 1);
            ++rows;
          }
          ptx::mbar_wait_spin(dq_free, (step & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t pA = p0mn + sb * (C::kPdsTile >> 4);
          const uint32_t dsA = ds0mn + sb * (C::kPdsTile >> 4);
          const uint32_t dsK = ds0k + sb * (C::kPdsTile >> 4);
          const uint32_t qB = q0n + qs * (C::kTileQ >> 4);
          const uint32_t doB = do0n + qs * (C::kTileQ >> 4);
          const uint32_t kB = k0n + ks * (C::kTileK >> 4);
          if (ptx::elect_one()) {
            trace(p, kTbGradsStart, step);
            // dQ first: the epilogue drains it while dK / dV run, so the next step's dQ never waits
#pragma unroll
            for (int kk = 0; kk < ((EVO_BWD_EXP & 2) ? 0 : kBN / 16); ++kk) {  // dQ = dS K: K = 64 keys
              if (EVO_BWD_DS_TMEM)  // A = dS block kk, bf16 in TMEM at S columns [16kk, 16kk + 8)
                ptx::mma_ts(tdQ, tmem + sb * 128 + kk * 16, ptx::desc_make(kB + kk * kRow16, kHiMN), idQ, kk > 0);
              else  // A = dS from shared memory (+32 B in the dS rows)
                ptx::mma_ss(tdQ, ptx::desc_make(dsK + kk * 2, kHiP), ptx::desc_make(kB + kk * kRow16, kHiMN), idQ,
                            kk > 0);
            }
            ptx::tc_commit(dq_full);
#pragma unroll
            for (int kk = 0; kk < ((EVO_BWD_EXP & 1) ? 0 : kBM / 16); ++kk) {  // K = 128 queries: 16 rows per step
              // A = P^T / dS^T: MN-major SW128 (64 keys wide), 16 query rows = 2 x 8-row atoms (+2048 B)
              // B = dO / Q: MN-major (D wide), 16 query rows (+16 * 2D B)
              const uint32_t acc = (!first || kk > 0) ? 1u : 0u;
              ptx::mma_ss(tdKV + (16u << 16), ptx::desc_make(pA + kk * 128, kHiP),
                          ptx::desc_make(doB + kk * kRow16, kHiMN), idKV, acc);  // dV (lanes 16-31 of each quadrant)
              ptx::mma_ss(tdKV, ptx::desc_make(dsA + kk * 128, kHiP), ptx::desc_make(qB + kk * kRow16, kHiMN), idKV,
                          acc);                                                  // dK (lanes 0-15)
              if (p.dbias1)  // dBias1 partial: dS^T (keys x queries) times a ones column block
                ptx::mma_ss(tmem + kDb1Col, ptx::desc_make(dsA + kk * 128, kHiP), bOnes, idB1, acc);
            }
            if (p.dbias2) {
              // dBias2 strip (this q-tile's 128 x 64 fp32 block in TMEM) += dS: four N = 16 column blocks,
              // dS block kk (K-major, 16 keys) times a 16 x 16 identity; the unit's first row initialises
              const uint32_t st = tmem + kStripCol + (uint32_t)(it - (CH ? u.it0 : 0)) * 64;
#pragma unroll
              for (int kk = 0; kk < ((EVO_BWD_EXP & 64) ? 0 : kBN / 16); ++kk) {
                if (EVO_BWD_DS_TMEM)
                  ptx::mma_ts(st + kk * 16, tmem + sb * 128 + kk * 16, bIdent, idStrip, a > 0 ? 1u : 0u);
                else
                  ptx::mma_ss(st + kk * 16, ptx::desc_make(dsK + kk * 2, kHiP), bIdent, idStrip, a > 0 ? 1u : 0u);
              }
              if (last && a == cnt - 1) ptx::tc_commit(strip_full);
            }
            ptx::tc_commit(&pds_free[sb]);
            if (EVO_BWD_DS_TMEM) ptx::tc_commit(&s_free[sb]);  // dS (in the S/dP buffer) read
            ptx::tc_commit(&q_empty[qs]);  // S/dP of this step completed before P/dS existed
            if (last) {
              ptx::tc_commit(kv_done);
              ptx::tc_commit(&k_empty[ks]);
            }
            trace(p, kTbGrads, step);
          }
          __syncwarp();
          ++step;
          if (++qs == C::kQStages) qs = 0;
        }
        if (++ks == C::kKStages) ks = 0;
      }
    }
  } else if (warp == 2) {
    // ===================================================== S / dP issuer (runs up to two steps ahead)
    const uint32_t idS = ptx::instr_desc(kBM, kBN, F16, false, false);   // S, dP: K-major A, K-major B
    constexpr uint32_t kHiK = ptx::desc_hi(8 * C::kRowBytes, kSw);
    constexpr uint32_t kHiAug = ptx::desc_hi(256, 6);                  // 32-byte rows, SW32
    const uint32_t q0 = ptx::desc_lo(ptx::smem_u32(sQ), 16), do0 = ptx::desc_lo(ptx::smem_u32(sdO), 16);
    const uint32_t k0 = ptx::desc_lo(ptx::smem_u32(sK), 16), v0 = ptx::desc_lo(ptx::smem_u32(sV), 16);
    const uint32_t aA = ptx::desc_lo(ptx::smem_u32(sAaug), 16), aB0 = ptx::desc_lo(ptx::smem_u32(sBaug), 16);
    int qs = 0; uint32_t qph = 0;
    int ks = 0; uint32_t kph = 0;
    uint32_t step = 0;
    for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
      const int cnt = (int)(W.seg_end(s0) - s0);
      const Unit u = unit_of(s0, p, X.nw);
      for (int a = 0; a < cnt; ++a) {
        ptx::mbar_wait(&k_full[ks], kph);
        if (p.aug) {
          // B_aug row j = (b1[j], b1[j] or 0 if non-finite) for keys < L, (-inf, 0) past L; 2 rows per lane
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jj = lane + 32 * h;
            const bool in = u.jt * kBN + jj < p.L;
            uint32_t v0b = 0u, v1b = 0u;
            if (!in) {
              v0b = F16 ? 0xFC00u : 0xFF80u;
            } else if (p.bias1) {
              v0b = sB1[ks * 64 + jj];
              const bool fin = F16 ? (v0b & 0x7C00u) != 0x7C00u : (v0b & 0x7F80u) != 0x7F80u;
              v1b = fin ? v0b : 0u;
            }
            const uint32_t c = (uint32_t)((jj >> 2) & 1);
            uint4* row = (uint4*)(sBaug + ks * kAugB + jj * 32);
            row[c] = make_uint4(v0b | (v1b << 16), 0u, 0u, 0u);
            row[c ^ 1] = make_uint4(0u, 0u, 0u, 0u);
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
        }
        if (lane == 0) trace(p, kTbKFull, step);
        const uint32_t kA = k0 + ks * (C::kTileK >> 4);
        const uint32_t vA = v0 + ks * (C::kTileK >> 4);
        const uint32_t bA = aB0 + ks * (kAugB >> 4);
        for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it) {
          const uint32_t sb = step & 1;
          ptx::mbar_wait(&q_full[qs], qph);
          if (lane == 0) trace(p, kTbQFull, step);
          ptx::mbar_wait(&s_free[sb], ((step >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t qA = q0 + qs * (C::kTileQ >> 4);
          const uint32_t doA = do0 + qs * (C::kTileQ >> 4);
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {  // +32 B along the K-major rows
              ptx::mma_ss(tmem + sb * 128, ptx::desc_make(qA + kk * 2, kHiK), ptx::desc_make(kA + kk * 2, kHiK), idS,
                          kk > 0);  // S
              ptx::mma_ss(tmem + sb * 128 + 64, ptx::desc_make(doA + kk * 2, kHiK), ptx::desc_make(vA + kk * 2, kHiK),
                          idS, kk > 0);  // dP
            }
            if (p.aug && !(EVO_BWD_EXP & 256)) ptx::mma_ss(tmem + sb * 128, ptx::desc_make(aA, kHiAug), ptx::desc_make(bA, kHiAug), idS, 1u);
            ptx::tc_commit(&s_full[sb]);
            trace(p, kTbSIssue, step);
          }
          __syncwarp();
          if (EVO_TRACE && p.trace && blockIdx.x == 0 && step - kTrFirst < 64u) {  // bring-up: S completion time
            ptx::mbar_wait(&s_full[sb], (step >> 1) & 1);
            if (lane == 0) trace(p, kTbLoopTop, step);
          }
          ++step;
          if (++qs == C::kQStages) { qs = 0; qph ^= 1; }
        }
        if (++ks == C::kKStages) { ks = 0; kph ^= 1; }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ===================================================== softmax warpgroups (kSoftWG x 16 keys)
    const int wg = (warp - kSoftWarp0) / 4;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                 // query row in tile == TMEM lane
    const int tid_wg = (warp - kSoftWarp0 - 4 * wg) * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t col = (uint32_t)(wg * kKeysPerThread);  // this warpgroup's strip columns (flush)
    const int grp = wg / (kSoftWG / kGroups), sub = wg % (kSoftWG / kGroups);
    const float2 scl2 = make_float2(p.scale_log2, p.scale_log2);
    const float2 lg2 = make_float2(kLog2e, kLog2e);
    const uint32_t r7 = (uint32_t)(r & 7) << 4;
    int qs = 0; uint32_t qph = 0;
    uint32_t step = 0, bph = 0, uph = 0;
    for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
      const int cnt = (int)(W.seg_end(s0) - s0);
      const Unit u = unit_of(s0, p, X.nw);
      if (p.has_bias2) ptx::mbar_wait(bias_full, bph);
      for (int a = 0; a < cnt; ++a) {
        for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it) {
          const uint32_t sb = step & 1, ph = (step >> 1) & 1;
          if ((int)(step % kGroups) != grp) {  // the other group's step
            ++step;
            if (++qs == C::kQStages) { qs = 0; qph ^= 1; }
            continue;
          }
          ptx::mbar_wait(&q_full[qs], qph);
          const float lse2 = ptx::lds_f32(ptx::smem_u32(sLse + qs * kBM + r));
          const float dl = ptx::lds_f32(ptx::smem_u32(sDel + qs * kBM + r));
          const float2 nl = make_float2(-lse2, -lse2);
          const float2 nd = make_float2(-dl, -dl);
          ptx::mbar_wait(&s_full[sb], ph);
          if (tid_wg == 0 && wg == 0) trace(p, kTbSSeen, step);
          if (!EVO_BWD_LATE_PDS) ptx::mbar_wait(&pds_free[sb], ph ^ 1);  // P/dS buffer sb: MMAs of step-2 done
          ptx::tc_fence_after();
          const uint32_t bt = ptx::smem_u32(sBias + (size_t)(it - (CH ? u.it0 : 0)) * C::kBiasTile) + r * 128;
          const uint32_t pbase = ptx::smem_u32(sP + sb * C::kPdsTile) + r * 128;
          const uint32_t dbase = ptx::smem_u32(sdS + sb * C::kPdsTile) + r * 128;
#pragma unroll(kCbUnroll)
          for (int cb = 0; cb < kBlocksPerWG; ++cb) {
            const int kb = sub * kBlocksPerWG + cb;  // 16-key block of the step
            const uint32_t col = (uint32_t)(kb * 16);
            // all loads of the block in flight together: S, dP (TMEM) and the bias2 row (smem)
            uint32_t sv[16], dp[16];
            ptx::tmem_ld16(tmem + lane_off + sb * 128 + col, sv);
            ptx::tmem_ld16(tmem + lane_off + sb * 128 + 64 + col, dp);
            uint4 braw[2] = {make_uint4(0u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u)};
            if (p.has_bias2 && !(EVO_BWD_EXP & 4)) {
              braw[0] = lds128(bt + ((uint32_t)((2 * kb) << 4) ^ r7));
              braw[1] = lds128(bt + ((uint32_t)((2 * kb + 1) << 4) ^ r7));
            }
            ptx::tmem_ld_wait();
            if (!EVO_BWD_DS_TMEM && cb == kBlocksPerWG - 1) {
              ptx::tc_fence_before();
              ptx::mbar_arrive(&s_free[sb]);  // S/dP buffer may be recomputed
            }
            uint32_t pk[8], dk[8];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const uint32_t wv[4] = {braw[c].x, braw[c].y, braw[c].z, braw[c].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int k = c * 8 + 2 * e;
                const float2 bb = __ffma2_rn(unpack2<F16>(wv[e]), lg2, nl);  // bias2 * log2e - lse * log2e
                const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[k]), __uint_as_float(sv[k + 1])), scl2, bb);
                float2 pr;
                if (EVO_BWD_EXP & 16) {
                  pr = x;
                } else if (EVO_BWD_POLY && e == 3) {
                  pr = ex2_poly2(x);  // one pair in four on the FMA pipe (relieves MUFU)
                } else {
                  pr.x = ex2(x.x);
                  pr.y = ex2(x.y);
                }
                const float2 d =
                    __fmul2_rn(pr, __fadd2_rn(make_float2(__uint_as_float(dp[k]), __uint_as_float(dp[k + 1])), nd));
                pk[k / 2] = F16 ? ptx::pack_f16(pr.x, pr.y) : ptx::pack_bf16(pr.x, pr.y);
                dk[k / 2] = F16 ? ptx::pack_f16(d.x, d.y) : ptx::pack_bf16(d.x, d.y);
              }
            }
            if (EVO_BWD_DS_TMEM) ptx::tmem_st8(tmem + lane_off + sb * 128 + col, dk);  // dS over this block's S
            // P and dS -> shared (128B swizzle; chunks 2kb, 2kb+1 of row r). The buffer's previous
            // readers (the gradient MMAs of step - 2) are waited for only now: the first block's
            // loads and exponentials overlap their tail
            if (EVO_BWD_LATE_PDS && cb == 0) ptx::mbar_wait(&pds_free[sb], ph ^ 1);
#pragma unroll
            for (int c = 0; c < ((EVO_BWD_EXP & 8) ? 0 : 2); ++c) {
              const uint32_t off = (uint32_t)((2 * kb + c) << 4) ^ r7;
              sts128(pbase + off, make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
              sts128(dbase + off, make_uint4(dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]));
            }
          }
          if (EVO_BWD_DS_TMEM) {
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
          }
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&pds_full[sb]);
          if (tid_wg == 0 && (wg == 0 || wg == kSoftWG - 1)) trace(p, wg == 0 ? kTbPds0 : kTbPds1, step);
          ++step;
          if (++qs == C::kQStages) { qs = 0; qph ^= 1; }
        }
      }
      // ---- unit end: flush the dBias2 strip (fp32 red.add; one partial per CTA and unit) once the
      // unit's last strip MMA completed; the next unit's first strip MMA waits on this WG's next P/dS
      if (p.dbias2) {
        ptx::mbar_wait(strip_full, uph);
        uph ^= 1;
        ptx::tc_fence_after();
        const long long unit = s0 / X.nw;
        if (SAFE && X.det) {  // the unit's CTAs flush in part order: wait for the lower parts' warpgroups
          const int part = unit_part(p, unit, X.nw);
          if (tid_wg == 0)
            while (ld_acquire(X.tickets + unit) < part * kSoftWG) __nanosleep(64);
          ptx::named_bar_sync(1 + wg, 128);
        }
        for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it)
#pragma unroll
        for (int c16 = 0; c16 < kKeysPerThread; c16 += 16) {  // 16-column chunks of this warpgroup's strip
          const int j0 = u.jt * kBN + (int)col + c16;
          const int i = it * kBM + r;
          uint32_t st[16];
          ptx::tmem_ld16(tmem + lane_off + kStripCol + (it - (CH ? u.it0 : 0)) * 64 + col + c16, st);
          ptx::tmem_ld_wait();
          if (i < p.L) {
            float* dst = p.dbias2 + (((size_t)u.ob * p.H + u.h) * p.L + i) * p.L + j0;
#pragma unroll
            for (int k = 0; k < 16; k += 4)
              if (j0 + k < p.L) {
                if (p.dbias2_mc)
                  red_v4_multimem(dst + k, __uint_as_float(st[k]), __uint_as_float(st[k + 1]),
                                  __uint_as_float(st[k + 2]), __uint_as_float(st[k + 3]));
                else
                  red_v4(dst + k, __uint_as_float(st[k]), __uint_as_float(st[k + 1]), __uint_as_float(st[k + 2]),
                         __uint_as_float(st[k + 3]));
              }
          }
        }
      }
      if (p.dbias2 && SAFE && X.det) {  // this warpgroup's adds are performed before the next part may start
        __threadfence();
        ptx::named_bar_sync(1 + wg, 128);
        if (tid_wg == 0) atomicAdd(X.tickets + s0 / X.nw, 1);
      }
      if (p.dbias2) ptx::tc_fence_before();  // strip reads ordered before the next P/dS arrival (its MMAs overwrite)
      if (p.dbias2 && p.dbias2_mc) __threadfence_system();  // remote adds ordered before the ranks' barrier
      if (p.has_bias2) {
        ptx::named_bar_sync(1 + wg, 128);
        if (tid_wg == 0) ptx::mbar_arrive(bias_empty);
        bph ^= 1;
      }
    }
  } else {
    // ===================================================== epilogue warpgroup: dQ partials, dK/dV
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const int tid_e = (warp - kEpiWarp0) * 32 + lane;
    constexpr uint32_t kDqSwzMask = D == 32 ? 7u : D == 16 ? 3u : 1u;  // SW128 / SW64 / SW32
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    uint32_t step = 0, rows = 0;
    for (long long s0 = W.t0; s0 < W.t1; s0 = W.seg_end(s0)) {
      const int cnt = (int)(W.seg_end(s0) - s0);
      const Unit u = unit_of(s0, p, X.nw);
      int n = u.n0;
      for (int a = 0; a < cnt; ++a, ++n) {
        const int b = u.ob * p.N + X.n0w + n;
        const int wrow = u.ob * X.nw + n;  // row of the window (deterministic partial slots)
        const int Bw = p.Bo * X.nw;
        for (int it = (CH ? u.it0 : 0); it < (CH ? u.it1 : p.nQT); ++it) {
          // ---- dQ partial: TMEM -> staging (fp32, swizzled rows) -> TMA reduce-add into dQacc
          ptx::mbar_wait(dq_full, step & 1);
          if (tid_e == 0) trace(p, kTbDqSeen, step);
          ptx::tc_fence_after();
          uint32_t v[D];
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 16) ptx::tmem_ld16(tmem + lane_off + kDqCol + c0, *(uint32_t(*)[16])(&v[c0]));
          ptx::tmem_ld_wait();
          ptx::tc_fence_before();
          ptx::mbar_arrive(dq_free);
          float* stg = sDq + (C::kDqBufs == 2 ? (step & 1) * kBM * D : 0);
          if (EVO_BWD_EXP & 32) { ++step; continue; }
          if (tid_e == 0) {  // the reduce that last used this staging tile has read it
            if constexpr (C::kDqBufs == 2) ptx::bulk_wait_read<1>(); else ptx::bulk_wait_read<0>();
          }
          ptx::named_bar_sync(kEpiBar, 128);
          // row r of the staging tile, 16B chunks swizzled like the fp32 dQ tensor map (D*4-byte rows)
          const uint32_t sa = ptx::smem_u32(stg) + r * (D * 4);
#pragma unroll
          for (int c = 0; c < D; c += 4) {
            const uint32_t off = sa + c * 4;
            sts128(off ^ (((off >> 7) & kDqSwzMask) << 4), make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]));
          }
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(kEpiBar, 128);
          if (tid_e == 0) {
            if (SAFE && X.det) ptx::tma_store_4d(&tmdQ, stg, 0, u.h, it * kBM, u.jt * Bw + wrow);  // key tile jt's slot
            else ptx::tma_reduce_add_4d(&tmdQ, stg, 0, u.h, it * kBM, (SAFE && X.win) ? wrow : b);
            ptx::bulk_commit();
            trace(p, kTbDqOut, step);
          }
          ++step;
        }
        // ---- dK (x scale), dV of this row: lanes 0-15 hold dK rows, 16-31 dV rows of quadrant q4
        ptx::mbar_wait(kv_done, rows & 1);
        ptx::tc_fence_after();
        uint32_t v[D];
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 16) ptx::tmem_ld16(tmem + lane_off + kDkvCol + c0, *(uint32_t(*)[16])(&v[c0]));
        uint32_t b1v[4];
        if (p.dbias1) ptx::tmem_ld4(tmem + lane_off + kDb1Col, b1v);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(kv_free);
        if (p.dbias1 && lane < 16) {  // lanes 0-15 of quadrant q4 hold keys q4*16 + lane (M=64 layout)
          const int jj = u.jt * kBN + q4 * 16 + lane;
          if (jj < p.L) {
            if (SAFE && X.det) X.db1_part[(((size_t)u.h * p.nIC + u.ic) * Bw + wrow) * p.L + jj] = __uint_as_float(b1v[0]);
            else atomicAdd(p.dbias1 + (size_t)b * p.L + jj, __uint_as_float(b1v[0]));
          }
        }
        ++rows;
        const int krow = q4 * 16 + (lane & 15);
        const bool isk = lane < 16;
        if (CH && p.dkv_reduce) {
          // this query chunk's dK / dV partial of the row: fp32 rows (dK 0-63, dV 64-127) into a staging
          // tile, TMA reduce-add into the fp32 accumulators (scaled and converted after the kernel)
          float* stg = sDq + (C::kDqBufs == 2 ? (step & 1) * kBM * D : 0);
          if (tid_e == 0) {  // the previous user of this staging tile was read
            if constexpr (C::kDqBufs == 2) ptx::bulk_wait_read<1>(); else ptx::bulk_wait_read<0>();
          }
          ptx::named_bar_sync(kEpiBar, 128);
          const uint32_t sa = ptx::smem_u32(stg) + (krow + (isk ? 0 : 64)) * (D * 4);
#pragma unroll
          for (int c = 0; c < D; c += 4) {
            const uint32_t off = sa + c * 4;
            sts128(off ^ (((off >> 7) & kDqSwzMask) << 4), make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]));
          }
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(kEpiBar, 128);
          if (tid_e == 0) {
            if (SAFE && X.det) {  // chunk ic's slot
              ptx::tma_store_4d(&tmdK, stg, 0, u.h, u.jt * kBN, u.ic * Bw + wrow);
              ptx::tma_store_4d(&tmdV, stg + 64 * D, 0, u.h, u.jt * kBN, u.ic * Bw + wrow);
            } else {
              const int ar = (SAFE && X.win) ? wrow : b;
              ptx::tma_reduce_add_4d(&tmdK, stg, 0, u.h, u.jt * kBN, ar);
              ptx::tma_reduce_add_4d(&tmdV, stg + 64 * D, 0, u.h, u.jt * kBN, ar);
            }
            ptx::bulk_commit();
            ptx::bulk_wait_read<0>();  // the buffer is the next dQ step's
          }
          continue;
        }
        const int j = u.jt * kBN + krow;
        if (j < p.L) {
          if (SAFE && X.flag) {
            bool nan = false;
#pragma unroll
            for (int d = 0; d < D; ++d) nan |= isnan(__uint_as_float(v[d]));
            flag_if(X.flag, nan);
          }
          const float sc = isk ? p.scale : 1.f;
          uint32_t ow[D / 2];
#pragma unroll
          for (int d = 0; d < D; d += 2)
            ow[d / 2] = F16 ? ptx::pack_f16(__uint_as_float(v[d]) * sc, __uint_as_float(v[d + 1]) * sc)
                            : ptx::pack_bf16(__uint_as_float(v[d]) * sc, __uint_as_float(v[d + 1]) * sc);
          ptx::st_row16<D>((uint16_t*)(isk ? p.dk : p.dv) +
                               ((SW ? (size_t)j * p.B + b : (size_t)b * p.L + j) * p.H + u.h) * X.dreal,
                           ow, X.dreal);
        }
      }
    }
    if (tid_e == 0) ptx::bulk_wait<0>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// Backward preamble (one pass over dO and O): delta[b,h,i] = sum_d dO*O (attention_tiled.cpp:254-262)
// and lse2 = lse * log2e, both laid out [B, H, Lp] with the rows past L padded (+inf / 0).
// Thread per (b, i, h): D contiguous elements of dO and O, 16-byte loads (neighbouring threads read
// neighbouring rows: the dO / O streams, 2/3 of the bytes, are fully contiguous).
template <int D, typename T, bool SW>
__global__ void prep_kernel(const T* __restrict__ dout, const T* __restrict__ o, const float* __restrict__ lse,
                            float* __restrict__ lse2, float* __restrict__ delta_p, int B, int L, int H, int Lp,
                            float4* __restrict__ zero, long long nzero4, int* __restrict__ flag,
                            const T* __restrict__ gate, T* __restrict__ dog, T* __restrict__ dgate) {
  // gate (fused OpenFold output gate; dout, o are the gated output's gradient and value): also writes
  // dO = dout * sigmoid(G) for the main kernel and dG = dout * o * (1 - sigmoid(G)); delta = sum dout*o
  constexpr bool swapped = SW;
  ptx::pdl_launch_dependents();
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < nzero4; x += (long long)gridDim.x * blockDim.x)
    zero[x] = make_float4(0.f, 0.f, 0.f, 0.f);  // fp32 gradient accumulators of the main kernel
  const long long n = (long long)B * Lp * H;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
    const int h = (int)(x % H);
    const long long bi = x / H;
    const int i = (int)(bi % Lp);
    const int b = (int)(bi / Lp);
    const size_t orow = ((size_t)b * H + h) * Lp + i;
    if (i >= L) {
      lse2[orow] = INFINITY;
      delta_p[orow] = 0.f;
      continue;
    }
    const size_t r = ((swapped ? (size_t)i * B + b : (size_t)b * L + i) * H + h) * D;
    const uint4* a4 = (const uint4*)(dout + r);
    const uint4* b4 = (const uint4*)(o + r);
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
      const uint4 u = __ldg(a4 + c), w = __ldg(b4 + c);
      const T* ue = (const T*)&u;
      const T* we = (const T*)&w;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(to_f(ue[e]), to_f(we[e]), acc);
      if (gate) {
        const uint4 gv = __ldg((const uint4*)(gate + r) + c);
        const T* ge = (const T*)&gv;
        T go[8], gg[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float sg = sigmoidf_fast(to_f(ge[e])), d = to_f(ue[e]);
          go[e] = from_f<T>(d * sg);
          gg[e] = from_f<T>(d * to_f(we[e]) * (1.f - sg));
        }
        ((uint4*)(dog + r))[c] = *(const uint4*)go;
        ((uint4*)(dgate + r))[c] = *(const uint4*)gg;
      }
    }
    delta_p[orow] = acc;
    flag_if(flag, !isfinite(acc));  // NaN in dO (attention_tiled.cpp:209) or O
    lse2[orow] = lse[((size_t)b * H + h) * L + i] * kLog2e;
  }
}

// lse2 / delta padded to whole 128-row tiles: lse2 = lse * log2e (+inf past L), delta (0 past L)
static __global__ void pad_rows_kernel(const float* __restrict__ lse, const float* __restrict__ delta, float* __restrict__ lse2,
                                float* __restrict__ delta_p, int L, int Lp, long long rows, float4* __restrict__ zero,
                                long long nzero4) {
  ptx::pdl_launch_dependents();
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < nzero4; x += (long long)gridDim.x * blockDim.x)
    zero[x] = make_float4(0.f, 0.f, 0.f, 0.f);
  const long long n = rows * Lp;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
    const long long row = x / Lp;
    const int i = (int)(x - row * Lp);
    const bool in = i < L;
    lse2[x] = in ? lse[row * L + i] * kLog2e : INFINITY;
    delta_p[x] = in ? delta[row * L + i] : 0.f;
  }
}

__device__ __forceinline__ size_t out_off(size_t x, int B, int L, int HD, int swapped) {
  if (!swapped) return x;
  const size_t bi = x / (size_t)HD, e = x - bi * (size_t)HD;
  const size_t b = bi / (size_t)L, i = bi - b * (size_t)L;
  return (i * (size_t)B + b) * (size_t)HD + e;
}

// dQ (bf16/f16) = scale * dQacc (fp32); 8 elements per thread and iteration (n % 8 == 0: D >= 16):
// two 16-byte loads, one 16-byte store
// acc is canonical [B, L, H, D]; swapped writes the [L, B, H, D] layout (8-element groups stay in one row)
template <typename T, bool SW>
__global__ void dq_convert_kernel(const float* __restrict__ acc, T* __restrict__ dq, size_t n, float scale,
                                  int B, int L, int HD, int* __restrict__ flag) {
  constexpr int swapped = SW;
  ptx::pdl_wait();  // programmatic dependent of the main kernel
  ptx::pdl_launch_dependents();
  constexpr bool F16 = std::is_same<T, __half>::value;
  if (((uintptr_t)dq & 15) != 0) {  // caller buffer not 16-byte aligned: element stores
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n; x += (size_t)gridDim.x * blockDim.x)
      dq[out_off(x, B, L, HD, swapped)] = from_f<T>(acc[x] * scale);
    return;
  }
  for (size_t x = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 8; x < n; x += (size_t)gridDim.x * blockDim.x * 8) {
    const float4 a = __ldcs((const float4*)(acc + x)), c = __ldcs((const float4*)(acc + x + 4));
    if (flag)
      flag_if(flag, isnan(a.x) || isnan(a.y) || isnan(a.z) || isnan(a.w) || isnan(c.x) || isnan(c.y) || isnan(c.z) ||
                        isnan(c.w));
    uint4 w;
    w.x = F16 ? ptx::pack_f16(a.x * scale, a.y * scale) : ptx::pack_bf16(a.x * scale, a.y * scale);
    w.y = F16 ? ptx::pack_f16(a.z * scale, a.w * scale) : ptx::pack_bf16(a.z * scale, a.w * scale);
    w.z = F16 ? ptx::pack_f16(c.x * scale, c.y * scale) : ptx::pack_bf16(c.x * scale, c.y * scale);
    w.w = F16 ? ptx::pack_f16(c.z * scale, c.w * scale) : ptx::pack_bf16(c.z * scale, c.w * scale);
    *(uint4*)(dq + out_off(x, B, L, HD, swapped)) = w;
  }
}

// Deterministic mode: out = scale * (part[0] + part[1] + ... + part[np-1]) for the rows of one window,
// the partial slots (key tiles for dQ, query chunks for dK / dV) added in ascending order — the
// fixed-order reduction that makes two runs bit-identical. Element x of the window: window row
// wrow = ob * nw + r is canonical row b = ob * N + n0w + r; 8 elements per thread (HD % 8 == 0).
template <typename T, bool SW>
__global__ void det_convert_kernel(const float* __restrict__ part, int np, size_t pstride, T* __restrict__ out,
                                   size_t n, float scale, int B, int L, int HD, int N, int n0w, int nw,
                                   int* __restrict__ flag, int zero_after) {
  // zero_after (windowed accumulators, np == 1): the accumulator is left zeroed for the next window
  ptx::pdl_wait();  // programmatic dependent of the main kernel
  ptx::pdl_launch_dependents();
  constexpr bool F16 = std::is_same<T, __half>::value;
  const size_t rowlen = (size_t)L * HD;
  for (size_t x = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 8; x < n; x += (size_t)gridDim.x * blockDim.x * 8) {
    float a[8];
    {
      const float4 u = *(const float4*)(part + x), w = *(const float4*)(part + x + 4);
      a[0] = u.x; a[1] = u.y; a[2] = u.z; a[3] = u.w; a[4] = w.x; a[5] = w.y; a[6] = w.z; a[7] = w.w;
    }
    for (int k = 1; k < np; ++k) {
      const float4 u = *(const float4*)(part + (size_t)k * pstride + x), w = *(const float4*)(part + (size_t)k * pstride + x + 4);
      a[0] += u.x; a[1] += u.y; a[2] += u.z; a[3] += u.w; a[4] += w.x; a[5] += w.y; a[6] += w.z; a[7] += w.w;
    }
    if (zero_after) {
      *(float4*)(part + x) = make_float4(0.f, 0.f, 0.f, 0.f);
      *(float4*)(part + x + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    bool nan = false;
    uint32_t wv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      nan |= isnan(a[2 * e]) || isnan(a[2 * e + 1]);
      wv[e] = F16 ? ptx::pack_f16(a[2 * e] * scale, a[2 * e + 1] * scale)
                  : ptx::pack_bf16(a[2 * e] * scale, a[2 * e + 1] * scale);
    }
    flag_if(flag, nan);
    size_t off;
    if constexpr (!SW) {  // canonical: the window of outer batch ob is one contiguous block of rows
      const size_t blk = (size_t)nw * rowlen;
      const size_t ob = blk >= n ? 0 : (size_t)((uint32_t)x / (uint32_t)blk);  // window < 2^32 elements
      off = x + (ob * (size_t)(N - nw) + n0w) * rowlen;
    } else {  // raw [L, B, H, D] (Bo == 1): row b = n0w + x / rowlen, scattered by i
      const uint32_t wrow = (uint32_t)x / (uint32_t)rowlen, rem = (uint32_t)x - wrow * (uint32_t)rowlen;
      const uint32_t i = rem / (uint32_t)HD, e = rem - i * (uint32_t)HD;
      off = ((size_t)i * B + n0w + wrow) * HD + e;
    }
    if (((uintptr_t)(out + off) & 15) == 0) {
      *(uint4*)(out + off) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    } else {
      const uint16_t* hv = (const uint16_t*)wv;
      for (int q = 0; q < 8; ++q) ((uint16_t*)out)[off + q] = hv[q];
    }
  }
}

}  // namespace bk
}  // namespace tc
}  // namespace evo

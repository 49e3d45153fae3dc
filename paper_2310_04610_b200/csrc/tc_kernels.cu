// tc_kernels.cu — host side of the tcgen05 kernels: TMA tensor maps, shared-memory
// budgets, persistent grid sizing (one CTA per SM) and launches.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "tc_bwd.cuh"
#include "tc_fwd.cuh"
#include "tc_kernels.cuh"

// The file is compiled as three translation units in parallel (build.py): EVO_TU 1 = forward launch +
// device queries, 2 = backward D = 32 (+ the backward entry points), 3 = backward D = 16. EVO_TU 0
// (default) compiles everything into one unit.
#ifndef EVO_TU
#define EVO_TU 0
#endif
#define EVO_TU_FWD (EVO_TU == 0 || EVO_TU == 1)
#define EVO_TU_BWD32 (EVO_TU == 0 || EVO_TU == 2)
#define EVO_TU_BWD16 (EVO_TU == 0 || EVO_TU == 3)

namespace evo {
namespace tc {

#if EVO_TU_FWD
unsigned long long* g_trace = nullptr;
unsigned long long* g_trace_bwd = nullptr;
#else
extern unsigned long long* g_trace;
extern unsigned long long* g_trace_bwd;
#endif

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

CUtensorMapSwizzle swz(int row_bytes) {
  return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                           : CU_TENSOR_MAP_SWIZZLE_32B;
}

// (B, L, H, D) row-major as a 4-D map (D, H, L, B); box (D, 1, rows, 1).
// box_d: the kernel's head dim (D = 8 problems run the D = 16 kernels: the 16-wide box reads 8 real
// columns and TMA zero-fills the rest; stores / reduces of the padded columns are clipped)
bool map_bl_hd(CUtensorMap* m, const void* base, const Shape& s, int rows, CUtensorMapDataType dt,
               int esize, std::string* err, bool canonical = false, int box_d = 0) {
  if (box_d == 0) box_d = s.D;
  const bool swapped = s.swapped && !canonical;
  cuuint64_t dims[4] = {(cuuint64_t)s.D, (cuuint64_t)s.H, (cuuint64_t)s.L, (cuuint64_t)s.B};
  // swapped (raw msa_col / tri_end layout, (L, B, H, D)): the L and B strides trade places
  const cuuint64_t hd = (cuuint64_t)s.H * s.D * esize;
  cuuint64_t strides[3] = {(cuuint64_t)s.D * esize, swapped ? hd * (cuuint64_t)s.B : hd,
                           swapped ? hd : hd * (cuuint64_t)s.L};
  cuuint32_t box[4] = {(cuuint32_t)box_d, 1, (cuuint32_t)rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(m, dt, 4, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz(box_d * esize), CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (B,L,H,D) failed: " + std::to_string((int)r);
    return false;
  }
  return true;
}

// bias2 [Bo*H, L, L] as 3-D (Lj, Li, plane); box (64, 128, 1), 128B swizzle.
bool map_bias(CUtensorMap* m, const void* base, const Shape& s, int Bo, CUtensorMapDataType dt,
              std::string* err) {
  cuuint64_t dims[3] = {(cuuint64_t)s.L, (cuuint64_t)s.L, (cuuint64_t)Bo * s.H};
  cuuint64_t strides[2] = {(cuuint64_t)s.L * 2, (cuuint64_t)s.L * s.L * 2};
  cuuint32_t box[3] = {kBN, kBM, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(m, dt, 3, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (bias2) failed: " + std::to_string((int)r);
    return false;
  }
  return true;
}

template <int D>
size_t fwd_smem_bytes(int nbias_slots, int nKT, bool b1_rows) {
  using C = FwdCfg<D>;
  const size_t LP = (size_t)nKT * kBN;
  size_t b = 1024;  // alignment slack
  b += (size_t)C::NWG * 2 * C::kTileQ + 2 * (size_t)C::kStages * C::kTileKV;
  b += (size_t)nbias_slots * C::kBiasTile;
  b += (size_t)kAugA + (size_t)C::kStages * kAugB;  // bias1 augmentation tiles
  if (b1_rows) b += (size_t)C::NWG * 2 * LP * 2;  // bias1 rows (raw), double buffered per WG
  b += (size_t)(11 * C::NWG + 4 * C::kStages + 2 * nbias_slots) * 8 + 16 + 8 * C::NWG;
  return b;
}

constexpr size_t kMaxSmem = 227 * 1024;

// 16-bit two-term split of c (c ~= hi + lo) packed as (lo << 16) | hi, for the bias1 augmentation
// step: an exact-to-~2^-16 multiplier carried by a bf16/f16 UMMA operand.
uint32_t aug_split(double c, bool f16) {
  uint16_t hi, lo;
  if (f16) {
    const __half h = __double2half(c);
    const __half l = __double2half(c - (double)__half2float(h));
    hi = *(const uint16_t*)&h;
    lo = *(const uint16_t*)&l;
  } else {
    const __nv_bfloat16 h = __double2bfloat16(c);
    const __nv_bfloat16 l = __double2bfloat16(c - (double)__bfloat162float(h));
    hi = *(const uint16_t*)&h;
    lo = *(const uint16_t*)&l;
  }
  return (uint32_t)hi | ((uint32_t)lo << 16);
}

#if EVO_TU_FWD
template <int D, bool F16>
evo_status launch_fwd(const evo_attn_desc* d, const Shape& s, const void* q, const void* k, const void* v,
                      void* o, float* lse, cudaStream_t st, int* launches, std::string* err) {
  const CUtensorMapDataType dt = F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUtensorMap tq, tk, tv, tb;
  memset(&tb, 0, sizeof(tb));
  if (!map_bl_hd(&tq, q, s, kBM, dt, 2, err, false, D) || !map_bl_hd(&tk, k, s, kBN, dt, 2, err, false, D) ||
      !map_bl_hd(&tv, v, s, kBN, dt, 2, err, false, D))
    return EVO_ERR_CUDA;
  FwdParams p{};
  int bias_mode = kBiasNone;
  p.B = s.B; p.N = s.N; p.L = s.L; p.H = s.H; p.Bo = (int)d->Bo;
  p.swapped = s.swapped;
  p.nQT = (s.L + kBM - 1) / kBM;
  p.nKT = (s.L + kBN - 1) / kBN;
  p.total = (long long)p.Bo * p.H * p.nQT * p.N;
  p.scale_log2 = s.scale_log2;
  p.bias1 = s.bias1;
  p.bias2 = s.bias2;
  p.o = o;
  p.dreal = s.D;
  p.lse = lse;
  if (s.gate) {  // the gate pointer shares its slot with the bring-up trace buffer
    if (EVO_TRACE) {
      *err = "the output gate is not available in EVO_TRACE bring-up builds";
      return EVO_ERR_UNSUPPORTED;
    }
    p.gate = s.gate;
  } else {
    p.trace = g_trace;
  }
  p.nbias_slots = 0;
  p.b1_tma = (s.L % 8 == 0) ? 1 : 0;
  p.aug = (s.bias1 != nullptr || s.L % kBN != 0) ? 1 : 0;
  p.aug_c = aug_split(1.0 / (double)s.scale, F16);
  p.flag = s.flag;
  // bias1 rows staged per Q slot when they are bulk-copyable and fit; otherwise the UMMA warp reads
  // them from global (long L)
  p.b1_rows = (s.bias1 && p.b1_tma && fwd_smem_bytes<D>(3, p.nKT, true) <= kMaxSmem) ? 1 : 0;
  if (s.bias2) {
    if (s.L % 8 != 0) {
      bias_mode = kBiasGlobal;
    } else {
      if (!map_bias(&tb, s.bias2, s, p.Bo, dt, err)) return EVO_ERR_CUDA;
      if (fwd_smem_bytes<D>(p.nKT, p.nKT, p.b1_rows) <= kMaxSmem) {
        bias_mode = kBiasResident;
        p.nbias_slots = p.nKT;
      } else {
        bias_mode = kBiasStreamed;
        p.nbias_slots = 3;
      }
    }
  }
  const size_t smem = fwd_smem_bytes<D>(p.nbias_slots, p.nKT, p.b1_rows);
  if (smem > kMaxSmem) {
    *err = "forward shared-memory budget exceeded (L too large)";
    return EVO_ERR_UNSUPPORTED;
  }
  auto pick = [&](auto safe) {
    constexpr bool S = decltype(safe)::value;
    return bias_mode == kBiasResident   ? fwd_kernel<D, F16, kBiasResident, S>
           : bias_mode == kBiasStreamed ? fwd_kernel<D, F16, kBiasStreamed, S>
           : bias_mode == kBiasGlobal   ? fwd_kernel<D, F16, kBiasGlobal, S>
                                          : fwd_kernel<D, F16, kBiasNone, S>;
  };
  auto kern = (p.flag || s.gate || s.D != D) ? pick(std::true_type{}) : pick(std::false_type{});
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // Grid: one CTA per SM. If every (ob, h, q-tile) unit can get >= 4 CTAs, give each unit the same
  // number of CTAs with aligned row ranges (the q-tiles of a row then run concurrently and share
  // K/V through L2); otherwise split the flat item list evenly over the SMs.
  const int G = sm_count();
  const long long units = (long long)p.Bo * p.H * p.nQT;
  long long grid = std::min<long long>(p.total, G);
  p.aligned = 0;
  p.split = 1;
  if (units * 4 <= G) {
    p.split = (int)std::min<long long>(G / units, p.N);
    p.aligned = 1;
    grid = units * p.split;
  }
  kern<<<(unsigned)grid, FwdCfg<D>::kThreads, smem, st>>>(tq, tk, tv, tb, p);
  ++*launches;
  return EVO_OK;
}

#endif  // EVO_TU_FWD

// ---------------------------------------------------------------------------------- backward
constexpr int kBwdChunk = 3;  // query tiles per backward unit: its dBias2 strip (3 x 64 TMEM columns) fits
int bwd_nqt(const evo_attn_desc* d) { return (int)((d->L + bk::kBM - 1) / bk::kBM); }
int bwd_nkt(const evo_attn_desc* d) { return (int)((d->L + bk::kBN - 1) / bk::kBN); }
// dBias1 needs 16 TMEM columns: its chunks hold 2 query tiles (strip 128 columns) instead of 3
// without a pair bias there is no dBias2 strip in TMEM and no bias strip in shared memory: the whole
// query axis is one chunk at any L (MSA column attention: bias-free plus mask, L = N_seq)
int bwd_chunk(const evo_attn_desc* d, bool db1) {
  return d->has_bias2 ? std::min(bwd_nqt(d), db1 ? 2 : kBwdChunk) : bwd_nqt(d);
}
int bwd_nic(const evo_attn_desc* d, bool db1 = false) {
  const int c = bwd_chunk(d, db1);
  return (bwd_nqt(d) + c - 1) / c;
}
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Scratch of the tcgen05 backward.
//  default:       fp32 accumulators dQ (and dK, dV when the query axis is chunked) [B, L, H, D]
//                 (zeroed by the preamble, TMA reduce-add targets), padded lse*log2e and delta.
//  deterministic: per-slot partials of one row window — dQ [nKT][Bw, L, H, D], chunked dK / dV
//                 [nIC][Bw, L, H, D], dBias1 [H * nIC][Bw][L] — plus the dBias2 flush tickets of
//                 every window; windows of nw rows per outer batch keep the partials under kDetCap.
constexpr size_t kDetCap = (size_t)2 << 30;
// default mode: the fp32 accumulators (dQ; dK, dV when chunked) cover all rows when they fit kAccCap,
// else one row window at a time (C5: 3 x 1 MB per row -> windows of ~340 rows, 1 GB instead of 6.4 GB)
constexpr size_t kAccCap = (size_t)1 << 30;
struct BwdScratch {
  size_t dq, dk, dv, lse2, delta, db1p, tickets, total;
  int nw, nwin;  // deterministic row window (rows per outer batch), number of windows
};
BwdScratch bwd_scratch_layout(const evo_attn_desc* d) {
  BwdScratch w{};
  const size_t B = (size_t)d->Bo * d->N;
  const size_t Lp = (size_t)bwd_nqt(d) * bk::kBM;
  const size_t row = (size_t)d->L * d->H * d->D * 4;  // one row's fp32 [L, H, D]
  const bool db1 = d->has_bias1 && d->need_dbias1;
  const int nic = bwd_nic(d, db1), nkt = bwd_nkt(d);
  const bool chunked = nic > 1;
  w.nw = (int)d->N;
  w.nwin = 1;
  size_t dq_bytes, kv_bytes, db1p = 0, tickets = 0;
  if (d->deterministic) {
    const size_t per = row * ((size_t)nkt + (chunked ? 2 * (size_t)nic : 0)) + (db1 ? (size_t)d->H * nic * d->L * 4 : 0);
    w.nw = (int)std::max<int64_t>(1, std::min<int64_t>(d->N, (int64_t)(kDetCap / (per * d->Bo))));
    if (const char* e = getenv("EVO_DET_WINDOW_ROWS"))  // test hook: force smaller row windows
      if (atoi(e) > 0) w.nw = std::min(w.nw, atoi(e));
    w.nwin = (int)((d->N + w.nw - 1) / w.nw);
    const size_t Bw = (size_t)d->Bo * w.nw;
    dq_bytes = align256((size_t)nkt * Bw * row);
    kv_bytes = chunked ? align256((size_t)nic * Bw * row) : 0;
    db1p = db1 ? align256((size_t)d->H * nic * Bw * d->L * 4) : 0;
    tickets = align256((size_t)w.nwin * d->Bo * d->H * nkt * nic * 4);
  } else {
    const size_t per = row * (chunked ? 3 : 1);
    size_t cap = kAccCap;
    if (const char* e = getenv("EVO_BWD_ACC_CAP_MB")) cap = (size_t)atoll(e) << 20;  // experiments
    w.nw = (int)std::max<int64_t>(1, std::min<int64_t>(d->N, (int64_t)(cap / (per * d->Bo))));
    if (const char* e = getenv("EVO_BWD_WINDOW_ROWS"))  // test hook: force the row window (0: all rows)
      w.nw = atoi(e) > 0 ? std::min(w.nw, atoi(e)) : (int)d->N;
    w.nwin = (int)((d->N + w.nw - 1) / w.nw);
    dq_bytes = align256((size_t)d->Bo * w.nw * row);
    kv_bytes = chunked ? dq_bytes : 0;  // dK/dV accumulators when the query axis is chunked
  }
  w.dq = 0;
  w.dk = dq_bytes;
  w.dv = w.dk + kv_bytes;
  w.lse2 = w.dv + kv_bytes;
  w.delta = w.lse2 + align256(B * d->H * Lp * 4);
  w.db1p = w.delta + align256(B * d->H * Lp * 4);
  w.tickets = w.db1p + db1p;
  w.total = w.tickets + tickets;
  return w;
}

// fp32 [rows, L, H, D] (canonical) as a 4-D map (D, H, L, rows), box (D, 1, box_rows, 1), row-size swizzle
bool map_f32_rows(CUtensorMap* m, void* base, const Shape& s, long long rows, int box_rows, std::string* err,
                  int box_d) {
  cuuint64_t dims[4] = {(cuuint64_t)s.D, (cuuint64_t)s.H, (cuuint64_t)s.L, (cuuint64_t)rows};
  const cuuint64_t hd = (cuuint64_t)s.H * s.D * 4;
  cuuint64_t strides[3] = {(cuuint64_t)s.D * 4, hd, hd * (cuuint64_t)s.L};
  cuuint32_t box[4] = {(cuuint32_t)box_d, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz(box_d * 4), CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (fp32 partials) failed: " + std::to_string((int)r);
    return false;
  }
  return true;
}

template <int D, bool CH>
size_t bwd_smem_bytes(int nQT) {
  using C = bk::Cfg<D, CH>;
  size_t b = 1024;
  b += (size_t)C::kQStages * 2 * C::kTileQ + (size_t)C::kKStages * 2 * C::kTileK + 4 * (size_t)C::kPdsTile;
  b += (size_t)nQT * C::kBiasTile + (size_t)C::kDqBufs * bk::kBM * D * 4;
  b += (size_t)bk::kAugA + (size_t)C::kKStages * bk::kAugB + bk::kOnes + bk::kIdent;
  b += (size_t)C::kQStages * bk::kBM * 4 * 2 + (size_t)C::kKStages * 64 * 2;
  b += (size_t)(2 * C::kQStages + 2 * C::kKStages + 8 + 7) * 8 + 16;
  return b;
}

template <int D, bool F16>
evo_status launch_bwd(const evo_attn_desc* d, const Shape& s, const void* dout, const void* q, const void* k,
                      const void* v, const void* o, const float* lse, const float* delta, void* dq, void* dk, void* dv,
                      float* dbias1, float* dbias2, void* scratch, cudaStream_t st, int* launches,
                      std::string* err) {
  const CUtensorMapDataType dt = F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const BwdScratch w = bwd_scratch_layout(d);
  const bool det = d->deterministic != 0;
  const bool win = !det && w.nwin > 1;  // windowed accumulators
  char* ws = (char*)scratch;
  float* dqacc = (float*)(ws + w.dq);
  float* lse2 = (float*)(ws + w.lse2);
  float* delta_p = (float*)(ws + w.delta);
  CUtensorMap tq, tk, tv, tdo, tb, tdq, tdk, tdv;
  memset(&tb, 0, sizeof(tb));
  const bool want_db1 = dbias1 != nullptr;
  const bool dkv_reduce = bwd_nic(d, want_db1) > 1;
  float* dkacc = (float*)(ws + w.dk);
  float* dvacc = (float*)(ws + w.dv);
  const int nkt = bwd_nkt(d), nic = bwd_nic(d, want_db1);
  const long long Bw = (long long)d->Bo * w.nw;  // rows of a (full) deterministic window
  if (dkv_reduce) {
    const long long kvrows = det ? nic * Bw : Bw;
    const bool ok = (det || win) ? map_f32_rows(&tdk, dkacc, s, kvrows, bk::kBN, err, D) &&
                                       map_f32_rows(&tdv, dvacc, s, kvrows, bk::kBN, err, D)
                                 : map_bl_hd(&tdk, dkacc, s, bk::kBN, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, err, true, D) &&
                                       map_bl_hd(&tdv, dvacc, s, bk::kBN, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, err, true, D);
    if (!ok) return EVO_ERR_CUDA;
  } else {
    tdk = tdv = tb;
  }
  // with a fused output gate the main kernel reads the gated dO the preamble writes (s.dog)
  const void* dout_k = s.gate ? s.dog : dout;
  if (!map_bl_hd(&tq, q, s, bk::kBM, dt, 2, err, false, D) || !map_bl_hd(&tk, k, s, bk::kBN, dt, 2, err, false, D) ||
      !map_bl_hd(&tv, v, s, bk::kBN, dt, 2, err, false, D) || !map_bl_hd(&tdo, dout_k, s, bk::kBM, dt, 2, err, false, D) ||
      !((det || win) ? map_f32_rows(&tdq, dqacc, s, det ? nkt * Bw : Bw, bk::kBM, err, D)
            : map_bl_hd(&tdq, dqacc, s, bk::kBM, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, err, true, D)))
    return EVO_ERR_CUDA;
  if (s.bias2 && !map_bias(&tb, s.bias2, s, (int)d->Bo, dt, err)) return EVO_ERR_CUDA;
  bk::ParamsSafe p{};  // the plain variants get its base (bk::Params) slice
  p.B = s.B; p.N = s.N; p.L = s.L; p.H = s.H; p.Bo = (int)d->Bo;
  p.swapped = s.swapped;
  p.nQT = (s.L + bk::kBM - 1) / bk::kBM;
  p.nKT = nkt;
  p.nQC = bwd_chunk(d, want_db1);
  p.nIC = nic;
  p.dbias1 = dbias1;
  p.dkv_reduce = dkv_reduce ? 1 : 0;
  p.scale = s.scale;
  p.scale_log2 = s.scale_log2;
  p.bias1 = s.bias1;
  p.lse2 = lse2;
  p.delta = delta_p;
  p.dk = dk;
  p.dv = dv;
  p.dbias2 = dbias2;
  if (d->dbias2_multicast && dbias2) {  // cross-GPU dBias2 reduction fused into the strip flush (NVLS)
    p.dbias2 = (float*)d->dbias2_multicast;
    p.dbias2_mc = 1;
  }
  p.has_bias2 = s.bias2 != nullptr;
  p.trace = g_trace_bwd;
  p.x.det = det ? 1 : 0;
  p.x.win = win ? 1 : 0;
  p.x.dreal = s.D;
  p.x.db1_part = (float*)(ws + w.db1p);
  p.x.flag = s.flag;
  // bias1 (and the key mask past L) enter S through one extra K=16 MMA step: A_aug rows hold a
  // 16-bit two-term split of 1/scale, B_aug rows the bias1 value of each key.
  p.aug = (s.bias1 != nullptr || s.L % bk::kBN != 0) ? 1 : 0;
  p.aug_c = aug_split(1.0 / (double)s.scale, F16);
  p.nBT = s.bias2 ? p.nQC : 0;  // resident pair-bias tiles
  const size_t smem = dkv_reduce ? bwd_smem_bytes<D, true>(p.nBT) : bwd_smem_bytes<D, false>(p.nBT);
  if (smem > kMaxSmem) {
    *err = "backward shared-memory budget exceeded";
    return EVO_ERR_UNSUPPORTED;
  }
  const int Lp = p.nQT * bk::kBM;
  const long long prow = (long long)s.B * s.H;
  // the preamble also zeroes the fp32 accumulators this call reduces into ([0, w.lse2): dQ, and dK / dV
  // when chunked) — or, deterministic, only the dBias2 flush tickets (partials are stored, not added)
  float4* zero4 = det ? (float4*)(ws + w.tickets) : (float4*)dqacc;
  const long long nzero4 = det ? (long long)((w.total - w.tickets) / 16)
                               : (long long)((dkv_reduce ? w.lse2 : w.dk) / 16);
  using T = typename std::conditional<F16, __half, __nv_bfloat16>::type;
  if (delta) {  // delta supplied by the caller: only pad
    bk::pad_rows_kernel<<<(unsigned)std::min<long long>((prow * Lp + 255) / 256, 148 * 16), 256, 0, st>>>(
        lse, delta, lse2, delta_p, s.L, Lp, prow, zero4, nzero4);
  } else {
    auto prep = s.D == 8 ? (s.swapped ? bk::prep_kernel<8, T, true> : bk::prep_kernel<8, T, false>)
                         : (s.swapped ? bk::prep_kernel<D, T, true> : bk::prep_kernel<D, T, false>);
    prep<<<(unsigned)std::min<long long>((prow * Lp + 255) / 256, 148 * 32), 256, 0, st>>>(
        (const T*)dout, (const T*)o, lse, lse2, delta_p, s.B, s.L, s.H, Lp, zero4, nzero4, s.flag,
        (const T*)s.gate, (T*)s.dog, (T*)s.dgate);
  }
  ++*launches;
  const bool safe = det || win || s.flag || s.D != D;
  auto kern_of = [&](auto sf) {
    constexpr bool S = decltype(sf)::value;
    return s.swapped ? (dkv_reduce ? bk::bwd_kernel<D, F16, true, true, S> : bk::bwd_kernel<D, F16, false, true, S>)
                     : (dkv_reduce ? bk::bwd_kernel<D, F16, true, false, S> : bk::bwd_kernel<D, F16, false, false, S>);
  };
  cudaFuncSetAttribute(safe ? (const void*)kern_of(std::true_type{}) : (const void*)kern_of(std::false_type{}),
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int G = sm_count();
  auto pdl_launch = [&](auto fn, dim3 grid, dim3 block, size_t shm, auto... args) {
    cudaLaunchConfig_t cfg = {};  // programmatic dependent launch: the prologue overlaps the predecessor's tail
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = getenv("EVO_NO_PDL") ? 0 : 1;
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = shm;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, fn, args...);
    ++*launches;
  };
  const long long units = (long long)p.Bo * p.H * p.nKT * p.nIC;
  const int HD = s.H * s.D;
  for (int wi = 0; wi < w.nwin; ++wi) {
    p.x.n0w = wi * w.nw;
    p.x.nw = std::min<int>(w.nw, s.N - p.x.n0w);
    p.total = units * p.x.nw;
    p.x.tickets = det ? (int*)(ws + w.tickets) + (size_t)wi * units : nullptr;
    long long grid = std::min<long long>(p.total, G);
    p.aligned = 0;
    p.split = 1;
    if (units <= G) {
      p.split = (int)std::min<long long>(G / units, p.x.nw);
      p.aligned = 1;
      grid = units * p.split;
    }
    if (safe)
      pdl_launch(kern_of(std::true_type{}), dim3((unsigned)grid), dim3(bk::kThreads), smem, tq, tk, tv, tdo, tb, tdq,
                 tdk, tdv, p);
    else
      pdl_launch(kern_of(std::false_type{}), dim3((unsigned)grid), dim3(bk::kThreads), smem, tq, tk, tv, tdo, tb, tdq,
                 tdk, tdv, static_cast<const bk::Params&>(p));
    if (det) {
      // ordered sums of this window's partial slots (dQ over key tiles; dK / dV over query chunks)
      const size_t n = (size_t)p.Bo * p.x.nw * s.L * HD, pstride = n;
      const unsigned cg = (unsigned)std::min<size_t>((n / 8 + 255) / 256, 148 * 16);
      auto conv = [&](float* part, int np, void* out, float scale) {
        pdl_launch(s.swapped ? bk::det_convert_kernel<T, true> : bk::det_convert_kernel<T, false>, dim3(cg), dim3(256),
                   0, (const float*)part, np, pstride, (T*)out, n, scale, s.B, s.L, HD, s.N, p.x.n0w, p.x.nw, s.flag, 0);
      };
      conv(dqacc, nkt, dq, s.scale);
      if (dkv_reduce) {
        conv(dkacc, nic, dk, s.scale);
        conv(dvacc, nic, dv, 1.f);
      }
    } else if (win) {
      // this window's accumulators into their rows (the streaming conversion, per outer batch: the rows
      // of one window and outer batch are contiguous), then zeroed for the next window
      const size_t rowlen = (size_t)s.L * HD, nob = (size_t)p.x.nw * rowlen;
      const unsigned cg = (unsigned)std::min<size_t>((nob / 8 + 255) / 256, 148 * 16);
      auto conv = [&](const float* acc, void* out, float scale) {
        for (int ob = 0; ob < p.Bo; ++ob) {
          const size_t shift = s.swapped ? (size_t)p.x.n0w * HD : ((size_t)ob * s.N + p.x.n0w) * rowlen;
          pdl_launch(s.swapped ? bk::dq_convert_kernel<T, true> : bk::dq_convert_kernel<T, false>, dim3(cg), dim3(256),
                     0, acc + ob * nob, (T*)out + shift, nob, scale, s.B, s.L, HD, s.flag);
        }
      };
      conv(dqacc, dq, s.scale);
      if (dkv_reduce) {
        conv(dkacc, dk, s.scale);
        conv(dvacc, dv, 1.f);
      }
      if (wi + 1 < w.nwin) cudaMemsetAsync(dqacc, 0, dkv_reduce ? w.lse2 : w.dk, st);
    }
    if (det) {
      if (dbias1) {  // dBias1 partials of (head, chunk) slots in order, per outer batch of the window
        const size_t nl = (size_t)p.x.nw * s.L;
        for (int ob = 0; ob < p.Bo; ++ob) {
          ordered_sum_kernel<float><<<(unsigned)std::min<size_t>((nl + 255) / 256, 148 * 4), 256, 0, st>>>(
              p.x.db1_part + (size_t)ob * nl, s.H * nic, (size_t)p.Bo * nl, dbias1 + ((size_t)ob * s.N + p.x.n0w) * s.L, nl);
          ++*launches;
        }
      }
    }
  }
  if (!det && !win) {
    const size_t n = (size_t)s.B * s.L * HD;
    const unsigned cg = (unsigned)std::min<size_t>((n / 8 + 255) / 256, 148 * 16);
    auto convert = [&](const float* acc, void* out, float scale) {  // programmatic dependents of the main kernel
      pdl_launch(s.swapped ? bk::dq_convert_kernel<T, true> : bk::dq_convert_kernel<T, false>, dim3(cg), dim3(256), 0,
                 acc, (T*)out, n, scale, s.B, s.L, HD, s.flag);
    };
    convert(dqacc, dq, s.scale);
    if (dkv_reduce) {  // dK = scale * dK_acc, dV = dV_acc
      convert(dkacc, dk, s.scale);
      convert(dvacc, dv, 1.f);
    }
  }
  return EVO_OK;
}

}  // namespace

#define EVO_BWD_ARGS                                                                                               \
  const evo_attn_desc *d, const Shape &s, const void *dout, const void *q, const void *k, const void *v,           \
      const void *o, const float *lse, const float *delta, void *dq, void *dk, void *dv, float *dbias1,             \
      float *dbias2, void *scratch, cudaStream_t st, int *launches, std::string *err
#define EVO_BWD_PASS d, s, dout, q, k, v, o, lse, delta, dq, dk, dv, dbias1, dbias2, scratch, st, launches, err
evo_status launch_bwd16(EVO_BWD_ARGS);
#if EVO_TU_BWD16
evo_status launch_bwd16(EVO_BWD_ARGS) {
  return d->dtype == EVO_F16 ? launch_bwd<16, true>(EVO_BWD_PASS) : launch_bwd<16, false>(EVO_BWD_PASS);
}
#endif

#if EVO_TU_FWD
bool device_supported() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    ok = (major == 10 && minor == 0 && encode_fn() != nullptr) ? 1 : 0;
  }
  return ok == 1;
}

size_t fwd_scratch_bytes(const evo_attn_desc*) { return 0; }
#endif

#if EVO_TU_BWD32
size_t bwd_scratch_bytes(const evo_attn_desc* d) { return bwd_scratch_layout(d).total; }

// tcgen05 backward: 16-bit inputs, D in {16, 32}, L % 8 == 0 (16B-aligned rows for the bulk copies).
// L > 384 splits the query axis into chunks of 3 tiles (a chunk's dBias2 strip fits in TMEM next to
// S/dP, dQ, dK|dV) and reduces dK/dV over the chunks in fp32.
bool bwd_available(const evo_attn_desc* d) {
  return d->dtype != EVO_F32 && (d->D == 8 || d->D == 16 || d->D == 32) && d->L % 8 == 0 && device_supported();
}

evo_status bwd(EVO_BWD_ARGS) {
  switch (d->D) {
    case 8:  // zero-padded to the D = 16 kernels (TMA fills the padded columns with zeros)
    case 16: return launch_bwd16(EVO_BWD_PASS);
    case 32: return d->dtype == EVO_F16 ? launch_bwd<32, true>(EVO_BWD_PASS) : launch_bwd<32, false>(EVO_BWD_PASS);
    default: *err = "tcgen05 backward supports D in {16, 32}"; return EVO_ERR_UNSUPPORTED;
  }
}
#endif  // EVO_TU_BWD32

#if EVO_TU_FWD
evo_status fwd(const evo_attn_desc* d, const Shape& s, const void* q, const void* k, const void* v, void* o,
               float* lse, void*, cudaStream_t st, int* launches, std::string* err) {
  const bool f16 = d->dtype == EVO_F16;
  switch (d->D) {
    case 8:  // zero-padded to the D = 16 kernel (TMA fills the padded columns with zeros)
    case 16: return f16 ? launch_fwd<16, true>(d, s, q, k, v, o, lse, st, launches, err)
                        : launch_fwd<16, false>(d, s, q, k, v, o, lse, st, launches, err);
    case 32: return f16 ? launch_fwd<32, true>(d, s, q, k, v, o, lse, st, launches, err)
                        : launch_fwd<32, false>(d, s, q, k, v, o, lse, st, launches, err);
    case 64: return f16 ? launch_fwd<64, true>(d, s, q, k, v, o, lse, st, launches, err)
                        : launch_fwd<64, false>(d, s, q, k, v, o, lse, st, launches, err);
    default: *err = "tcgen05 forward supports D in {16, 32, 64}"; return EVO_ERR_UNSUPPORTED;
  }
}

#endif  // EVO_TU_FWD

}  // namespace tc
}  // namespace evo

// Bring-up aid (not part of include/evoattn.h): record a clock64 timeline of CTA 0 of the next
// forward launches into a device buffer of 8 x 64 uint64 (null disables).
#if EVO_TU_FWD
extern "C" void evo_attn_debug_set_trace(void* dev_buf) { evo::tc::g_trace = (unsigned long long*)dev_buf; }
extern "C" void evo_attn_debug_set_trace_bwd(void* dev_buf) { evo::tc::g_trace_bwd = (unsigned long long*)dev_buf; }
#endif

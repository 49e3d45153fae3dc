// evoattn_capi.cu — the C-ABI (include/evoattn.h): validation with the
// reference's error taxonomy, workspace carving, and kernel dispatch.
//
// Validation mirrors AttentionProblem::validate (attention.cpp:49-86) and
// attn_backward_tiled's stats checks (attention_tiled.cpp:196-209), mapped to
// evo_status codes instead of exceptions (errors.hpp:15-30).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "simt_kernels.cuh"
#include "tc_kernels.cuh"

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

evo_status fail(evo_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

evo_status validate(const evo_attn_desc* d) {
  if (!d) return fail(EVO_ERR_USAGE, "null descriptor");
  if (d->Bo < 1 || d->N < 1 || d->L < 1 || d->H < 1 || d->D < 1)
    return fail(EVO_ERR_VALIDATION, "extents must be >= 1 (Bo, N, L, H, D)");
  if (d->dtype != EVO_F32 && d->dtype != EVO_BF16 && d->dtype != EVO_F16)
    return fail(EVO_ERR_VALIDATION, "unknown dtype");
  if (d->dbias_dtype != EVO_F32 && d->dbias_dtype != d->dtype)
    return fail(EVO_ERR_VALIDATION, "dbias_dtype must be EVO_F32 or equal to dtype");
  if (!std::isfinite(d->scale)) return fail(EVO_ERR_NUMERIC, "attention scale must be finite");
  if (d->has_gate != 0 && d->has_gate != 1) return fail(EVO_ERR_VALIDATION, "has_gate must be 0 or 1");
  if (d->axes_swapped != 0 && d->axes_swapped != 1)
    return fail(EVO_ERR_VALIDATION, "axes_swapped must be 0 or 1");
  if (d->axes_swapped && d->Bo != 1)
    return fail(EVO_ERR_VALIDATION, "axes_swapped (raw [L, N, H, D] layout) requires Bo == 1");
  if (d->Bo * d->N > 0x7fffffffLL || d->L > 65535 * 64LL || d->H > 65535)
    return fail(EVO_ERR_UNSUPPORTED, "extents exceed the kernels' index range");
  return EVO_OK;
}

// The tcgen05 kernels carry 1/scale in 16-bit UMMA operands (the bias augmentation steps): it must be
// a finite normal number of the problem's 16-bit format; other scales take the SIMT kernels.
bool scale_fits_16bit(const evo_attn_desc* d) {
  const double c = std::fabs(1.0 / d->scale);
  return d->dtype == EVO_F16 ? (c >= 6.103515625e-05 && c <= 65504.0) : (c >= 1.1754943508222875e-38 && c <= 3.3e38);
}

bool tc_eligible(const evo_attn_desc* d) {
  return d->dtype != EVO_F32 && (d->D == 8 || d->D == 16 || d->D == 32 || d->D == 64) && scale_fits_16bit(d) &&
         evo::tc::device_supported();
}

int resolve(const evo_attn_desc* d) {
  if (d->path == EVO_PATH_SIMT) return EVO_PATH_SIMT;
  if (d->path == EVO_PATH_TCGEN05) return tc_eligible(d) ? EVO_PATH_TCGEN05 : -1;
  return tc_eligible(d) ? EVO_PATH_TCGEN05 : EVO_PATH_SIMT;
}

evo::Shape make_shape(const evo_attn_desc* d, const void* b1, const void* b2, int* flag = nullptr) {
  evo::Shape s;
  s.B = (int)(d->Bo * d->N);
  s.N = (int)d->N;
  s.L = (int)d->L;
  s.H = (int)d->H;
  s.D = (int)d->D;
  s.scale = (float)d->scale;
  s.scale_log2 = (float)(d->scale * 1.4426950408889634);
  s.bias1 = b1;
  s.bias2 = b2;
  s.swapped = d->axes_swapped;
  s.flag = d->check_numerics ? flag : nullptr;
  s.gate = nullptr;
  s.dgate = nullptr;
  s.dog = nullptr;
  return s;
}

// Every workspace starts with a 256-byte header: word 0 is the numeric-check flag.
constexpr size_t kHeader = 256;

// SIMT backward: dBias2 / dBias1 partial planes of one row batch (ordered, atomic-free reduction);
// batches stay inside one outer batch and are sized so the dBias2 planes fit kSimtPartCap.
constexpr size_t kSimtPartCap = (size_t)512 << 20;
int64_t simt_batch_rows(const evo_attn_desc* d) {
  if (!d->has_bias2) return d->N;
  const size_t plane = (size_t)d->H * d->L * d->L * 4;
  return std::max<int64_t>(1, std::min<int64_t>(d->N, (int64_t)(kSimtPartCap / plane)));
}

// Bwd workspace layout: [header][delta B*H*L f32][dbias2 acc Bo*H*L*L f32][dbias1 acc B*L f32]
// [gated dO, has_gate][SIMT partial planes of one row batch][tc scratch]
struct BwdWs {
  size_t delta, db2, db1, dog, db2p, db1p, tc, total;
};
size_t elem_bytes(const evo_attn_desc* d) { return d->dtype == EVO_F32 ? 4 : 2; }

// Workspace sizing follows the kernels the call will run on the target device (sm_100a); on a host
// without one (sizing only) the tcgen05 envelope is assumed.
bool simt_bwd_path(const evo_attn_desc* d) {
  if (d->path == EVO_PATH_SIMT) return true;
  const bool tc = d->dtype != EVO_F32 && (d->D == 8 || d->D == 16 || d->D == 32) && d->L % 8 == 0 && scale_fits_16bit(d);
  return !tc;
}

BwdWs bwd_layout(const evo_attn_desc* d) {
  BwdWs w{};
  const size_t B = (size_t)(d->Bo * d->N);
  size_t off = kHeader;
  w.delta = off;
  off += align_up(B * d->H * d->L * 4);
  w.db2 = off;
  if (d->has_bias2) off += align_up((size_t)d->Bo * d->H * d->L * d->L * 4);
  w.db1 = off;
  if (d->has_bias1 && d->need_dbias1) off += align_up(B * d->L * 4);
  w.dog = off;
  if (d->has_gate) off += align_up(B * d->L * d->H * d->D * elem_bytes(d));
  w.db2p = w.db1p = w.tc = off;
  if (simt_bwd_path(d)) {
    const size_t nb = (size_t)simt_batch_rows(d);
    if (d->has_bias2) off += align_up(nb * d->H * d->L * d->L * 4);
    w.db1p = off;
    if (d->has_bias1 && d->need_dbias1) off += align_up((size_t)d->H * nb * d->L * 4);
    w.tc = off;
  } else {
    off += align_up(evo::tc::bwd_scratch_bytes(d));
  }
  w.total = off;
  return w;
}

template <typename T, int DP>
void simt_fwd(const evo::Shape& s, const void* q, const void* k, const void* v, void* o,
              float* lse, cudaStream_t st) {
  dim3 grid((s.L + evo::simt::Tiles<DP>::kRows - 1) / evo::simt::Tiles<DP>::kRows, s.H, s.B);
  evo::simt::fwd_kernel<T, DP><<<grid, evo::simt::Tiles<DP>::kRows, 0, st>>>(
      s, (const T*)q, (const T*)k, (const T*)v, (T*)o, lse);
  ++g_launches;
}

template <typename T>
evo_status simt_fwd_dispatch(const evo::Shape& s, const void* q, const void* k, const void* v,
                             void* o, float* lse, cudaStream_t st) {
  if (s.D <= 8) simt_fwd<T, 8>(s, q, k, v, o, lse, st);
  else if (s.D <= 16) simt_fwd<T, 16>(s, q, k, v, o, lse, st);
  else if (s.D <= 32) simt_fwd<T, 32>(s, q, k, v, o, lse, st);
  else if (s.D <= 64) simt_fwd<T, 64>(s, q, k, v, o, lse, st);
  else return fail(EVO_ERR_UNSUPPORTED, "SIMT kernels support D <= 64");
  return EVO_OK;
}

void launch_ordered_sum(const float* part, int np, size_t stride, float* acc, size_t n, cudaStream_t st) {
  const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  evo::ordered_sum_kernel<float><<<blocks, 256, 0, st>>>(part, np, stride, acc, n);
  ++g_launches;
}

// SIMT backward over row batches inside each outer batch: dK/dV (+ the batch's dBias partial planes),
// dQ, then the planes added in ascending order into the fp32 accumulators (no atomics: the result
// is bit-reproducible, the reference's deterministic policy).
template <typename T, int DP>
void simt_bwd(const evo_attn_desc* d, const evo::Shape& s, const void* dout, const void* q, const void* k,
              const void* v, const float* lse, const float* delta, void* dq, void* dk, void* dv, float* db1,
              float* db2, float* db1p, float* db2p, cudaStream_t st) {
  const int64_t nb = simt_batch_rows(d);
  const size_t plane = (size_t)s.H * s.L * s.L;
  for (int ob = 0; ob < (int)d->Bo; ++ob)
    for (int64_t n0 = 0; n0 < d->N; n0 += nb) {
      const int rows = (int)std::min<int64_t>(nb, d->N - n0);
      const int b0 = (int)(ob * d->N + n0);
      dim3 grid((s.L + evo::simt::Tiles<DP>::kRows - 1) / evo::simt::Tiles<DP>::kRows, s.H, rows);
      evo::simt::dkdv_kernel<T, DP><<<grid, evo::simt::Tiles<DP>::kRows, 0, st>>>(
          s, (const T*)q, (const T*)k, (const T*)v, (const T*)dout, lse, delta, (T*)dk, (T*)dv, b0,
          db1 ? db1p : nullptr, db2 ? db2p : nullptr);
      evo::simt::dq_kernel<T, DP><<<grid, evo::simt::Tiles<DP>::kRows, 0, st>>>(
          s, (const T*)q, (const T*)k, (const T*)v, (const T*)dout, lse, delta, (T*)dq, b0);
      g_launches += 2;
      if (db2) launch_ordered_sum(db2p, rows, plane, db2 + (size_t)ob * plane, plane, st);
      if (db1) launch_ordered_sum(db1p, s.H, (size_t)rows * s.L, db1 + (size_t)b0 * s.L, (size_t)rows * s.L, st);
    }
}

template <typename T>
evo_status simt_bwd_dispatch(const evo_attn_desc* d, const evo::Shape& s, const void* dout, const void* q,
                             const void* k, const void* v, const float* lse, const float* delta, void* dq,
                             void* dk, void* dv, float* db1, float* db2, float* db1p, float* db2p,
                             cudaStream_t st) {
  if (s.D <= 8) simt_bwd<T, 8>(d, s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, db1p, db2p, st);
  else if (s.D <= 16) simt_bwd<T, 16>(d, s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, db1p, db2p, st);
  else if (s.D <= 32) simt_bwd<T, 32>(d, s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, db1p, db2p, st);
  else if (s.D <= 64) simt_bwd<T, 64>(d, s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, db1p, db2p, st);
  else return fail(EVO_ERR_UNSUPPORTED, "SIMT kernels support D <= 64");
  return EVO_OK;
}

template <typename T>
void launch_delta(const evo::Shape& s, const void* dout, const void* o, float* delta,
                  cudaStream_t st) {
  const size_t rows = (size_t)s.B * s.L * s.H;
  const int blocks = (int)std::min<size_t>((rows + 255) / 256, 148 * 16);
  evo::simt::delta_kernel<T><<<blocks, 256, 0, st>>>(s, (const T*)dout, (const T*)o, delta);
  ++g_launches;
}

template <typename T>
void launch_convert(const float* src, void* dst, size_t n, cudaStream_t st) {
  const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  evo::convert_kernel<T><<<blocks, 256, 0, st>>>(src, (T*)dst, n);
  ++g_launches;
}

evo_status check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(EVO_ERR_CUDA, std::string("CUDA: ") + cudaGetErrorString(e));
  return EVO_OK;
}

// check_numerics: the kernels OR the header flag; the call waits for its stream and maps a raised
// flag to NumericError (the reference throws from inside the operator: attention_tiled.cpp:49-65,
// 125-127, 209).
evo_status numeric_begin(const evo_attn_desc* d, int* flag, cudaStream_t st) {
  if (d->check_numerics && cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess)
    return fail(EVO_ERR_CUDA, "numeric-check flag reset failed");
  return EVO_OK;
}
evo_status numeric_end(const evo_attn_desc* d, const int* flag, cudaStream_t st, const char* what) {
  evo_status e = check_launch();
  if (e || !d->check_numerics) return e;
  int h = 0;
  if (cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return fail(EVO_ERR_CUDA, std::string("CUDA: ") + cudaGetErrorString(cudaGetLastError()));
  if (h) return fail(EVO_ERR_NUMERIC, what);
  return EVO_OK;
}

}  // namespace

namespace evo {
void set_last_error(const char* msg) { g_err = msg; }  // errors of the other translation units
}  // namespace evo

extern "C" {

const char* evo_attn_version(void) { return "evoattn 0.2 sm_100a"; }
const char* evo_attn_last_error(void) { return g_err.c_str(); }
int evo_attn_last_launch_count(void) { return g_launches; }

int evo_attn_resolved_path(const evo_attn_desc* d) {
  if (validate(d) != EVO_OK) return -1;
  return resolve(d);
}

int evo_attn_resolved_bwd_path(const evo_attn_desc* d) {
  if (validate(d) != EVO_OK) return -1;
  const int p = resolve(d);
  if (p < 0) return -1;
  if (p == EVO_PATH_TCGEN05 && !evo::tc::bwd_available(d)) return d->path == EVO_PATH_TCGEN05 ? -1 : EVO_PATH_SIMT;
  return p;
}

size_t evo_attn_fwd_workspace_size(const evo_attn_desc* d) {
  if (validate(d) != EVO_OK) return 0;
  return kHeader + evo::tc::fwd_scratch_bytes(d);
}

size_t evo_attn_bwd_workspace_size(const evo_attn_desc* d) {
  if (validate(d) != EVO_OK) return 0;
  return bwd_layout(d).total;
}

static evo_status fwd_impl(const evo_attn_desc* d, const void* q, const void* k, const void* v,
                           const void* bias1, const void* bias2, const void* gate, void* o, float* lse,
                           void* workspace, size_t workspace_bytes, evo_stream_t stream) {
  evo_status st = EVO_OK;
  if (!q || !k || !v || !o || !lse) return fail(EVO_ERR_VALIDATION, "q, k, v, o, lse must be non-null");
  if (d->has_bias1 != (bias1 != nullptr)) return fail(EVO_ERR_VALIDATION, "bias1 presence does not match the descriptor");
  if (d->has_bias2 != (bias2 != nullptr)) return fail(EVO_ERR_VALIDATION, "bias2 presence does not match the descriptor");
  if (!workspace || workspace_bytes < evo_attn_fwd_workspace_size(d)) return fail(EVO_ERR_VALIDATION, "workspace too small");
  const int path = resolve(d);
  if (path < 0) return fail(EVO_ERR_UNSUPPORTED, "tcgen05 path requested for an ineligible shape/dtype/scale/device");
  cudaStream_t cs = (cudaStream_t)stream;
  int* flag = (int*)workspace;
  if ((st = numeric_begin(d, flag, cs))) return st;
  evo::Shape s = make_shape(d, bias1, bias2, flag);
  s.gate = gate;
  if (path == EVO_PATH_TCGEN05) {
    st = evo::tc::fwd(d, s, q, k, v, o, lse, (char*)workspace + kHeader, cs, &g_launches, &g_err);
    if (st) return st;
  } else {
    switch (d->dtype) {
      case EVO_F32: st = simt_fwd_dispatch<float>(s, q, k, v, o, lse, cs); break;
      case EVO_BF16: st = simt_fwd_dispatch<__nv_bfloat16>(s, q, k, v, o, lse, cs); break;
      default: st = simt_fwd_dispatch<__half>(s, q, k, v, o, lse, cs); break;
    }
    if (st) return st;
  }
  return numeric_end(d, flag, cs, "attention logits are not finite or an input contains NaN (Q, K, V, bias)");
}

evo_status evo_attn_fwd(const evo_attn_desc* d, const void* q, const void* k, const void* v,
                        const void* bias1, const void* bias2, void* o, float* lse,
                        void* workspace, size_t workspace_bytes, evo_stream_t stream) {
  g_launches = 0;
  g_err.clear();
  evo_status st = validate(d);
  if (st) return st;
  if (d->has_gate) return fail(EVO_ERR_VALIDATION, "desc.has_gate: use evo_attn_fwd_gated");
  return fwd_impl(d, q, k, v, bias1, bias2, nullptr, o, lse, workspace, workspace_bytes, stream);
}

evo_status evo_attn_fwd_gated(const evo_attn_desc* d, const void* q, const void* k, const void* v,
                              const void* bias1, const void* bias2, const void* gate, void* o, float* lse,
                              void* workspace, size_t workspace_bytes, evo_stream_t stream) {
  g_launches = 0;
  g_err.clear();
  evo_status st = validate(d);
  if (st) return st;
  if (!d->has_gate || !gate) return fail(EVO_ERR_VALIDATION, "the gated forward needs desc.has_gate and a gate tensor");
  return fwd_impl(d, q, k, v, bias1, bias2, gate, o, lse, workspace, workspace_bytes, stream);
}

static evo_status bwd_impl(const evo_attn_desc* d, const void* dout, const void* q, const void* k,
                           const void* v, const void* bias1, const void* bias2, const void* gate, const void* o,
                           const float* lse, void* dq, void* dk, void* dv, void* dgate, void* dbias1,
                           void* dbias2, int accumulate_dbias, void* workspace, size_t workspace_bytes,
                           evo_stream_t stream) {
  evo_status st = EVO_OK;
  if (!dout || !q || !k || !v || !o || !lse || !dq || !dk || !dv)
    return fail(EVO_ERR_VALIDATION, "dout, q, k, v, o, lse, dq, dk, dv must be non-null");
  if (d->has_bias1 != (bias1 != nullptr)) return fail(EVO_ERR_VALIDATION, "bias1 presence does not match the descriptor");
  if (d->has_bias2 != (bias2 != nullptr)) return fail(EVO_ERR_VALIDATION, "bias2 presence does not match the descriptor");
  if (dbias1 && !d->has_bias1) return fail(EVO_ERR_VALIDATION, "dbias1 requested without bias1");
  if (dbias1 && !d->need_dbias1)
    return fail(EVO_ERR_VALIDATION, "dbias1 requested but desc.need_dbias1 == 0 (workspace sized without it)");
  if (dbias2 && !d->has_bias2) return fail(EVO_ERR_VALIDATION, "dbias2 requested without bias2");
  if (accumulate_dbias && d->dbias_dtype != EVO_F32)
    return fail(EVO_ERR_VALIDATION, "accumulate_dbias requires dbias_dtype == EVO_F32");
  if (d->dbias2_multicast && (!dbias2 || d->dbias_dtype != EVO_F32 || !accumulate_dbias))
    return fail(EVO_ERR_VALIDATION,
                "dbias2_multicast needs dbias2 (this rank's replica), dbias_dtype EVO_F32 and accumulate_dbias");
  if (d->dbias2_multicast && d->deterministic)
    return fail(EVO_ERR_VALIDATION, "dbias2_multicast reduces across GPUs in arrival order: not deterministic");
  const BwdWs w = bwd_layout(d);
  if (!workspace || workspace_bytes < w.total) return fail(EVO_ERR_VALIDATION, "workspace too small");
  const int path = resolve(d);
  if (path < 0) return fail(EVO_ERR_UNSUPPORTED, "tcgen05 path requested for an ineligible shape/dtype/scale/device");
  const bool tc_bwd = path == EVO_PATH_TCGEN05 && evo::tc::bwd_available(d);
  if (d->path == EVO_PATH_TCGEN05 && !tc_bwd)
    return fail(EVO_ERR_UNSUPPORTED, "tcgen05 backward requested outside its envelope (16-bit, D 16/32, L % 8 == 0)");
  if (d->dbias2_multicast && !tc_bwd)
    return fail(EVO_ERR_UNSUPPORTED, "the multicast dBias2 reduction needs the tcgen05 backward (16-bit, D 16/32, L % 8 == 0)");
  cudaStream_t cs = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  int* flag = (int*)ws;
  if ((st = numeric_begin(d, flag, cs))) return st;
  evo::Shape s = make_shape(d, bias1, bias2, flag);
  s.gate = gate;
  s.dgate = dgate;
  s.dog = gate ? ws + w.dog : nullptr;
  float* delta = (float*)(ws + w.delta);
  // fp32 reduction targets: the caller's buffer when it is fp32, else workspace.
  const bool direct = d->dbias_dtype == EVO_F32;
  float* db2 = dbias2 ? (direct ? (float*)dbias2 : (float*)(ws + w.db2)) : nullptr;
  float* db1 = dbias1 ? (direct ? (float*)dbias1 : (float*)(ws + w.db1)) : nullptr;
  const size_t n2 = (size_t)d->Bo * d->H * d->L * d->L, n1 = (size_t)s.B * s.L;
  if (!accumulate_dbias) {
    if (db2) cudaMemsetAsync(db2, 0, n2 * 4, cs);
    if (db1) cudaMemsetAsync(db1, 0, n1 * 4, cs);
  }
  if (tc_bwd) {
    // the tcgen05 preamble computes delta itself
    st = evo::tc::bwd(d, s, dout, q, k, v, o, lse, nullptr, dq, dk, dv, db1, db2, ws + w.tc, cs,
                      &g_launches, &g_err);
  } else {
    switch (d->dtype) {  // delta = sum dout * o (with a gate: the gated output and its gradient)
      case EVO_F32: launch_delta<float>(s, dout, o, delta, cs); break;
      case EVO_BF16: launch_delta<__nv_bfloat16>(s, dout, o, delta, cs); break;
      default: launch_delta<__half>(s, dout, o, delta, cs); break;
    }
    if (gate) {  // gate backward: the attention kernels take dO = dout * sigmoid(G); dG written
      const size_t n = (size_t)s.B * s.L * s.H * s.D;
      const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
      switch (d->dtype) {
        case EVO_F32:
          evo::simt::gate_bwd_kernel<float><<<blocks, 256, 0, cs>>>(n, (const float*)dout, (const float*)o,
                                                                    (const float*)gate, (float*)s.dog, (float*)dgate);
          break;
        case EVO_BF16:
          evo::simt::gate_bwd_kernel<__nv_bfloat16><<<blocks, 256, 0, cs>>>(
              n, (const __nv_bfloat16*)dout, (const __nv_bfloat16*)o, (const __nv_bfloat16*)gate,
              (__nv_bfloat16*)s.dog, (__nv_bfloat16*)dgate);
          break;
        default:
          evo::simt::gate_bwd_kernel<__half><<<blocks, 256, 0, cs>>>(n, (const __half*)dout, (const __half*)o,
                                                                     (const __half*)gate, (__half*)s.dog, (__half*)dgate);
          break;
      }
      ++g_launches;
      dout = s.dog;
    }
    float* db1p = (float*)(ws + w.db1p);
    float* db2p = (float*)(ws + w.db2p);
    switch (d->dtype) {
      case EVO_F32:
        st = simt_bwd_dispatch<float>(d, s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, db1p, db2p, cs);
        break;
      case EVO_BF16:
        st = simt_bwd_dispatch<__nv_bfloat16>(d, s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, db1p, db2p, cs);
        break;
      default:
        st = simt_bwd_dispatch<__half>(d, s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, db1p, db2p, cs);
        break;
    }
  }
  if (st) return st;
  if (!direct) {
    if (d->dtype == EVO_BF16) {
      if (db2) launch_convert<__nv_bfloat16>(db2, dbias2, n2, cs);
      if (db1) launch_convert<__nv_bfloat16>(db1, dbias1, n1, cs);
    } else {
      if (db2) launch_convert<__half>(db2, dbias2, n2, cs);
      if (db1) launch_convert<__half>(db1, dbias1, n1, cs);
    }
  }
  return numeric_end(d, flag, cs, "dO or the recomputed gradients contain NaN / non-finite values");
}

evo_status evo_attn_bwd(const evo_attn_desc* d, const void* dout, const void* q, const void* k,
                        const void* v, const void* bias1, const void* bias2, const void* o,
                        const float* lse, void* dq, void* dk, void* dv, void* dbias1,
                        void* dbias2, int accumulate_dbias, void* workspace,
                        size_t workspace_bytes, evo_stream_t stream) {
  g_launches = 0;
  g_err.clear();
  evo_status st = validate(d);
  if (st) return st;
  if (d->has_gate) return fail(EVO_ERR_VALIDATION, "desc.has_gate: use evo_attn_bwd_gated");
  return bwd_impl(d, dout, q, k, v, bias1, bias2, nullptr, o, lse, dq, dk, dv, nullptr, dbias1, dbias2,
                  accumulate_dbias, workspace, workspace_bytes, stream);
}

evo_status evo_attn_bwd_gated(const evo_attn_desc* d, const void* dout, const void* q, const void* k,
                              const void* v, const void* bias1, const void* bias2, const void* gate,
                              const void* o, const float* lse, void* dq, void* dk, void* dv, void* dgate,
                              void* dbias1, void* dbias2, int accumulate_dbias, void* workspace,
                              size_t workspace_bytes, evo_stream_t stream) {
  g_launches = 0;
  g_err.clear();
  evo_status st = validate(d);
  if (st) return st;
  if (!d->has_gate || !gate || !dgate)
    return fail(EVO_ERR_VALIDATION, "the gated backward needs desc.has_gate, the gate and a dgate buffer");
  return bwd_impl(d, dout, q, k, v, bias1, bias2, gate, o, lse, dq, dk, dv, dgate, dbias1, dbias2,
                  accumulate_dbias, workspace, workspace_bytes, stream);
}

}  // extern "C"

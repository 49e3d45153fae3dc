// evoattn_capi.cu — the C-ABI (include/evoattn.h): validation with the
// reference's error taxonomy, workspace carving, and kernel dispatch.
//
// Validation mirrors AttentionProblem::validate (attention.cpp:49-86) and
// attn_backward_tiled's stats checks (attention_tiled.cpp:196-209), mapped to
// evo_status codes instead of exceptions (errors.hpp:15-30).
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
  if (d->axes_swapped != 0 && d->axes_swapped != 1)
    return fail(EVO_ERR_VALIDATION, "axes_swapped must be 0 or 1");
  if (d->axes_swapped && d->Bo != 1)
    return fail(EVO_ERR_VALIDATION, "axes_swapped (raw [L, N, H, D] layout) requires Bo == 1");
  if (d->Bo * d->N > 0x7fffffffLL || d->L > 65535 * 64LL || d->H > 65535)
    return fail(EVO_ERR_UNSUPPORTED, "extents exceed the kernels' index range");
  return EVO_OK;
}

bool tc_eligible(const evo_attn_desc* d) {
  return d->dtype != EVO_F32 && (d->D == 16 || d->D == 32 || d->D == 64) &&
         evo::tc::device_supported();
}

int resolve(const evo_attn_desc* d) {
  if (d->path == EVO_PATH_SIMT) return EVO_PATH_SIMT;
  if (d->path == EVO_PATH_TCGEN05) return tc_eligible(d) ? EVO_PATH_TCGEN05 : -1;
  return tc_eligible(d) ? EVO_PATH_TCGEN05 : EVO_PATH_SIMT;
}

evo::Shape make_shape(const evo_attn_desc* d, const void* b1, const void* b2) {
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
  return s;
}

// Bwd workspace layout: [delta B*H*L f32][dbias2 acc Bo*H*L*L f32][dbias1 acc B*L f32][tc scratch]
struct BwdWs {
  size_t delta, db2, db1, tc, total;
};

BwdWs bwd_layout(const evo_attn_desc* d) {
  BwdWs w{};
  const size_t B = (size_t)(d->Bo * d->N);
  size_t off = 0;
  w.delta = off;
  off += align_up(B * d->H * d->L * 4);
  w.db2 = off;
  if (d->has_bias2) off += align_up((size_t)d->Bo * d->H * d->L * d->L * 4);
  w.db1 = off;
  if (d->has_bias1 && d->need_dbias1) off += align_up(B * d->L * 4);
  w.tc = off;
  off += align_up(evo::tc::bwd_scratch_bytes(d));
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

template <typename T, int DP>
void simt_bwd(const evo::Shape& s, const void* dout, const void* q, const void* k, const void* v,
              const float* lse, const float* delta, void* dq, void* dk, void* dv, float* db1,
              float* db2, cudaStream_t st) {
  dim3 grid((s.L + evo::simt::Tiles<DP>::kRows - 1) / evo::simt::Tiles<DP>::kRows, s.H, s.B);
  evo::simt::dkdv_kernel<T, DP><<<grid, evo::simt::Tiles<DP>::kRows, 0, st>>>(
      s, (const T*)q, (const T*)k, (const T*)v, (const T*)dout, lse, delta, (T*)dk, (T*)dv, db1,
      db2);
  evo::simt::dq_kernel<T, DP><<<grid, evo::simt::Tiles<DP>::kRows, 0, st>>>(
      s, (const T*)q, (const T*)k, (const T*)v, (const T*)dout, lse, delta, (T*)dq);
  g_launches += 2;
}

template <typename T>
evo_status simt_bwd_dispatch(const evo::Shape& s, const void* dout, const void* q, const void* k,
                             const void* v, const float* lse, const float* delta, void* dq,
                             void* dk, void* dv, float* db1, float* db2, cudaStream_t st) {
  if (s.D <= 8) simt_bwd<T, 8>(s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, st);
  else if (s.D <= 16) simt_bwd<T, 16>(s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, st);
  else if (s.D <= 32) simt_bwd<T, 32>(s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, st);
  else if (s.D <= 64) simt_bwd<T, 64>(s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, st);
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

}  // namespace

extern "C" {

const char* evo_attn_version(void) { return "evoattn 0.1 sm_100a"; }
const char* evo_attn_last_error(void) { return g_err.c_str(); }
int evo_attn_last_launch_count(void) { return g_launches; }

int evo_attn_resolved_path(const evo_attn_desc* d) {
  if (validate(d) != EVO_OK) return -1;
  return resolve(d);
}

size_t evo_attn_fwd_workspace_size(const evo_attn_desc* d) {
  if (validate(d) != EVO_OK) return 0;
  return evo::tc::fwd_scratch_bytes(d);
}

size_t evo_attn_bwd_workspace_size(const evo_attn_desc* d) {
  if (validate(d) != EVO_OK) return 0;
  return bwd_layout(d).total;
}

evo_status evo_attn_fwd(const evo_attn_desc* d, const void* q, const void* k, const void* v,
                        const void* bias1, const void* bias2, void* o, float* lse,
                        void* workspace, size_t workspace_bytes, evo_stream_t stream) {
  g_launches = 0;
  g_err.clear();
  evo_status st = validate(d);
  if (st) return st;
  if (!q || !k || !v || !o || !lse) return fail(EVO_ERR_VALIDATION, "q, k, v, o, lse must be non-null");
  if (d->has_bias1 != (bias1 != nullptr)) return fail(EVO_ERR_VALIDATION, "bias1 presence does not match the descriptor");
  if (d->has_bias2 != (bias2 != nullptr)) return fail(EVO_ERR_VALIDATION, "bias2 presence does not match the descriptor");
  if (workspace_bytes < evo_attn_fwd_workspace_size(d)) return fail(EVO_ERR_VALIDATION, "workspace too small");
  const int path = resolve(d);
  if (path < 0) return fail(EVO_ERR_UNSUPPORTED, "tcgen05 path requested for an ineligible shape/dtype/device");
  cudaStream_t cs = (cudaStream_t)stream;
  const evo::Shape s = make_shape(d, bias1, bias2);
  if (path == EVO_PATH_TCGEN05) {
    st = evo::tc::fwd(d, s, q, k, v, o, lse, workspace, cs, &g_launches, &g_err);
    if (st) return st;
  } else {
    switch (d->dtype) {
      case EVO_F32: st = simt_fwd_dispatch<float>(s, q, k, v, o, lse, cs); break;
      case EVO_BF16: st = simt_fwd_dispatch<__nv_bfloat16>(s, q, k, v, o, lse, cs); break;
      default: st = simt_fwd_dispatch<__half>(s, q, k, v, o, lse, cs); break;
    }
    if (st) return st;
  }
  return check_launch();
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
  const BwdWs w = bwd_layout(d);
  if (!workspace || workspace_bytes < w.total) return fail(EVO_ERR_VALIDATION, "workspace too small");
  const int path = resolve(d);
  if (path < 0) return fail(EVO_ERR_UNSUPPORTED, "tcgen05 path requested for an ineligible shape/dtype/device");
  cudaStream_t cs = (cudaStream_t)stream;
  const evo::Shape s = make_shape(d, bias1, bias2);
  char* ws = (char*)workspace;
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
  const bool tc_bwd = path == EVO_PATH_TCGEN05 && evo::tc::bwd_available(d);
  if (d->dbias2_multicast && !tc_bwd)
    return fail(EVO_ERR_UNSUPPORTED, "the multicast dBias2 reduction needs the tcgen05 backward (16-bit, D 16/32, L % 8 == 0)");
  if (tc_bwd) {
    // the tcgen05 preamble computes delta itself
    st = evo::tc::bwd(d, s, dout, q, k, v, o, lse, nullptr, dq, dk, dv, db1, db2, ws + w.tc, cs,
                      &g_launches, &g_err);
  } else {
    switch (d->dtype) {
      case EVO_F32: launch_delta<float>(s, dout, o, delta, cs); break;
      case EVO_BF16: launch_delta<__nv_bfloat16>(s, dout, o, delta, cs); break;
      default: launch_delta<__half>(s, dout, o, delta, cs); break;
    }
    switch (d->dtype) {
      case EVO_F32:
        st = simt_bwd_dispatch<float>(s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, cs);
        break;
      case EVO_BF16:
        st = simt_bwd_dispatch<__nv_bfloat16>(s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, cs);
        break;
      default:
        st = simt_bwd_dispatch<__half>(s, dout, q, k, v, lse, delta, dq, dk, dv, db1, db2, cs);
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
  return check_launch();
}

}  // extern "C"

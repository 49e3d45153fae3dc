// evomem_gpu_adapter.cpp — the reference's tiled-attention operator API, served by the B200 kernels.
//
// Defines evomem::attn_forward_tiled / evomem::attn_backward_tiled with exactly the signatures of
// /root/reference/proj/core/include/evomem/attention_tiled.hpp:85-97, so any caller of the
// reference (its attn-bench / gradcheck harness in run.cpp:191-365, the benchmarks) links against
// this translation unit instead of attention_tiled.cpp and runs unchanged on the GPU. The adapter
// is a thin host shim over the C-ABI of include/evoattn.h: host Tensor -> device buffers -> one
// evo_attn_fwd / evo_attn_bwd call -> host Tensor. It mirrors the reference's contract:
//   * validation order and error taxonomy of attention_tiled.cpp:57-65, 182-209 (p.validate(),
//     tc.validate(), closed ledger -> UsageError, NaN in Q/K/V/bias/dO -> NumericError, row-stat
//     and output shape/format checks -> ValidationError); C-ABI statuses map 1:1 onto the same
//     exception classes;
//   * outputs in the problem format, RowStats.logsumexp (H, B, L) in widened_to_f32(format),
//     dbias (H, L, L) in F32 (AccumMode::UpcastF32);
//   * ledger records under the reference labels: "tiled/stats" (kept until the caller frees it),
//     "tiled/delta" and "tiled/work/..." (transient) — with the device working set as the bytes.
//   * AccumPolicy::deterministic (attention_tiled.hpp:35-44, the reference default) -> the C-ABI's
//     deterministic backward (every cross-CTA reduction in a fixed order: two runs are bit-identical,
//     SPEC.md:211); non-finite logits (attention_tiled.cpp:125-127) -> the kernels' numeric checks.
// Differences (documented in INTEGRATION.md): F64 problems and AccumMode::NativeFormat are not
// served by the GPU kernels (ValidationError); TileConfig is validated but does not steer the kernels, which use
// their own B200 tiling, results are tile-independent within the format tolerance; the
// deterministic order is the kernels' own fixed order, not the reference's ascending-b recurrence.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <optional>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "evoattn.h"
#include "evomem/attention.hpp"
#include "evomem/attention_tiled.hpp"
#include "evomem/errors.hpp"
#include "evomem/ledger.hpp"
#include "evomem/tensor.hpp"

namespace evomem {
namespace {

[[noreturn]] void raise(evo_status st, const std::string& where) {
  const std::string msg = where + ": " + evo_attn_last_error();
  switch (st) {
    case EVO_ERR_VALIDATION: throw ValidationError(msg);
    case EVO_ERR_NUMERIC: throw NumericError(msg);
    case EVO_ERR_USAGE: throw UsageError(msg);
    default: throw Error(msg);
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

void reject_nan(const Tensor& t, const char* name) {
  for (std::int64_t i = 0; i < t.size(); ++i)
    if (std::isnan(t.at(i))) throw NumericError(std::string(name) + " has a NaN entry");
}

evo_dtype dtype_of(NumericFormat f) {
  switch (f) {
    case NumericFormat::F32: return EVO_F32;
    case NumericFormat::BF16: return EVO_BF16;
    case NumericFormat::F16: return EVO_F16;
    default: throw ValidationError("the GPU backend serves F32, BF16 and F16 problems (got F64)");
  }
}
int elem_bytes(evo_dtype t) { return t == EVO_F32 ? 4 : 2; }

// Stored values are exactly representable in the tensor's format, so these conversions are exact.
uint16_t to_bf16_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}
float from_bf16_bits(uint16_t b) {
  const uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
uint16_t to_f16_bits(float f) {  // exact for values already on the binary16 grid
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t sign = (u >> 16) & 0x8000u;
  const int exp = (int)((u >> 23) & 0xFF) - 127;
  const uint32_t man = u & 0x7FFFFFu;
  if (((u >> 23) & 0xFF) == 0xFF) return (uint16_t)(sign | 0x7C00u | (man ? 0x200u : 0u));
  if (exp > 15) return (uint16_t)(sign | 0x7C00u);
  if (exp >= -14) return (uint16_t)(sign | ((uint32_t)(exp + 15) << 10) | (man >> 13));
  if (exp >= -25) return (uint16_t)(sign | ((man | 0x800000u) >> (-exp - 1)));  // subnormal grid
  return (uint16_t)sign;
}
float from_f16_bits(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t exp = (h >> 10) & 0x1F, man = h & 0x3FFu;
  float f;
  if (exp == 0) {
    f = std::ldexp((float)man, -24);
    if (sign) f = -f;
    return f;
  }
  const uint32_t u = exp == 0x1F ? (sign | 0x7F800000u | (man << 13)) : (sign | ((exp + 112) << 23) | (man << 13));
  std::memcpy(&f, &u, 4);
  return f;
}

// A device copy of a host Tensor in the GPU dtype (or a zeroed output buffer).
class DeviceBuffer {
 public:
  DeviceBuffer(std::int64_t n, evo_dtype t) : n_(n), t_(t) {
    cuda_check(cudaMalloc(&p_, (size_t)std::max<std::int64_t>(n, 1) * elem_bytes(t)), "cudaMalloc");
  }
  DeviceBuffer(const Tensor& src, evo_dtype t) : DeviceBuffer(src.size(), t) {
    std::vector<uint8_t> h((size_t)n_ * elem_bytes(t_));
    for (std::int64_t i = 0; i < n_; ++i) {
      const float f = (float)src.at(i);
      if (t_ == EVO_F32) std::memcpy(h.data() + 4 * i, &f, 4);
      else {
        const uint16_t b = t_ == EVO_BF16 ? to_bf16_bits(f) : to_f16_bits(f);
        std::memcpy(h.data() + 2 * i, &b, 2);
      }
    }
    cuda_check(cudaMemcpy(p_, h.data(), h.size(), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
  ~DeviceBuffer() { cudaFree(p_); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void* get() const { return p_; }
  std::vector<double> fetch() const {
    std::vector<uint8_t> h((size_t)n_ * elem_bytes(t_));
    cuda_check(cudaMemcpy(h.data(), p_, h.size(), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    std::vector<double> v((size_t)n_);
    for (std::int64_t i = 0; i < n_; ++i) {
      if (t_ == EVO_F32) {
        float f;
        std::memcpy(&f, h.data() + 4 * i, 4);
        v[(size_t)i] = f;
      } else {
        uint16_t b;
        std::memcpy(&b, h.data() + 2 * i, 2);
        v[(size_t)i] = t_ == EVO_BF16 ? from_bf16_bits(b) : from_f16_bits(b);
      }
    }
    return v;
  }

 private:
  void* p_ = nullptr;
  std::int64_t n_;
  evo_dtype t_;
};

evo_attn_desc describe(const AttentionProblem& p) {
  evo_attn_desc d{};
  d.Bo = 1;  // the reference has one bias shared by every batch row (attention.hpp:24-31)
  d.N = p.batch();
  d.L = p.seq();
  d.H = p.heads();
  d.D = p.head_dim();
  d.dtype = dtype_of(p.format());
  d.scale = p.scale;
  d.has_bias1 = 0;  // the reference has no mask bias
  d.has_bias2 = p.bias.has_value() ? 1 : 0;
  d.dbias_dtype = EVO_F32;
  d.path = EVO_PATH_AUTO;
  d.check_numerics = 1;  // NumericError for non-finite logit rows, as attention_tiled.cpp:125-127
  return d;
}

}  // namespace

// ---- the host-side helpers declared next to the operator (attention_tiled.hpp:18-20, 67-71)
void TileConfig::validate() const {
  if (tile_q >= 1 && tile_k >= 1 && tile_b >= 1) return;
  throw ValidationError("tile extents (q, k, b) must all be >= 1, got (" + std::to_string(tile_q) + ", " +
                        std::to_string(tile_k) + ", " + std::to_string(tile_b) + ")");
}

Tensor broadcast_bias_tile(const Tensor& bias, std::int64_t head, std::int64_t q_origin, std::int64_t k_origin,
                           const TileConfig& tc) {
  tc.validate();
  if (bias.rank() != 3 || bias.extent(1) != bias.extent(2))
    throw ValidationError("bias must be (H, L, L); got " + bias.shape_str());
  const std::int64_t H = bias.extent(0), L = bias.extent(1);
  if (head < 0 || head >= H) throw ValidationError("bias head " + std::to_string(head) + " outside [0, H)");
  if (q_origin < 0 || k_origin < 0 || q_origin >= L || k_origin >= L)
    throw ValidationError("bias tile origin outside the (L, L) plane");
  const std::int64_t nq = std::min(tc.tile_q, L - q_origin), nk = std::min(tc.tile_k, L - k_origin);
  std::vector<double> vals((size_t)(nq * nk));
  const std::int64_t plane = head * L * L;
  for (std::int64_t r = 0; r < nq; ++r)
    for (std::int64_t c = 0; c < nk; ++c) vals[(size_t)(r * nk + c)] = bias.at(plane + (q_origin + r) * L + k_origin + c);
  return Tensor::from_values({nq, nk}, bias.format(), vals);
}

TiledForwardResult attn_forward_tiled(const AttentionProblem& p, const TileConfig& tc, AllocationLedger& ledger) {
  p.validate();
  tc.validate();
  if (ledger.closed()) throw UsageError("allocation ledger is closed");
  reject_nan(p.query, "Q");
  reject_nan(p.key, "K");
  reject_nan(p.value, "V");
  if (p.bias.has_value()) reject_nan(*p.bias, "bias");

  const evo_attn_desc d = describe(p);
  const std::int64_t B = p.batch(), L = p.seq(), H = p.heads(), D = p.head_dim();
  DeviceBuffer q(p.query, d.dtype), k(p.key, d.dtype), v(p.value, d.dtype);
  std::optional<DeviceBuffer> b2;
  if (p.bias.has_value()) b2.emplace(*p.bias, d.dtype);
  DeviceBuffer o(B * L * H * D, d.dtype), lse(B * H * L, EVO_F32);
  const size_t ws_bytes = evo_attn_fwd_workspace_size(&d);
  DeviceBuffer ws((std::int64_t)ws_bytes, EVO_BF16);

  Tensor lse_t({H, B, L}, widened_to_f32(p.format()));
  LedgerScope scope(ledger, "tiled");
  ledger.record_alloc("stats", lse_t.emulated_bytes());
  {
    ScopedAllocation work(&ledger, "work/device_workspace", (std::int64_t)ws_bytes);
    const evo_status st = evo_attn_fwd(&d, q.get(), k.get(), v.get(), nullptr, b2 ? b2->get() : nullptr, o.get(),
                                       (float*)lse.get(), ws.get(), ws_bytes, nullptr);
    if (st != EVO_OK) raise(st, "evo_attn_fwd");
    cuda_check(cudaDeviceSynchronize(), "evo_attn_fwd");
  }
  const std::vector<double> ov = o.fetch(), lv = lse.fetch();
  Tensor out = Tensor::from_values({B, L, H, D}, p.format(), ov);
  // kernel LSE is [B, H, L]; the reference keeps (H, B, L)
  for (std::int64_t b = 0; b < B; ++b)
    for (std::int64_t h = 0; h < H; ++h)
      for (std::int64_t i = 0; i < L; ++i) lse_t.set((h * B + b) * L + i, lv[(size_t)((b * H + h) * L + i)]);
  return TiledForwardResult{std::move(out), RowStats{std::move(lse_t)}};
}

AttentionGrads attn_backward_tiled(const AttentionProblem& p, const Tensor& output, const RowStats& stats,
                                   const Tensor& grad_output, const TileConfig& tc, const AccumPolicy& policy,
                                   AllocationLedger& ledger) {
  p.validate();
  tc.validate();
  if (ledger.closed()) throw UsageError("allocation ledger is closed");
  const std::int64_t B = p.batch(), L = p.seq(), H = p.heads(), D = p.head_dim();
  const NumericFormat fmt = p.format();
  const Tensor& lse = stats.logsumexp;
  if (lse.rank() != 3 || lse.extent(0) != H || lse.extent(1) != B || lse.extent(2) != L)
    throw ValidationError("row stats must be (H, B, L), got " + lse.shape_str());
  if (lse.format() != widened_to_f32(fmt)) throw ValidationError("row stats format does not match the problem");
  if (!output.same_shape(p.query) || !grad_output.same_shape(p.query))
    throw ValidationError("output and grad_output must have the Q/K/V shape");
  if (output.format() != fmt || grad_output.format() != fmt)
    throw ValidationError("output and grad_output must be in the problem format");
  reject_nan(grad_output, "dO");
  if (policy.mode != AccumMode::UpcastF32)
    throw ValidationError("the GPU backend reduces the bias gradient in F32 (AccumMode::UpcastF32)");

  evo_attn_desc d = describe(p);
  d.deterministic = policy.deterministic ? 1 : 0;  // AccumPolicy::deterministic (attention_tiled.cpp:246-252)
  DeviceBuffer q(p.query, d.dtype), k(p.key, d.dtype), v(p.value, d.dtype);
  DeviceBuffer o(output, d.dtype), dout(grad_output, d.dtype);
  std::optional<DeviceBuffer> b2;
  if (p.bias.has_value()) b2.emplace(*p.bias, d.dtype);
  // LSE back to the kernel layout [B, H, L]
  Tensor lse_k({B, H, L}, NumericFormat::F32);
  for (std::int64_t h = 0; h < H; ++h)
    for (std::int64_t b = 0; b < B; ++b)
      for (std::int64_t i = 0; i < L; ++i) lse_k.set((b * H + h) * L + i, lse.at((h * B + b) * L + i));
  DeviceBuffer lse_d(lse_k, EVO_F32);
  DeviceBuffer dq(B * L * H * D, d.dtype), dk(B * L * H * D, d.dtype), dv(B * L * H * D, d.dtype);
  std::optional<DeviceBuffer> db2;
  if (p.bias.has_value()) db2.emplace(H * L * L, EVO_F32);
  const size_t ws_bytes = evo_attn_bwd_workspace_size(&d);
  DeviceBuffer ws((std::int64_t)ws_bytes, EVO_BF16);

  LedgerScope scope(ledger, "tiled");
  {
    ScopedAllocation delta(&ledger, "delta", B * L * H * 4);
    ScopedAllocation work(&ledger, "work/device_workspace", (std::int64_t)ws_bytes);
    const evo_status st =
        evo_attn_bwd(&d, dout.get(), q.get(), k.get(), v.get(), nullptr, b2 ? b2->get() : nullptr, o.get(),
                     (const float*)lse_d.get(), dq.get(), dk.get(), dv.get(), nullptr, db2 ? db2->get() : nullptr,
                     /*accumulate_dbias=*/0, ws.get(), ws_bytes, nullptr);
    if (st != EVO_OK) raise(st, "evo_attn_bwd");
    cuda_check(cudaDeviceSynchronize(), "evo_attn_bwd");
  }
  AttentionGrads g;
  g.dquery = Tensor::from_values({B, L, H, D}, fmt, dq.fetch());
  g.dkey = Tensor::from_values({B, L, H, D}, fmt, dk.fetch());
  g.dvalue = Tensor::from_values({B, L, H, D}, fmt, dv.fetch());
  if (db2) g.dbias = Tensor::from_values({H, L, L}, widened_to_f32(fmt), db2->fetch());
  return g;
}

}  // namespace evomem

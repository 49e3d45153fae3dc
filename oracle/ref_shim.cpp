// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference
// library (evomem, /root/reference/proj/core), compiled by oracle/Makefile
// into oracle/_ref/libevomem_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (evo_oracle.c) to
// the reference bit for bit, to generate tests/golden fixtures, and as the
// CPU baseline (`bench.py --impl reference`). It calls the reference's own
// public operator API:
//   attn_forward_tiled   attention_tiled.hpp:85-86
//   attn_backward_tiled  attention_tiled.hpp:94-97
//   attn_forward_ref / attn_backward_ref  attention.hpp:90-97
// The reference has no bias1 (mask) term; callers pass the pair bias only.
#include <evomem/attention.hpp>
#include <evomem/attention_tiled.hpp>
#include <evomem/errors.hpp>
#include <evomem/ledger.hpp>
#include <evomem/memory_model.hpp>
#include <evomem/rng.hpp>

#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using namespace evomem;

namespace {

thread_local std::string g_err;

Tensor make_tensor(std::vector<std::int64_t> shape, NumericFormat f, const double* src) {
  Tensor t(std::move(shape), f);
  for (std::int64_t i = 0; i < t.size(); ++i) t.set(i, src[i]);
  return t;
}

void copy_out(const Tensor& t, double* dst) {
  for (std::int64_t i = 0; i < t.size(); ++i) dst[i] = t.at(i);
}

NumericFormat fmt_of(int f) {
  switch (f) {
    case 0: return NumericFormat::F64;
    case 1: return NumericFormat::F32;
    case 2: return NumericFormat::BF16;
    default: return NumericFormat::F16;
  }
}

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ValidationError*>(&e)) return 1;
  if (dynamic_cast<const NumericError*>(&e)) return 2;
  if (dynamic_cast<const UsageError*>(&e)) return 3;
  return 4;
}

AttentionProblem problem(int variant, int fmt, std::int64_t B, std::int64_t L, std::int64_t H,
                         std::int64_t D, const double* q, const double* k, const double* v,
                         const double* bias, double scale) {
  const NumericFormat f = fmt_of(fmt);
  std::optional<Tensor> b;
  if (bias) b = make_tensor({H, L, L}, f, bias);
  return AttentionProblem::make(static_cast<AttentionVariant>(variant),
                                make_tensor({B, L, H, D}, f, q), make_tensor({B, L, H, D}, f, k),
                                make_tensor({B, L, H, D}, f, v), std::move(b), scale);
}

}  // namespace

extern "C" {

const char* evomem_ref_last_error() { return g_err.c_str(); }

// Tiled forward + backward through the reference API on one problem.
// Outputs: o (B,L,H,D), lse (H,B,L), dq/dk/dv (B,L,H,D), dbias (H,L,L) or null.
// Returns 0, or 1/2/3/4 for Validation/Numeric/Usage/other errors.
int evomem_ref_tiled(int variant, int fmt, std::int64_t B, std::int64_t L, std::int64_t H,
                     std::int64_t D, const double* q, const double* k, const double* v,
                     const double* bias, const double* dout, double scale, std::int64_t tile_q,
                     std::int64_t tile_k, std::int64_t tile_b, int deterministic, double* o,
                     double* lse, double* dq, double* dk, double* dv, double* dbias,
                     std::int64_t* peak_bytes) {
  try {
    AttentionProblem p = problem(variant, fmt, B, L, H, D, q, k, v, bias, scale);
    const TileConfig tc{tile_q, tile_k, tile_b};
    AllocationLedger ledger;
    TiledForwardResult fwd = attn_forward_tiled(p, tc, ledger);
    copy_out(fwd.output, o);
    copy_out(fwd.stats.logsumexp, lse);
    if (dout) {
      Tensor g = make_tensor({B, L, H, D}, p.format(), dout);
      AccumPolicy pol;
      pol.deterministic = deterministic != 0;
      AttentionGrads gr = attn_backward_tiled(p, fwd.output, fwd.stats, g, tc, pol, ledger);
      copy_out(gr.dquery, dq);
      copy_out(gr.dkey, dk);
      copy_out(gr.dvalue, dv);
      if (dbias && gr.dbias) copy_out(*gr.dbias, dbias);
    }
    if (peak_bytes) *peak_bytes = ledger.measure_peak().peak_bytes;
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Materialising oracle of the reference (attention.cpp:168-353).
int evomem_ref_naive(int variant, int fmt, std::int64_t B, std::int64_t L, std::int64_t H,
                     std::int64_t D, const double* q, const double* k, const double* v,
                     const double* bias, const double* dout, double scale, double* o, double* dq,
                     double* dk, double* dv, double* dbias, std::int64_t* peak_bytes) {
  try {
    AttentionProblem p = problem(variant, fmt, B, L, H, D, q, k, v, bias, scale);
    AllocationLedger ledger;
    ForwardResult fwd = attn_forward_ref(p, &ledger);
    copy_out(fwd.output, o);
    if (dout) {
      Tensor g = make_tensor({B, L, H, D}, p.format(), dout);
      AttentionGrads gr = attn_backward_ref(p, fwd.probs, g, &ledger);
      copy_out(gr.dquery, dq);
      copy_out(gr.dkey, dk);
      copy_out(gr.dvalue, dv);
      if (dbias && gr.dbias) copy_out(*gr.dbias, dbias);
    }
    if (peak_bytes) *peak_bytes = ledger.measure_peak().peak_bytes;
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// The CPU baseline: reference tiled fwd+bwd in F32 on `threads` row shards
// (one problem + ledger per shard; the reference is reentrant),
// per-shard dbias summed in ascending shard order. Inputs are float arrays.
int evomem_ref_tiled_threaded_f32(std::int64_t B, std::int64_t L, std::int64_t H, std::int64_t D,
                                  const float* q, const float* k, const float* v,
                                  const float* bias, const float* dout, double scale, int threads,
                                  float* o, float* dq, float* dk, float* dv, float* dbias) {
  if (threads < 1) threads = 1;
  if (threads > B) threads = static_cast<int>(B);
  const std::int64_t row = L * H * D;
  std::vector<std::vector<float>> dbias_part(threads);
  std::vector<int> status(threads, 0);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const std::int64_t r0 = B * t / threads, r1 = B * (t + 1) / threads, nb = r1 - r0;
      try {
        auto mk = [&](const float* src) {
          Tensor x({nb, L, H, D}, NumericFormat::F32);
          for (std::int64_t i = 0; i < x.size(); ++i) x.set(i, src[r0 * row + i]);
          return x;
        };
        std::optional<Tensor> bt;
        if (bias) {
          Tensor b({H, L, L}, NumericFormat::F32);
          for (std::int64_t i = 0; i < b.size(); ++i) b.set(i, bias[i]);
          bt = std::move(b);
        }
        AttentionProblem p = AttentionProblem::make(
            bias ? AttentionVariant::MsaRowWise : AttentionVariant::MsaColumnWise, mk(q), mk(k),
            mk(v), std::move(bt), scale);
        AllocationLedger ledger;
        TileConfig tc;
        TiledForwardResult fwd = attn_forward_tiled(p, tc, ledger);
        Tensor g = mk(dout);
        AttentionGrads gr = attn_backward_tiled(p, fwd.output, fwd.stats, g, tc, AccumPolicy{}, ledger);
        for (std::int64_t i = 0; i < nb * row; ++i) {
          o[r0 * row + i] = static_cast<float>(fwd.output.at(i));
          dq[r0 * row + i] = static_cast<float>(gr.dquery.at(i));
          dk[r0 * row + i] = static_cast<float>(gr.dkey.at(i));
          dv[r0 * row + i] = static_cast<float>(gr.dvalue.at(i));
        }
        if (gr.dbias) {
          dbias_part[t].resize(static_cast<std::size_t>(gr.dbias->size()));
          for (std::int64_t i = 0; i < gr.dbias->size(); ++i)
            dbias_part[t][static_cast<std::size_t>(i)] = static_cast<float>(gr.dbias->at(i));
        }
      } catch (const std::exception& e) {
        status[t] = status_of(e);
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int s : status)
    if (s) return s;
  if (bias && dbias) {
    const std::int64_t n = H * L * L;
    for (std::int64_t i = 0; i < n; ++i) {
      float a = 0.f;
      for (int t = 0; t < threads; ++t) a += dbias_part[t][static_cast<std::size_t>(i)];
      dbias[i] = a;
    }
  }
  return 0;
}

// The reference's own instance generator (rng.hpp:41-47, rng.cpp:5-10): `skip` draws of
// derived_rng(seed, stream) are consumed, then n values of random_uniform in format `fmt` (values
// out as doubles). Pins the product-side port (evo_random_uniform) bit for bit.
int evomem_ref_random_uniform(std::uint64_t seed, std::uint64_t stream, std::int64_t skip, std::int64_t n,
                              int fmt, double lo, double hi, double* out) {
  try {
    SeededRng rng = derived_rng(seed, stream);
    for (std::int64_t i = 0; i < skip; ++i) rng.next_u64();
    Tensor t = random_uniform({n}, fmt_of(fmt), rng, lo, hi);
    copy_out(t, out);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// memory_model.hpp analytic bytes (naive vs tiled), for the peak-memory report.
std::int64_t evomem_ref_analytic_bytes(std::int64_t H, std::int64_t B, std::int64_t L,
                                       std::int64_t D, int bytes_per_elem, int tiled, int backward,
                                       std::int64_t tile_q, std::int64_t tile_k, std::int64_t workers) {
  try {
    AttentionDims dims{H, B, L, D, bytes_per_elem};
    TileConfig tc{tile_q, tile_k, 1};
    return analytic_attention_bytes(dims, tiled ? AttentionMode::Tiled : AttentionMode::Naive,
                                    backward ? AttentionPhase::Backward : AttentionPhase::Forward,
                                    &tc, workers)
        .total_bytes;
  } catch (const std::exception& e) {
    status_of(e);
    return -1;
  }
}

}  // extern "C"

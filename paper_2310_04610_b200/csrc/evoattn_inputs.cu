// evoattn_inputs.cu — host-side synthetic inputs identical to the reference's instance generator
// (not the hot path; no device code). The bench and the reference arm draw the same values, and
// tests pin this port bit for bit against the reference's own rng (oracle/_ref).
//
//   SeededRng         rng.hpp:16-37   std::mt19937_64; uniform() from the top 53 bits
//   derived_rng       rng.hpp:41-43   engine seeded with seed ^ (0x9E3779B97F4A7C15 * (stream + 1))
//   random_uniform    rng.cpp:5-10    lo + (hi - lo) * uniform(), rounded to the format on set()
//   round_to_format   numeric_format.cpp:42-78 (RNE with subnormals, saturating to +-inf),
//                     numeric_format.hpp:64-65 (F32 through a float cast)
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>

#include <cuda_fp16.h>

#include "../../include/evoattn.h"

namespace {

// numeric_format.cpp:42-78, the reference's exact formula (slow path: subnormals, overflow)
double round_emulated(double x, int mb, int eb) {
  if (x == 0.0 || !std::isfinite(x)) return x;
  const int bias = (1 << (eb - 1)) - 1;
  const int min_normal_exp = 1 - bias;
  int e2 = 0;
  std::frexp(x, &e2);
  const int lsb = std::max(e2 - 1, min_normal_exp) - mb;
  const double scaled = std::ldexp(x, -lsb);
  const double lower = std::floor(scaled);
  const double frac = scaled - lower;
  const double ri = frac > 0.5 ? lower + 1.0 : frac < 0.5 ? lower : (std::fmod(lower, 2.0) == 0.0 ? lower : lower + 1.0);
  const double r = std::ldexp(ri, lsb);
  const double maxf = (2.0 - std::ldexp(1.0, -mb)) * std::ldexp(1.0, bias);
  if (std::fabs(r) > maxf) return x > 0.0 ? std::numeric_limits<double>::infinity() : -std::numeric_limits<double>::infinity();
  return r;
}

// Same rounding on the double's bits for values whose result is a normal number of the format:
// keep mb fraction bits, round to nearest even (a carry into the exponent is the correct result).
inline double round_fast(double x, int mb, int eb) {
  const int bias = (1 << (eb - 1)) - 1;
  const double ax = std::fabs(x);
  if (!(ax >= std::ldexp(1.0, 1 - bias)) || ax >= std::ldexp(1.0, bias)) return round_emulated(x, mb, eb);
  uint64_t u;
  std::memcpy(&u, &x, 8);
  const int sh = 52 - mb;
  u += ((uint64_t)1 << (sh - 1)) - 1 + ((u >> sh) & 1);
  u &= ~(((uint64_t)1 << sh) - 1);
  double r;
  std::memcpy(&r, &u, 8);
  return r;
}

inline uint16_t bits16(double r, bool f16) {
  if (f16) {
    const __half h = __double2half(r);  // exact: r is on the f16 grid
    uint16_t b;
    std::memcpy(&b, &h, 2);
    return b;
  }
  const float f = (float)r;  // exact: r is on the bf16 grid (a subset of f32)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}

}  // namespace

extern "C" evo_status evo_random_uniform(uint64_t seed, uint64_t stream, int64_t skip, int64_t n, double lo,
                                         double hi, evo_dtype dtype, void* out) {
  if (!out || n < 0 || skip < 0) return EVO_ERR_VALIDATION;
  std::mt19937_64 eng(seed ^ (0x9E3779B97F4A7C15ULL * (stream + 1)));
  if (skip) eng.discard((unsigned long long)skip);
  const double span = hi - lo;
  auto draw = [&]() { return lo + span * ((double)(eng() >> 11) * 0x1.0p-53); };
  switch (dtype) {
    case EVO_F32: {
      float* o = (float*)out;
      for (int64_t i = 0; i < n; ++i) o[i] = (float)draw();
      return EVO_OK;
    }
    case EVO_BF16:
    case EVO_F16: {
      const bool f16 = dtype == EVO_F16;
      uint16_t* o = (uint16_t*)out;
      for (int64_t i = 0; i < n; ++i) o[i] = bits16(round_fast(draw(), f16 ? 10 : 7, f16 ? 5 : 8), f16);
      return EVO_OK;
    }
    default:
      return EVO_ERR_VALIDATION;
  }
}

extern "C" evo_status evo_random_mask(uint64_t seed, uint64_t stream, int64_t rows, int64_t row0, int64_t L,
                                      double rate, double neg, evo_dtype dtype, void* out) {
  if (!out || rows < 0 || row0 < 0 || L < 1) return EVO_ERR_VALIDATION;
  std::mt19937_64 eng(seed ^ (0x9E3779B97F4A7C15ULL * (stream + 1)));
  if (row0) eng.discard((unsigned long long)(row0 * L));
  const uint16_t nb = bits16(round_emulated(neg, dtype == EVO_F16 ? 10 : 7, dtype == EVO_F16 ? 5 : 8), dtype == EVO_F16);
  for (int64_t b = 0; b < rows; ++b)
    for (int64_t j = 0; j < L; ++j) {
      const bool m = ((double)(eng() >> 11) * 0x1.0p-53) < rate && j != 0;  // key 0 never masked
      if (dtype == EVO_F32) ((float*)out)[b * L + j] = m ? (float)neg : 0.f;
      else ((uint16_t*)out)[b * L + j] = m ? nb : (uint16_t)0;
    }
  return EVO_OK;
}

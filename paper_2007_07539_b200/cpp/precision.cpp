// Host binary16 helpers of the C++ drop-in layer (precision.hpp). Rounding
// is the library's own RNE-with-gradual-underflow routine (C ABI
// mpmg_round_fp16, csrc/mpmg_host.cpp), the same one every device kernel's
// level scalars go through. Single-rounded fma uses the round-to-odd
// argument: v = a*b + c is exact as s + e (TwoSum, e exact); replacing s by
// its odd neighbour toward e when e != 0 gives a binary64 value whose
// binary16 rounding equals that of v (53 >= 2*11 + 2).
#include <cmath>
#include <cstring>

#include "mpmg/precision.hpp"
#include "mpmg_gpu.h"

namespace mpmg {

namespace {

std::uint64_t bits_of(double x) {
  std::uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}

// exact a*b + c as a binary64 value rounded to odd
double sum_to_odd(double p, double c) {
  const double s = p + c;
  if (!std::isfinite(s)) return s;
  const double bb = s - p;
  const double e = (p - (s - bb)) + (c - bb);  // TwoSum error, exact
  if (e == 0.0 || (bits_of(s) & 1u)) return s;
  return std::nextafter(s, e > 0 ? INFINITY : -INFINITY);
}

}  // namespace

double quantize_fp16(double x, bool flush_subnormals) noexcept { return mpmg_round_fp16(x, flush_subnormals ? 1 : 0); }

Fp16Value round_to_fp16(double x, const ArithmeticPolicy& policy) noexcept {
  return pack_fp16(quantize_fp16(x, policy.flush_subnormals_to_zero));
}

double widen(Fp16Value h) noexcept {
  const unsigned s = h.bits >> 15, e = (h.bits >> 10) & 0x1Fu, m = h.bits & 0x3FFu;
  double v;
  if (e == 0) v = std::ldexp(static_cast<double>(m), -24);
  else if (e == 0x1F) v = m ? std::nan("") : INFINITY;
  else v = std::ldexp(static_cast<double>(m | 0x400u), static_cast<int>(e) - 25);
  return s ? -v : v;
}

float widen_f(Fp16Value h) noexcept { return static_cast<float>(widen(h)); }

Fp16Value pack_fp16(double v) noexcept {
  const std::uint16_t sign = std::signbit(v) ? 0x8000u : 0u;
  const double a = std::fabs(v);
  if (std::isnan(v)) return Fp16Value{0x7E00u};
  if (std::isinf(v)) return Fp16Value{static_cast<std::uint16_t>(sign | 0x7C00u)};
  if (a == 0.0) return Fp16Value{sign};
  if (a < kFp16MinNormal) return Fp16Value{static_cast<std::uint16_t>(sign | static_cast<unsigned>(std::ldexp(a, 24)))};
  int ex = 0;
  const double fr = std::frexp(a, &ex);  // a = fr * 2^ex, fr in [0.5, 1)
  const unsigned mant = static_cast<unsigned>(std::ldexp(fr, 11)) & 0x3FFu;
  return Fp16Value{static_cast<std::uint16_t>(sign | (static_cast<unsigned>(ex + 14) << 10) | mant)};
}

double fp16_add_value(double a, double b, bool flush) noexcept { return quantize_fp16(sum_to_odd(a, b), flush); }

double fp16_mul_value(double a, double b, bool flush) noexcept {
  return quantize_fp16(a * b, flush);  // exact: 11 x 11 bits
}

double fp16_fma_value(double a, double b, double c, const ArithmeticPolicy& p) noexcept {
  const bool f = p.flush_subnormals_to_zero;
  if (p.fused_multiply_add) return quantize_fp16(sum_to_odd(a * b, c), f);
  return fp16_add_value(fp16_mul_value(a, b, f), c, f);
}

Fp16Value fp16_add(Fp16Value a, Fp16Value b, const ArithmeticPolicy& p) noexcept {
  return pack_fp16(fp16_add_value(widen(a), widen(b), p.flush_subnormals_to_zero));
}
Fp16Value fp16_mul(Fp16Value a, Fp16Value b, const ArithmeticPolicy& p) noexcept {
  return pack_fp16(fp16_mul_value(widen(a), widen(b), p.flush_subnormals_to_zero));
}
Fp16Value fp16_fma(Fp16Value a, Fp16Value b, Fp16Value c, const ArithmeticPolicy& p) noexcept {
  return pack_fp16(fp16_fma_value(widen(a), widen(b), widen(c), p));
}

}  // namespace mpmg

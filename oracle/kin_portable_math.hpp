// oracle/kin_portable_math.hpp — TEST INFRASTRUCTURE ONLY.
//
// x^y for x > 0 built from IEEE-754 operations that are correctly rounded on
// every platform (+ - * /, floor, exponent bit manipulation) evaluated in a
// fixed order with no contraction.  The LSODA step/order heuristics use it
// instead of libm's pow so the CPU oracle and the CUDA kernel
// (paper_1309_7695_b200/csrc/kin_lsoda.cu, which carries an independent copy)
// produce bit-identical step sequences.  Accuracy ~1e-15 relative: far beyond
// what a step-size heuristic needs.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

namespace kin_oracle {

inline double pm_bits_to_double(std::uint64_t b) {
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}
inline std::uint64_t pm_double_to_bits(double d) {
  std::uint64_t b;
  std::memcpy(&b, &d, 8);
  return b;
}

// natural log of a positive normal x
inline double pm_log(double x) {
  const std::uint64_t b = pm_double_to_bits(x);
  int e = static_cast<int>((b >> 52) & 0x7FF) - 1023;
  double m = pm_bits_to_double((b & 0x000FFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL);  // [1,2)
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e = e + 1;
  }
  const double s = (m - 1.0) / (m + 1.0);  // |s| <= 0.1716
  const double s2 = s * s;
  // 2*atanh(s) = 2(s + s^3/3 + ... + s^21/21)
  double p = 1.0 / 21.0;
  p = p * s2 + 1.0 / 19.0;
  p = p * s2 + 1.0 / 17.0;
  p = p * s2 + 1.0 / 15.0;
  p = p * s2 + 1.0 / 13.0;
  p = p * s2 + 1.0 / 11.0;
  p = p * s2 + 1.0 / 9.0;
  p = p * s2 + 1.0 / 7.0;
  p = p * s2 + 1.0 / 5.0;
  p = p * s2 + 1.0 / 3.0;
  p = p * s2 + 1.0;
  const double lm = 2.0 * s * p;
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double de = static_cast<double>(e);
  return de * ln2_hi + (de * ln2_lo + lm);
}

// exp(z) for |z| < 700
inline double pm_exp(double z) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double inv_ln2 = 1.44269504088896338700e+00;
  const double n = std::floor(z * inv_ln2 + 0.5);
  const double r = (z - n * ln2_hi) - n * ln2_lo;  // |r| <= ~0.347
  double p = 1.0 / 479001600.0;                     // 1/12!
  p = p * r + 1.0 / 39916800.0;
  p = p * r + 1.0 / 3628800.0;
  p = p * r + 1.0 / 362880.0;
  p = p * r + 1.0 / 40320.0;
  p = p * r + 1.0 / 5040.0;
  p = p * r + 1.0 / 720.0;
  p = p * r + 1.0 / 120.0;
  p = p * r + 1.0 / 24.0;
  p = p * r + 1.0 / 6.0;
  p = p * r + 0.5;
  p = p * r + 1.0;
  p = p * r + 1.0;
  const int ni = static_cast<int>(n);
  return p * pm_bits_to_double(static_cast<std::uint64_t>(ni + 1023) << 52);
}

// x^y, x > 0 (clamped into the normal range), |y*log x| < 700
inline double pm_pow(double x, double y) {
  if (x < 1e-300) x = 1e-300;
  if (x > 1e300) x = 1e300;
  return pm_exp(y * pm_log(x));
}

}  // namespace kin_oracle

// kin_pmath.cuh — portable log/exp/pow for the step-size heuristics of the
// LSODA and hybrid kernels: IEEE-754 operations that are correctly rounded on
// every platform (+ - * /, floor, exponent bit manipulation) in a fixed order
// with no contraction (the including TUs compile with -fmad=false), so the
// kernels' step sequences are reproducible bit for bit.  The oracle carries an
// independent copy (oracle/kin_portable_math.hpp).  Accuracy ~1e-15 relative.
#pragma once
#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

namespace kin {
namespace pmath {

__device__ __forceinline__ double pm_log(double x) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  int e = static_cast<int>((b >> 52) & 0x7FF) - 1023;
  double m = __longlong_as_double(static_cast<long long>((b & 0x000FFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL));
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e = e + 1;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
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
__device__ __forceinline__ double pm_exp(double z) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double inv_ln2 = 1.44269504088896338700e+00;
  const double n = floor(z * inv_ln2 + 0.5);
  const double r = (z - n * ln2_hi) - n * ln2_lo;
  double p = 1.0 / 479001600.0;
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
  return p * __longlong_as_double(static_cast<long long>(static_cast<uint64_t>(ni + 1023) << 52));
}
__device__ __forceinline__ double pm_pow(double x, double y) {
  if (x < 1e-300) x = 1e-300;
  if (x > 1e300) x = 1e300;
  return pm_exp(y * pm_log(x));
}

}  // namespace pmath
}  // namespace kin

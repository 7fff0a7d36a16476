// kin_device.cuh — device-side model tables, RNG and propensity helpers.
//
// Every function here mirrors, operation for operation, the CPU oracle
// (oracle/kin_oracle.cpp, oracle/kin_rng.hpp), which restates the reference
// (proj/src/rng.cpp, model.hpp, stochastic.hpp).  The stochastic translation
// unit is compiled with -fmad=false so + - * / round exactly as the oracle's
// -ffp-contract=off build; integer work (xoshiro256++, firing counts, state
// updates) is exact by construction.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#endif

#include "kin_tables.h"
#include "kin_pmath.cuh"
#include "../../include/kin_abi.h"

namespace kin {

constexpr uint64_t kPhi64 = 0x9E3779B97F4A7C15ULL;

// ---- table accessors (warp-uniform index -> constant-bank broadcast) -------
__device__ __forceinline__ double tab_rate(const KinTables& T, int j) {
  return reinterpret_cast<const double*>(T.blob + T.off_rate)[j];
}
__device__ __forceinline__ int tab_rate_axis(const KinTables& T, int j) {
  return reinterpret_cast<const int8_t*>(T.blob + T.off_rate_axis)[j];
}
__device__ __forceinline__ double tab_x0(const KinTables& T, int i) {
  return reinterpret_cast<const double*>(T.blob + T.off_x0)[i];
}
__device__ __forceinline__ int tab_x0_axis(const KinTables& T, int i) {
  return reinterpret_cast<const int8_t*>(T.blob + T.off_x0_axis)[i];
}
__device__ __forceinline__ double tab_g(const KinTables& T, int i) {
  return reinterpret_cast<const double*>(T.blob + T.off_g)[i];
}
__device__ __forceinline__ int tab_rt_ptr(const KinTables& T, int j) {
  return reinterpret_cast<const int16_t*>(T.blob + T.off_rt_ptr)[j];
}
__device__ __forceinline__ uint32_t tab_rt(const KinTables& T, int p) {
  return reinterpret_cast<const uint32_t*>(T.blob + T.off_rt)[p];
}
__device__ __forceinline__ int tab_col_ptr(const KinTables& T, int j) {
  return reinterpret_cast<const int16_t*>(T.blob + T.off_col_ptr)[j];
}
__device__ __forceinline__ uint32_t tab_col(const KinTables& T, int p) {
  return reinterpret_cast<const uint32_t*>(T.blob + T.off_col)[p];
}
__device__ __forceinline__ int tab_row_ptr(const KinTables& T, int i) {
  return reinterpret_cast<const int16_t*>(T.blob + T.off_row_ptr)[i];
}
__device__ __forceinline__ uint32_t tab_row(const KinTables& T, int p) {
  return reinterpret_cast<const uint32_t*>(T.blob + T.off_row)[p];
}
__device__ __forceinline__ uint64_t tab_rdesc(const KinTables& T, int j) {
  return reinterpret_cast<const uint64_t*>(T.blob + T.off_rdesc)[j];
}
__device__ __forceinline__ int tab_dep_ptr(const KinTables& T, int j) {
  return reinterpret_cast<const int16_t*>(T.blob + T.off_dep_ptr)[j];
}
__device__ __forceinline__ int tab_dep(const KinTables& T, int p) {
  return reinterpret_cast<const uint16_t*>(T.blob + T.off_dep)[p];
}
__device__ __forceinline__ double tab_grid(const KinTables& T, const KinSweepDev& S, int g) {
  return T.off_grid ? reinterpret_cast<const double*>(T.blob + T.off_grid)[g] : __ldg(S.grid + g);
}

// ---- seeds (rng.cpp:18-23; ensemble.hpp:15-18) -------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64_mix(uint64_t v) {
  uint64_t z = v + kPhi64;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t derive_run_seed(uint64_t master, uint64_t i) {
  return splitmix64_mix(master + i * kPhi64);
}

// Global simulation index of launch-local simulation s (kin_tables.h
// KinSweepDev: contiguous or interleaved parts).
__device__ __forceinline__ uint64_t global_sim(const KinSweepDev& S, uint64_t s) {
  const uint64_t l = S.local_begin + s;
  if (S.pt_stride == 0) return S.sim_begin + l;
  const uint64_t k = l / S.runs;
  return (S.pt_first + k * S.pt_stride) * S.runs + (l - k * S.runs);
}

// Seed of global simulation `sim` (kin_abi.h enum kin_seed_mode).
__device__ __forceinline__ uint64_t sim_seed(const KinSweepDev& S, uint64_t sim) {
  if (S.seed_mode == 1) return derive_run_seed(S.master_seed, sim);
  if (S.seed_mode == 2) return sim == 0 ? S.master_seed : derive_run_seed(S.master_seed, sim);
  const uint64_t point = sim / S.runs, run = sim - point * S.runs;
  return derive_run_seed(derive_run_seed(S.master_seed, point), run);
}

// Sweep coordinates of global simulation `sim` (Cartesian points, last axis
// fastest, R runs per point: SPEC.md:438-446) into av[ax * stride].  Out of
// line: the 64-bit divisions are long instruction sequences, and this runs
// once per simulation.
static __device__ __noinline__ void decode_point(const KinSweepDev& S, uint64_t sim, double* av, int stride) {
  uint64_t rem = sim / S.runs;
  for (int ax = S.n_axes - 1; ax >= 0; --ax) {
    const uint64_t nv = static_cast<uint64_t>(S.axis_n[ax]);
    const uint64_t q = rem / nv;
    av[ax * stride] = __ldg(S.axis_values[ax] + (rem - q * nv));
    rem = q;
  }
}

// ---- xoshiro256++ stream (rng.cpp:25-52) ------------------------------------
// With a one-value lookahead: `nx` already holds the next output, so a draw
// hands it out at once and the state advance (a serial chain of 64-bit integer
// operations) overlaps the arithmetic that consumes the value.  Same outputs
// in the same order as rng.cpp; the cost is one extra step per stream.
struct Xoshiro {
  uint64_t s0, s1, s2, s3;
  uint64_t nx;

  __device__ __forceinline__ void seed(uint64_t seed) {
    s0 = splitmix64_mix(seed);
    s1 = splitmix64_mix(seed + kPhi64);
    s2 = splitmix64_mix(seed + 2 * kPhi64);
    s3 = splitmix64_mix(seed + 3 * kPhi64);
    if ((s0 | s1 | s2 | s3) == 0) s0 = kPhi64;
    nx = step();
  }
  __device__ __forceinline__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ __forceinline__ uint64_t step() {
    const uint64_t out = rotl(s0 + s3, 23) + s0;
    const uint64_t sh = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= sh;
    s3 = rotl(s3, 45);
    return out;
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t out = nx;
    nx = step();
    return out;
  }
  // ((x >> 11) + 0.5) * 2^-53: exact in double, identical on every platform.
  __device__ __forceinline__ double uniform() { return uniform_from_bits(bits53()); }
  __device__ __forceinline__ uint64_t bits53() { return next() >> 11; }
  __device__ __forceinline__ static double uniform_from_bits(uint64_t b) {
    return __dmul_rn(__dadd_rn(static_cast<double>(b), 0.5), 0x1.0p-53);
  }
};

// ---- Philox4x32-10 counter-based stream (KIN_RNG_PHILOX), mirrors
// oracle/kin_rng.hpp Philox/PhiloxSite: key = run seed, a draw site is
// (event index, slot), uniforms come from consecutive 128-bit blocks.
__device__ __forceinline__ void philox_block(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                                             uint32_t c3, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}
constexpr uint32_t kPhiloxSsaSite = 0xFFFFFFFFu;
struct PhiloxSite {
  uint32_t k0, k1, slot, ev_lo, ev_hi, blk;
  int half;
  uint32_t buf[4];
  __device__ __forceinline__ PhiloxSite(uint64_t seed, uint64_t event, uint32_t site)
      : k0(static_cast<uint32_t>(seed)), k1(static_cast<uint32_t>(seed >> 32)), slot(site),
        ev_lo(static_cast<uint32_t>(event)), ev_hi(static_cast<uint32_t>(event >> 32)), blk(0), half(0) {}
  __device__ __forceinline__ uint64_t bits53() {
    if (half == 0) philox_block(k0, k1, slot, ev_lo, ev_hi, blk, buf);
    const uint64_t x = half == 0 ? (static_cast<uint64_t>(buf[1]) << 32 | buf[0])
                                 : (static_cast<uint64_t>(buf[3]) << 32 | buf[2]);
    if (half == 1) ++blk;
    half ^= 1;
    return x >> 11;
  }
  __device__ __forceinline__ static double uniform_from_bits(uint64_t b) {
    return __dmul_rn(__dadd_rn(static_cast<double>(b), 0.5), 0x1.0p-53);
  }
  __device__ __forceinline__ double uniform() { return uniform_from_bits(bits53()); }
};

// mean / k, correctly rounded.  Division by a power of two is exact scaling, so
// mean*2^-j is bit-identical to mean/2^j; only other k need the IEEE divide.
__device__ __forceinline__ double div_small(double mean, int k) {
  switch (k) {
    case 1: return mean;
    case 2: return __dmul_rn(mean, 0.5);
    case 4: return __dmul_rn(mean, 0.25);
    case 8: return __dmul_rn(mean, 0.125);
    default: return __ddiv_rn(mean, static_cast<double>(k));
  }
}

// draw_poisson (rng.cpp:68-109): inversion below mean 10, Hormann PTRS above.
// `flops` receives the algorithmic op count (same accounting as the oracle).
// correctly rounded float reciprocals 1/k, k = 1..40 (index 0 unused, 41 a pad)
__device__ __constant__ float c_rcp40[42] = {
    0.0f, 1.0f / 1, 1.0f / 2, 1.0f / 3, 1.0f / 4, 1.0f / 5, 1.0f / 6, 1.0f / 7, 1.0f / 8, 1.0f / 9, 1.0f / 10,
    1.0f / 11, 1.0f / 12, 1.0f / 13, 1.0f / 14, 1.0f / 15, 1.0f / 16, 1.0f / 17, 1.0f / 18, 1.0f / 19, 1.0f / 20,
    1.0f / 21, 1.0f / 22, 1.0f / 23, 1.0f / 24, 1.0f / 25, 1.0f / 26, 1.0f / 27, 1.0f / 28, 1.0f / 29, 1.0f / 30,
    1.0f / 31, 1.0f / 32, 1.0f / 33, 1.0f / 34, 1.0f / 35, 1.0f / 36, 1.0f / 37, 1.0f / 38, 1.0f / 39, 1.0f / 40,
    0.0f};

// lgamma(z) for z >= KIN_LGAMMA_N + 1 by the Stirling series (terms to z^-7;
// truncation < 1e-25 there, i.e. within an ulp like libm's lgamma) — far
// smaller code than the general-purpose lgamma.
__device__ __forceinline__ double lgamma_stirling(double z) {
  const double r = 1.0 / z, r2 = r * r;
  const double series = r * (1.0 / 12.0 - r2 * (1.0 / 360.0 - r2 * (1.0 / 1260.0 - r2 * (1.0 / 1680.0))));
  return (z - 0.5) * log(z) - z + 0.91893853320467274178 + series;
}

// lgamma(k+1), k < KIN_LGAMMA_N, computed by the host's glibc (the oracle's libm)
// and uploaded once per context (see kin_engine.cpp).
#define KIN_LGAMMA_N 4096
template <bool kCount, class Rng>
__device__ __forceinline__ uint64_t poisson(Rng& rng, double mean, uint64_t& flops, const double* lgamma_tab) {
  if (!(mean > 0.0)) return 0;
  if (mean < 10.0) {
    const uint64_t ub = rng.bits53();  // u = ((ub + 0.5) * 2^-53), formed in double only if needed
    // Fast decision path (returns exactly the k of the reference algorithm):
    // search an approximate CDF c'_k in FP32.  Error budget relative to the
    // reference's c_k (whose own rounding, (k+2)*2^-52, is negligible):
    //   p'_0 = __expf(-float(mean)): <= 13 float ulp (1.55e-6) + mean*2^-24
    //          (<= 6e-7) = 2.15e-6 for mean in (0,10);
    //   each recursion step p' *= float(mean)*rcp(k): 4 roundings, <= 2.4e-7;
    //   each cumulative add: <= 6e-8;  u' = fma(float(ub), 2^-53, 2^-54) in FP32
    //   (the 53 bits rounded to 24, one FMA rounding): <= 1.2e-7 relative to u.
    // So |c'_k - c_k| <= (2.25e-6 + 3e-7*k) c_k <= 1.43e-5 c_k for k <= 40, and a
    // guard G = 4e-5 (> 2x that) makes "u < c'_k(1-G) and u > c'_{k-1}(1+G)"
    // imply the reference stops at exactly k.  Otherwise (probability ~1e-4 per
    // draw) run the exact algorithm below.
    {
      constexpr float G = 4e-5f;
      const float uf = __fmaf_rn(__ull2float_rn(ub), 0x1p-53f, 0x1p-54f);
      const float mf = static_cast<float>(mean);
      float pf = __expf(-mf);
      float cf = pf, cprev = 0.0f;
      int kk = 0;
      // Two terms per trip (the same float operations as one per trip): the
      // second term's multiply and add overlap the first one's test, halving
      // the loop's branch + dependent-compare chain.  c_rcp40[41] is a pad.
      while (uf > cf * (1.0f + G) && kk < 40) {
        const float p1 = pf * (mf * c_rcp40[kk + 1]);
        const float p2 = p1 * (mf * c_rcp40[kk + 2]);
        const float c1 = cf + p1;
        const float c2 = c1 + p2;
        if (!(uf > c1 * (1.0f + G)) || kk + 1 >= 40) {
          kk += 1;
          pf = p1;
          cprev = cf;
          cf = c1;
          break;
        }
        kk += 2;
        pf = p2;
        cprev = c1;
        cf = c2;
      }
      if (kk < 40 && uf < cf * (1.0f - G) && (kk == 0 || uf > cprev * (1.0f + G))) {
        if (kCount) flops += 3 + 3 * static_cast<uint64_t>(kk);
        return static_cast<uint64_t>(kk);
      }
    }
    const double u = Rng::uniform_from_bits(ub);
    double p = exp(-mean);
    double c = p;
    uint64_t k = 0;
    while (u > c && k < 256) {
      ++k;
      p = __dmul_rn(p, div_small(mean, static_cast<int>(k)));
      c = __dadd_rn(c, p);
    }
    if (kCount) flops += 3 + 3 * k;
    return k;
  }
  const double lm = log(mean);
  const double b = __dadd_rn(0.931, __dmul_rn(2.53, sqrt(mean)));
  const double a = __dadd_rn(-0.059, __dmul_rn(0.02483, b));
  const double inv_alpha = __dadd_rn(1.1239, __ddiv_rn(1.1328, __dsub_rn(b, 3.4)));
  const double v_r = __dsub_rn(0.9277, __ddiv_rn(3.6224, __dsub_rn(b, 2.0)));
  if (kCount) flops += 12;
  for (;;) {
    const double u = __dsub_rn(rng.uniform(), 0.5);
    const double v = rng.uniform();
    const double us = __dsub_rn(0.5, fabs(u));
    const double kf = floor(__dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(__ddiv_rn(__dmul_rn(2.0, a), us), b), u), mean), 0.43));
    if (kCount) flops += 12;
    if (kf < 0.0) continue;
    if (us >= 0.07 && v <= v_r) return static_cast<uint64_t>(kf);
    if (us < 0.013 && v > us) continue;
    const double arg = __ddiv_rn(__dmul_rn(v, inv_alpha), __dadd_rn(__ddiv_rn(a, __dmul_rn(us, us)), b));
    // lgamma(kf+1): glibc's own values (host table) for kf < KIN_LGAMMA_N
    const double lg = kf < static_cast<double>(KIN_LGAMMA_N) ? __ldg(lgamma_tab + static_cast<int>(kf))
                                                             : lgamma_stirling(__dadd_rn(kf, 1.0));
    const double rhs = __dsub_rn(__dadd_rn(-mean, __dmul_rn(kf, lm)), lg);
    if (kCount) flops += 11;
    // Fast decision on lhs = log(arg): __logf errs by <= 2^-21.41 absolute on
    // [0.5,2] and <= 3 ulp elsewhere, float rounding of arg adds <= 6e-8; a
    // guard of 1e-4*max(1,|lhs|) (> 100x that) decides lhs <= rhs exactly
    // unless lhs is within the guard of rhs, where the double log is used.
    const float lf = __logf(static_cast<float>(arg));
    const double lfa = static_cast<double>(lf);
    const double guard = 1e-4 * fmax(1.0, fabs(lfa));
    if (isfinite(lfa) && lfa + guard < rhs) return static_cast<uint64_t>(kf);
    if (isfinite(lfa) && lfa - guard > rhs) continue;
    const double lhs = log(arg);
    if (lhs <= rhs) return static_cast<uint64_t>(kf);
  }
}

// ---- Binomial(n, p) (KIN_FIRING_BINOMIAL): BINV inversion when
// n*min(p,1-p) < 10, Hormann's BTRD otherwise; p > 1/2 draws n - Bin(n, 1-p).
// Mirrors oracle/kin_rng.hpp binomial_from operation for operation (this code
// is compiled with -fmad=false and uses the portable log/exp), so every draw
// and its flop count are bit-identical to the oracle's.
__device__ __forceinline__ double binom_fc(double k) {
  if (k < 10.0) {
    switch (static_cast<int>(k)) {
      case 0: return 0.08106146679532726;
      case 1: return 0.04134069595540929;
      case 2: return 0.02767792568499834;
      case 3: return 0.02079067210376509;
      case 4: return 0.01664469118982119;
      case 5: return 0.01387612882307075;
      case 6: return 0.01189670994589177;
      case 7: return 0.01041126526197209;
      case 8: return 0.009255462182712733;
      default: return 0.008330563433362871;
    }
  }
  const double rk = 1.0 / (k + 1.0);
  const double rk2 = rk * rk;
  return (1.0 / 12.0 - (1.0 / 360.0 - rk2 / 1260.0) * rk2) * rk;
}

// BINV's exact CDF search (the guard-band fallback of the FP32 decision path
// in binomial() below, a few 1e-4 of the draws): out of line, so its portable
// log/exp stay out of the leap loop's instruction-cache working set.
static __device__ __noinline__ uint64_t binv_exact(double u, double q, double fn, uint64_t n) {
  const double s = q / (1.0 - q);
  const double a = (fn + 1.0) * s;
  double f = pmath::pm_exp(fn * pmath::pm_log(1.0 - q));
  double c = f;
  const uint64_t kmax = n < 255 ? n : 255;
  uint64_t k = 0;
  while (u > c && k < kmax) {
    ++k;
    f = f * (a / static_cast<double>(k) - s);
    c = c + f;
  }
  return k;
}

template <class Rng>
static __device__ __noinline__ uint64_t binomial_btrd(Rng& rng, double fn, double q, double np, uint64_t& fl) {
  using pmath::pm_log;
  const uint64_t n = static_cast<uint64_t>(fn);
  const double m = floor((fn + 1.0) * q);
  const double r = q / (1.0 - q);
  const double nr = (fn + 1.0) * r;
  const double npq = np * (1.0 - q);
  const double spq = sqrt(npq);
  const double b = 1.15 + 2.53 * spq;
  const double a = -0.0873 + 0.0248 * b + 0.01 * q;
  const double c = np + 0.5;
  const double alpha = (2.83 + 5.1 / b) * spq;
  const double vr = 0.92 - 4.2 / b;
  const double urvr = 0.86 * vr;
  fl += 22;
  for (;;) {
    double v = rng.uniform();
    double u;
    fl += 2;
    if (v <= urvr) {
      u = v / vr - 0.43;
      const double kf = floor((2.0 * a / (0.5 - fabs(u)) + b) * u + c);
      fl += 8;
      return kf < 0.0 ? 0 : (kf > fn ? n : static_cast<uint64_t>(kf));
    }
    if (v >= vr) {
      u = rng.uniform() - 0.5;
      fl += 3;
    } else {
      u = v / vr - 0.93;
      u = (u < 0.0 ? -0.5 : 0.5) - u;
      v = rng.uniform() * vr;
      fl += 6;
    }
    const double us = 0.5 - fabs(u);
    const double kf = floor((2.0 * a / us + b) * u + c);
    fl += 6;
    if (kf < 0.0 || kf > fn) continue;
    v = v * alpha / (a / (us * us) + b);
    const double km = fabs(kf - m);
    fl += 6;
    if (km <= 15.0) {
      double f = 1.0;
      if (m < kf) {
        double i = m;
        do {
          i = i + 1.0;
          f = f * (nr / i - r);
          fl += 4;
        } while (i != kf);
      } else if (m > kf) {
        double i = kf;
        do {
          i = i + 1.0;
          v = v * (nr / i - r);
          fl += 4;
        } while (i != m);
      }
      if (v <= f) return static_cast<uint64_t>(kf);
      continue;
    }
    v = pm_log(v);
    const double rho = (km / npq) * (((km / 3.0 + 0.625) * km + 1.0 / 6.0) / npq + 0.5);
    const double t = -km * km / (2.0 * npq);
    fl += 13;
    if (v < t - rho) return static_cast<uint64_t>(kf);
    if (v > t + rho) continue;
    const double nm = fn - m + 1.0;
    const double h = (m + 0.5) * pm_log((m + 1.0) / (r * nm)) + binom_fc(m) + binom_fc(fn - m);
    const double nk = fn - kf + 1.0;
    const double rhs = h + (fn + 1.0) * pm_log(nm / nk) + (kf + 0.5) * pm_log(nk * r / (kf + 1.0)) - binom_fc(kf) -
                       binom_fc(fn - kf);
    fl += 54;
    if (v <= rhs) return static_cast<uint64_t>(kf);
  }
}

template <bool kCount, class Rng>
__device__ __forceinline__ uint64_t binomial(Rng& rng, uint64_t n, double p, uint64_t& flops) {
  if (n == 0 || !(p > 0.0)) return 0;
  if (p >= 1.0) return n;
  const bool flip = p > 0.5;
  const double q = flip ? 1.0 - p : p;
  const double fn = static_cast<double>(n);
  const double np = fn * q;
  uint64_t fl = flip ? 2 : 1;
  uint64_t k = 0;
  if (np < 10.0) {  // BINV
    const uint64_t ub = rng.bits53();  // the one uniform, formed in double only if needed
    bool done = false;
    // Fast decision path (returns exactly the k of the algorithm below): the
    // CDF search in FP32.  Relative error of c'_k against the exact c_k:
    // f'_0 = __expf(n log1pf(-q)) <= 4e-6 (|n log(1-q)| < 14), each step
    // p' *= s (n+1-k) rcp(k) (no cancellation; n+1-k exact below 2^24) <= 5e-7,
    // each cumulative add 6e-8: <= 1.8e-5 for k <= 24, and u' from the 53 bits
    // <= 1.2e-7.  A guard G = 1e-4 (> 5x that) makes "u < c'_k (1-G) and
    // u > c'_{k-1} (1+G)" imply the exact search stops at k; otherwise (a few
    // 1e-4 of the draws, or n >= 2^24, or k > 24) the exact search runs.
    if (n < (1ull << 24)) {
      constexpr float G = 1e-4f;
      const float uf = __fmaf_rn(__ull2float_rn(ub), 0x1p-53f, 0x1p-54f);
      const float qf = static_cast<float>(q);
      const float sf = qf / (1.0f - qf);
      const float nf = static_cast<float>(n);
      float pf = __expf(nf * log1pf(-qf));
      float cf = pf, cprev = 0.0f;
      const int kcap = n < 24 ? static_cast<int>(n) : 24;
      int kk = 0;
      while (uf > cf * (1.0f + G) && kk < kcap) {
        ++kk;
        pf = pf * (sf * (nf + 1.0f - static_cast<float>(kk)) * c_rcp40[kk]);
        cprev = cf;
        cf = cf + pf;
      }
      if (kk < kcap && uf < cf * (1.0f - G) && (kk == 0 || uf > cprev * (1.0f + G))) {
        k = static_cast<uint64_t>(kk);
        fl += 10 + 4 * k;
        done = true;
      }
    }
    if (!done) {
      k = binv_exact(Rng::uniform_from_bits(ub), q, fn, n);
      fl += 10 + 4 * k;
    }
  } else {
    k = binomial_btrd(rng, fn, q, np, fl);
  }
  if (kCount) flops += fl;
  return flip ? n - k : k;
}

// x(x-1)(x-2)/6: out of line, so the runtime-stoichiometry propensity loops
// (inlined many times in the ODE/hybrid kernels) do not each carry a double
// division; the JIT's constant stoichiometries still fold it inline.
__device__ __forceinline__ double combinations3_inline(double x) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(x, __dsub_rn(x, 1.0)), __dsub_rn(x, 2.0)), 6.0);
}
static __device__ __noinline__ double combinations3(double x) { return combinations3_inline(x); }
// compile-time stoichiometry (the per-model JIT): everything inline
template <int kS>
__device__ __forceinline__ double combinations_c(double x) {
  double h;
  if constexpr (kS == 1) {
    h = x;
  } else if constexpr (kS == 2) {
    h = __dmul_rn(__dmul_rn(x, __dsub_rn(x, 1.0)), 0.5);
  } else if constexpr (kS == 3) {
    h = combinations3_inline(x);
  } else {
    return 1.0;
  }
  return h < 0.0 ? 0.0 : h;
}
// d h(x, kS) / dx as the LSODA Jacobian takes it (kin_lsoda_impl.cuh jac_row,
// the oracle's rre_jacobian): compile-time stoichiometry for the per-model JIT
template <int kS>
__device__ __forceinline__ double jac_dh(double x) {
  if constexpr (kS == 1) {
    return x < 0.0 ? 0.0 : 1.0;
  } else if constexpr (kS == 2) {
    return combinations_c<2>(x) > 0.0 ? __dsub_rn(x, 0.5) : 0.0;
  } else {
    return combinations_c<3>(x) > 0.0
               ? __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(3.0, x), 6.0), x), 2.0), 6.0)
               : 0.0;
  }
}

// combinations (model.hpp:145-149) + order-3 extension; clamp >= 0.
__device__ __forceinline__ double combinations(double x, int s) {
  double h;
  if (s == 1) {
    h = x;
  } else if (s == 2) {
    h = __dmul_rn(__dmul_rn(x, __dsub_rn(x, 1.0)), 0.5);  // == /2.0 exactly (power of two)
  } else if (s == 3) {
    h = combinations3(x);
  } else {
    return 1.0;
  }
  return h < 0.0 ? 0.0 : h;
}
__device__ __forceinline__ int combinations_flops(int s) { return s <= 1 ? 0 : (s == 2 ? 3 : 5); }

}  // namespace kin

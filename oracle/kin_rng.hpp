// oracle/kin_rng.hpp — TEST INFRASTRUCTURE ONLY (CPU oracle; never on the product path).
//
// Restatement of the reference RNG layer, proj/src/rng.cpp + proj/include/kinetics/rng.hpp:
//   splitmix64 finaliser ............ rng.cpp:18-23   (mix(0) = 0xE220A8397B1DCDAF, rng.hpp:10)
//   RngStream seeding ............... rng.cpp:25-36   (4 splitmix steps, all-zero guard)
//   xoshiro256++ next_u64 ........... rng.cpp:38-48
//   draw_uniform .................... rng.cpp:50-52   (((x>>11)+0.5)*2^-53, open interval)
//   draw_normal (Box-Muller+spare) .. rng.cpp:54-66
//   draw_poisson .................... rng.cpp:68-109  (inversion < 10, Hormann PTRS >= 10)
// Pinned against the reference itself: tests/test_oracle_rng.py compares this
// restatement with oracle/_ref/ (the reference rng.cpp compiled from
// /root/reference by oracle/Makefile) and with SURVEY Appendix A vectors.
//
// When KIN_ORACLE_REF_RNG is defined the oracle is built against the reference
// class kinetics::RngStream instead (oracle/_ref/libkin_oracle_refrng.so).
#pragma once

#include <cmath>
#include <cstdint>

#include "kin_portable_math.hpp"

#ifdef KIN_ORACLE_REF_RNG
#include "kinetics/rng.hpp"
#endif

namespace kin_oracle {

inline constexpr std::uint64_t kPhi64 = 0x9E3779B97F4A7C15ULL;

inline std::uint64_t splitmix64_mix(std::uint64_t v) {
  std::uint64_t z = v + kPhi64;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ensemble.hpp:15-18 / SPEC.md:411-419
inline std::uint64_t derive_run_seed(std::uint64_t master, std::uint64_t i) {
  return splitmix64_mix(master + i * kPhi64);
}

class Xoshiro256pp {
 public:
  explicit Xoshiro256pp(std::uint64_t seed) {
    // Seeding walks the splitmix64 sequence from `seed`; word w is mix(seed + w*phi)
    // (each step first advances the state by phi, then finalises it).
    for (int w = 0; w < 4; ++w) s_[w] = splitmix64_mix(seed + static_cast<std::uint64_t>(w) * kPhi64);
    if ((s_[0] | s_[1] | s_[2] | s_[3]) == 0) s_[0] = kPhi64;
  }

  std::uint64_t next_u64() {
    const std::uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
    const std::uint64_t sh = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= sh;
    s_[3] = rotl(s_[3], 45);
    return out;
  }

  double draw_uniform() {
    return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1.0p-53;
  }

  double draw_normal() {
    if (spare_valid_) {
      spare_valid_ = false;
      return spare_;
    }
    const double u1 = draw_uniform();
    const double u2 = draw_uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.141592653589793 * u2;  // 2*pi*u2, pi = std::numbers::pi
    spare_ = radius * std::sin(angle);
    spare_valid_ = true;
    return radius * std::cos(angle);
  }

  // Work-instrumented Poisson draw (rng.cpp:68-109); `flops` (may be null)
  // receives the algorithmic FP64 op count (FMA=2; + - * / sqrt exp log lgamma = 1).
  std::uint64_t draw_poisson(double mean, std::uint64_t* flops = nullptr);

 private:
  static std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  std::uint64_t s_[4];
  double spare_ = 0.0;
  bool spare_valid_ = false;
};

// draw_poisson's algorithm over any source of draw_uniform() values.
template <class Src>
std::uint64_t poisson_from(Src& src, double mean, std::uint64_t* flops) {
  if (mean <= 0.0) return 0;
  if (mean < 10.0) {
    const double u = src.draw_uniform();
    double p = std::exp(-mean);
    double c = p;
    std::uint64_t k = 0;
    while (u > c && k < 256) {
      ++k;
      p *= mean / static_cast<double>(k);
      c += p;
    }
    if (flops) *flops += 3 + 3 * k;
    return k;
  }
  const double lm = std::log(mean);
  const double b = 0.931 + 2.53 * std::sqrt(mean);
  const double a = -0.059 + 0.02483 * b;
  const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
  const double v_r = 0.9277 - 3.6224 / (b - 2.0);
  if (flops) *flops += 12;  // log, sqrt, 2 mul, 6 add/sub, 2 div
  for (;;) {
    const double u = src.draw_uniform() - 0.5;
    const double v = src.draw_uniform();
    const double us = 0.5 - std::fabs(u);
    const double kf = std::floor((2.0 * a / us + b) * u + mean + 0.43);
    if (flops) *flops += 12;  // 2 uniforms (4) + 8 arithmetic
    if (kf < 0.0) continue;
    if (us >= 0.07 && v <= v_r) return static_cast<std::uint64_t>(kf);
    if (us < 0.013 && v > us) continue;
    const double lhs = std::log(v * inv_alpha / (a / (us * us) + b));
    const double rhs = -mean + kf * lm - std::lgamma(kf + 1.0);
    if (flops) *flops += 11;
    if (lhs <= rhs) return static_cast<std::uint64_t>(kf);
  }
}

// ---- binomial draws (KIN_FIRING_BINOMIAL; no reference counterpart: the
// north star's "Poisson/binomial reaction firing").  Binomial(n, p) over any
// uniform source: BINV inversion (Kachitvichyanukul & Schmeiser 1988) when
// n*min(p,1-p) < 10, else Hormann's BTRD (1993); p > 1/2 draws n - Bin(n, 1-p).
// Only correctly rounded operations and the portable log/exp
// (kin_portable_math.hpp), so the CUDA sampler (kin_device.cuh binomial())
// reproduces every draw bit for bit.  Flop counting as draw_poisson's.
inline double binom_fc(double k) {  // Stirling correction of ln k! (Hormann 1993, table for k < 10)
  static constexpr double kTab[10] = {0.08106146679532726, 0.04134069595540929, 0.02767792568499834,
                                      0.02079067210376509, 0.01664469118982119, 0.01387612882307075,
                                      0.01189670994589177, 0.01041126526197209, 0.009255462182712733,
                                      0.008330563433362871};
  if (k < 10.0) return kTab[static_cast<int>(k)];
  const double rk = 1.0 / (k + 1.0);
  const double rk2 = rk * rk;
  return (1.0 / 12.0 - (1.0 / 360.0 - rk2 / 1260.0) * rk2) * rk;
}

template <class Src>
std::uint64_t binomial_from(Src& src, std::uint64_t n, double p, std::uint64_t* flops) {
  if (n == 0 || !(p > 0.0)) return 0;
  if (p >= 1.0) return n;
  const bool flip = p > 0.5;
  const double q = flip ? 1.0 - p : p;
  const double fn = static_cast<double>(n);
  const double np = fn * q;
  std::uint64_t fl = flip ? 2 : 1;
  std::uint64_t k = 0;
  if (np < 10.0) {  // BINV: one uniform, CDF search
    const double s = q / (1.0 - q);
    const double a = (fn + 1.0) * s;
    double f = pm_exp(fn * pm_log(1.0 - q));
    double c = f;
    const double u = src.draw_uniform();
    const std::uint64_t kmax = n < 255 ? n : 255;
    while (u > c && k < kmax) {
      ++k;
      f = f * (a / static_cast<double>(k) - s);
      c = c + f;
    }
    fl += 10 + 4 * k;
  } else {  // BTRD
    const double m = std::floor((fn + 1.0) * q);
    const double r = q / (1.0 - q);
    const double nr = (fn + 1.0) * r;
    const double npq = np * (1.0 - q);
    const double spq = std::sqrt(npq);
    const double b = 1.15 + 2.53 * spq;
    const double a = -0.0873 + 0.0248 * b + 0.01 * q;
    const double c = np + 0.5;
    const double alpha = (2.83 + 5.1 / b) * spq;
    const double vr = 0.92 - 4.2 / b;
    const double urvr = 0.86 * vr;
    fl += 22;
    for (;;) {
      double v = src.draw_uniform();
      double u;
      fl += 2;
      if (v <= urvr) {
        u = v / vr - 0.43;
        const double kf = std::floor((2.0 * a / (0.5 - std::fabs(u)) + b) * u + c);
        fl += 8;
        k = kf < 0.0 ? 0 : (kf > fn ? n : static_cast<std::uint64_t>(kf));
        break;
      }
      if (v >= vr) {
        u = src.draw_uniform() - 0.5;
        fl += 3;
      } else {
        u = v / vr - 0.93;
        u = (u < 0.0 ? -0.5 : 0.5) - u;
        v = src.draw_uniform() * vr;
        fl += 6;
      }
      const double us = 0.5 - std::fabs(u);
      const double kf = std::floor((2.0 * a / us + b) * u + c);
      fl += 6;
      if (kf < 0.0 || kf > fn) continue;
      v = v * alpha / (a / (us * us) + b);
      const double km = std::fabs(kf - m);
      fl += 6;
      if (km <= 15.0) {  // recursive f(k)/f(m)
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
        if (v <= f) { k = static_cast<std::uint64_t>(kf); break; }
        continue;
      }
      v = pm_log(v);  // squeeze, then the final acceptance test
      const double rho = (km / npq) * (((km / 3.0 + 0.625) * km + 1.0 / 6.0) / npq + 0.5);
      const double t = -km * km / (2.0 * npq);
      fl += 13;
      if (v < t - rho) { k = static_cast<std::uint64_t>(kf); break; }
      if (v > t + rho) continue;
      const double nm = fn - m + 1.0;
      const double h = (m + 0.5) * pm_log((m + 1.0) / (r * nm)) + binom_fc(m) + binom_fc(fn - m);
      const double nk = fn - kf + 1.0;
      const double rhs = h + (fn + 1.0) * pm_log(nm / nk) + (kf + 0.5) * pm_log(nk * r / (kf + 1.0)) -
                         binom_fc(kf) - binom_fc(fn - kf);
      fl += 54;
      if (v <= rhs) { k = static_cast<std::uint64_t>(kf); break; }
    }
  }
  if (flops) *flops += fl;
  return flip ? n - k : k;
}

inline std::uint64_t Xoshiro256pp::draw_poisson(double mean, std::uint64_t* flops) {
  return poisson_from(*this, mean, flops);
}

// ---- Philox4x32-10 counter-based stream (KIN_RNG_PHILOX; no reference
// counterpart: the north star's fast mode).  Salmon et al., SC'11.  Key =
// the run seed; a draw site is addressed by (event index, slot) and yields
// uniforms from consecutive 128-bit blocks (block b -> two 53-bit uniforms).
struct Philox {
  static void block(std::uint32_t k0, std::uint32_t k1, std::uint32_t c0, std::uint32_t c1, std::uint32_t c2,
                    std::uint32_t c3, std::uint32_t out[4]) {
    for (int r = 0; r < 10; ++r) {
      if (r > 0) {
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
      const std::uint64_t p0 = static_cast<std::uint64_t>(0xD2511F53u) * c0;
      const std::uint64_t p1 = static_cast<std::uint64_t>(0xCD9E8D57u) * c2;
      const std::uint32_t hi0 = static_cast<std::uint32_t>(p0 >> 32), lo0 = static_cast<std::uint32_t>(p0);
      const std::uint32_t hi1 = static_cast<std::uint32_t>(p1 >> 32), lo1 = static_cast<std::uint32_t>(p1);
      const std::uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
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
};

// Uniform source for one draw site: (seed, event, slot) -> blocks 0, 1, ...
struct PhiloxSite {
  std::uint32_t k0, k1, slot, ev_lo, ev_hi;
  std::uint32_t blk = 0;
  int half = 0;
  std::uint32_t buf[4];
  PhiloxSite(std::uint64_t seed, std::uint64_t event, std::uint32_t site)
      : k0(static_cast<std::uint32_t>(seed)), k1(static_cast<std::uint32_t>(seed >> 32)), slot(site),
        ev_lo(static_cast<std::uint32_t>(event)), ev_hi(static_cast<std::uint32_t>(event >> 32)) {}
  double draw_uniform() {
    if (half == 0) Philox::block(k0, k1, slot, ev_lo, ev_hi, blk, buf);
    const std::uint64_t x = half == 0 ? (static_cast<std::uint64_t>(buf[1]) << 32 | buf[0])
                                      : (static_cast<std::uint64_t>(buf[3]) << 32 | buf[2]);
    if (half == 1) ++blk;
    half ^= 1;
    return (static_cast<double>(x >> 11) + 0.5) * 0x1.0p-53;
  }
};
constexpr std::uint32_t kPhiloxSsaSite = 0xFFFFFFFFu;

#ifdef KIN_ORACLE_REF_RNG
// The reference stream itself (proj/src/rng.cpp compiled from /root/reference).
// Work counting is not available through the reference class.
class RefStream {
 public:
  explicit RefStream(std::uint64_t seed) : r_(seed) {}
  std::uint64_t next_u64() { return r_.next_u64(); }
  double draw_uniform() { return r_.draw_uniform(); }
  double draw_normal() { return r_.draw_normal(); }
  std::uint64_t draw_poisson(double mean, std::uint64_t* = nullptr) { return r_.draw_poisson(mean); }

 private:
  kinetics::RngStream r_;
};
using Stream = RefStream;
#else
using Stream = Xoshiro256pp;
#endif

}  // namespace kin_oracle

// kin_hybrid_impl.cuh — hybrid PDMP sweep kernel (hybrid.hpp:14-62).
//
// One thread per simulation, persistent warps.  Mirrors oracle/kin_oracle.cpp
// simulate_hybrid / hybrid_segment operation for operation (compiled with
// -fmad=false; step control and the jump threshold E = -ln u use the portable
// log/pow of kin_pmath.cuh), so trajectories are bit-identical to the oracle's:
//   per segment: partition_reactions (slow iff a_j < theta_a or a reactant
//   amount < theta_x), horizon min(t + repartition_interval, t_end), E = -ln u;
//   Dormand-Prince 5(4) on (x, G) with dx/dt = sum_fast nu_j a_j (row order)
//   and dG/dt = sum_slow a_j; where G reaches E, bisection on the dense output
//   to 1e-10 relative in t; the firing slow reaction by the ssa_select rule
//   over the slow set; nu_j added to the continuous state, clamped at 0.
// Per-simulation state: 8 vectors of N+1 doubles (y, k1..k6, ys), a[M], the
// sweep coordinates and a slow-set bitmask, in shared memory with the
// [slot][thread] layout (conflict-free; lanes touch consecutive words).  k7
// reuses k2's slot and yn reuses ys's (a72 = e2 = d2 = 0: k2 is dead once
// stage 6 is formed, ys once yn is); the dense-output coefficients r1..r5 are
// formed on demand from y, yn, k1, k3..k7 with the oracle's expressions, so
// they round identically.  The six stages run as one loop (each stage's input
// straight-line behind a warp-uniform switch) so the RHS (propensities +
// fast/slow sums) is inlined once, not six times (instruction-cache footprint).
#pragma once
#ifndef __CUDACC_RTC__
#include "kin_launch.h"
#endif
#include "kin_stochastic_impl.cuh"  // (first: it brings the fixed-width types NVRTC lacks)
#include "kin_pmath.cuh"

namespace kin {
namespace hyb {


using pmath::pm_log;
using pmath::pm_pow;
// x^y out of line (three sites in the step loop; each inlined copy is ~100
// instructions of the kernel's instruction-cache working set).  Same operations.
static __device__ __noinline__ double pm_pow_out(double x, double y) { return pm_pow(x, y); }
constexpr int kBlock = 32;  // one warp per block: the per-thread state is large
using stoch::TableModel;

// Dormand-Prince 5(4) tableau (the oracle's dp:: constants)
constexpr double c_a21 = 1.0 / 5.0;
constexpr double c_a31 = 3.0 / 40.0, c_a32 = 9.0 / 40.0;
constexpr double c_a41 = 44.0 / 45.0, c_a42 = -56.0 / 15.0, c_a43 = 32.0 / 9.0;
constexpr double c_a51 = 19372.0 / 6561.0, c_a52 = -25360.0 / 2187.0, c_a53 = 64448.0 / 6561.0, c_a54 = -212.0 / 729.0;
constexpr double c_a61 = 9017.0 / 3168.0, c_a62 = -355.0 / 33.0, c_a63 = 46732.0 / 5247.0, c_a64 = 49.0 / 176.0,
                 c_a65 = -5103.0 / 18656.0;
constexpr double c_a71 = 35.0 / 384.0, c_a73 = 500.0 / 1113.0, c_a74 = 125.0 / 192.0, c_a75 = -2187.0 / 6784.0,
                 c_a76 = 11.0 / 84.0;
constexpr double c_e1 = 71.0 / 57600.0, c_e3 = -71.0 / 16695.0, c_e4 = 71.0 / 1920.0, c_e5 = -17253.0 / 339200.0,
                 c_e6 = 22.0 / 525.0, c_e7 = -1.0 / 40.0;
constexpr double c_d1 = -12715105075.0 / 11282082432.0, c_d3 = 87487479700.0 / 32700410799.0,
                 c_d4 = -10690763975.0 / 1880347072.0, c_d5 = 701980252875.0 / 199316789632.0,
                 c_d6 = -1453857185.0 / 822651844.0, c_d7 = 69997945.0 / 29380423.0;
constexpr double kSafe = 0.9, kFacMinInv = 5.0, kFacMaxInv = 0.1;
constexpr double kBeta = 0.04, kExpo1 = 0.2 - kBeta * 0.75;
constexpr int kVecs = 8;
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min

// kN > 0: species count fixed at compile time (small models: loops over the
// N+1 components unroll); kN = 0: runtime T.n.
// PM: the propensity / row-sum policy — TableModel (walks the packed tables)
// or the per-model JIT's GenModel<double> (straight-line code, kin_jit.cpp):
// the same operations in the same order either way.
template <bool kCount, int kN, class PM>
struct Hybrid {
  const KinTables& T;
  const KinSweepDev& S;
  PM sm;  // propensities over y (x = y[0..n-1])
  int n_rt, m, n1_rt;
  __device__ __forceinline__ int N() const { return kN > 0 ? kN : n_rt; }
  __device__ __forceinline__ int N1() const { return kN > 0 ? kN + 1 : n1_rt; }
  double* V;         // kVecs vectors of N1(), [vec][comp][thread]
  uint32_t* slowm;   // [word][thread]
  uint64_t flops = 0;

  __device__ __forceinline__ double& v(int vec, int i) const { return V[(static_cast<size_t>(vec) * N1() + i) * kBlock]; }
  __device__ __forceinline__ double* vp(int vec) const { return V + static_cast<size_t>(vec) * N1() * kBlock; }
  __device__ __forceinline__ bool slow(int j) const { return (slowm[(j >> 5) * kBlock] >> (j & 31)) & 1u; }

  // augmented RHS: f = (sum_fast nu a (row order), sum_slow a) at state `yv`
  __device__ void rhs(int yv, int fv) {
    PM st{T, vp(yv), sm.a, sm.av};
    st.props_only();
    if (kCount) flops += static_cast<uint64_t>(T.fprop) + 2 * static_cast<uint64_t>(T.nnz) + static_cast<uint64_t>(m);
    st.hyb_rows(slowm, vp(fv), N());
  }

};

enum { Y = 0, K1, K2, K3, K4, K5, K6, YS, K7 = K2, YN = YS };

// Stage ST's input y + h * sum_k a_{ST+2,k+1} k_{k+1} as straight-line code
// (coefficients folded, the zero a72 skipped), summed left to right like the
// oracle; one instantiation per stage behind a warp-uniform switch, so the
// RHS call after it stays a single site.
__host__ __device__ constexpr double stage_coef(int st, int k) {
  return st == 0 ? c_a21
       : st == 1 ? (k == 0 ? c_a31 : c_a32)
       : st == 2 ? (k == 0 ? c_a41 : k == 1 ? c_a42 : c_a43)
       : st == 3 ? (k == 0 ? c_a51 : k == 1 ? c_a52 : k == 2 ? c_a53 : c_a54)
       : st == 4 ? (k == 0 ? c_a61 : k == 1 ? c_a62 : k == 2 ? c_a63 : k == 3 ? c_a64 : c_a65)
                 : (k == 0 ? c_a71 : k == 1 ? 0.0 : k == 2 ? c_a73 : k == 3 ? c_a74 : k == 4 ? c_a75 : c_a76);
}
template <int ST, int K>
__device__ __forceinline__ double stage_sum(double acc, double kv0, double kv1, double kv2, double kv3, double kv4) {
  if constexpr (K > ST) {
    return acc;
  } else if constexpr (ST == 5 && K == 1) {  // a72 = 0: not a term of the oracle's sum
    return stage_sum<ST, K + 1>(acc, kv0, kv1, kv2, kv3, kv4);
  } else {
    constexpr double c = stage_coef(ST, K);
    const double kv = K == 1 ? kv0 : K == 2 ? kv1 : K == 3 ? kv2 : K == 4 ? kv3 : kv4;  // k_{K+1}
    return stage_sum<ST, K + 1>(acc + c * kv, kv0, kv1, kv2, kv3, kv4);
  }
}
template <int ST, class HT>
__device__ __forceinline__ void stage_input(const HT& H, int n1, double hh) {
  for (int i = 0; i < n1; ++i) {
    constexpr double c0 = stage_coef(ST, 0);
    const double acc0 = c0 * H.v(K1, i);
    const double acc = stage_sum<ST, 1>(acc0, ST >= 1 ? H.v(K2, i) : 0.0, ST >= 2 ? H.v(K3, i) : 0.0,
                                        ST >= 3 ? H.v(K4, i) : 0.0, ST >= 4 ? H.v(K5, i) : 0.0,
                                        ST >= 5 ? H.v(K6, i) : 0.0);
    H.v(YS, i) = H.v(Y, i) + hh * acc;  // yn for ST = 5 (same slot)
  }
}

// Dense output of the accepted step for one component (the oracle's r1..r5).
struct Dense5 {
  double r1, r2, r3, r4, r5;
  template <class HT>
  __device__ __forceinline__ Dense5(const HT& H, int i, double hh) {
    r1 = H.v(Y, i);
    const double yd = H.v(YN, i) - H.v(Y, i);
    r2 = yd;
    const double bs = hh * H.v(K1, i) - yd;
    r3 = bs;
    r4 = yd - hh * H.v(K7, i) - bs;
    r5 = hh * (c_d1 * H.v(K1, i) + c_d3 * H.v(K3, i) + c_d4 * H.v(K4, i) + c_d5 * H.v(K5, i) + c_d6 * H.v(K6, i) +
               c_d7 * H.v(K7, i));
  }
  __device__ __forceinline__ double at(double th) const {
    const double th1 = 1.0 - th;
    return r1 + th * (r2 + th1 * (r3 + th * (r4 + th1 * r5)));
  }
};

template <bool kCount, bool kPhilox, int kN, class PM>
__device__ void simulate_hybrid_one(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, uint64_t s,
                                    double* V, double* a, double* av, uint32_t* slowm) {
  constexpr int B = kBlock;
  const uint64_t sim = global_sim(S, s);
  const int n = kN > 0 ? kN : T.n, m = T.m, G = T.n_grid, n1 = n + 1;
  Hybrid<kCount, kN, PM> H{T, S, PM{T, V, a, av}, T.n, m, T.n + 1, V, slowm};
  stoch::init_state<double, kBlock>(T, S, sim, n, V, av);  // y[0..n-1] = x0 (vector Y is the first)
  const uint64_t seed = sim_seed(S, sim);
  Xoshiro rng;
  if (!kPhilox) rng.seed(seed);
  const double t_end = S.t_end, rtol = S.rel_tol, atol = S.abs_tol;
  const double hmax = S.h_max > 0.0 ? S.h_max : KIN_INF;
  const double rep = S.hyb_rep > 0.0 ? S.hyb_rep : t_end / 100.0;
  uint64_t meta[6] = {0, 0, 0, 0, 0, 0};
  bool floored = false;
  int status = 0;
  double t = 0.0;
  int gi = 0;
  auto emit_state = [&]() {
    double* o = O.traj + (static_cast<size_t>(s) * G + gi) * n;
    for (int i = 0; i < n; ++i) o[i] = H.v(Y, i);
    ++gi;
  };
  while (gi < G && tab_grid(T, S, gi) <= t) emit_state();
  uint64_t attempts = 0, seg = 0;
  while (t < t_end) {
    // partition_reactions at the current state
    {
      TableModel<double, kBlock> st{T, V, a, av};
      const int words = (m + 31) >> 5;
      for (int w = 0; w < words; ++w) slowm[w * B] = 0u;
      for (int j = 0; j < m; ++j) {
        const double aj = st.prop(j);
        a[j * B] = aj;
        bool sl = aj < S.hyb_theta_a;
        const uint64_t d = tab_rdesc(T, j);
        const int nt = KIN_RD_NTERMS(d);
        for (int q = 0; q < nt; ++q) sl |= H.v(Y, KIN_RD_SPECIES(d, q)) < S.hyb_theta_x;
        if (sl) slowm[(j >> 5) * B] |= 1u << (j & 31);
      }
      if (kCount) H.flops += static_cast<uint64_t>(T.fprop);
    }
    const double t_hor = t + rep < t_end ? t + rep : t_end;
    PhiloxSite site(seed, seg, 0);
    const double u = kPhilox ? site.uniform() : rng.uniform();
    const double E = -pm_log(u);
    if (kCount) H.flops += 3;
    // ---- hybrid_segment ---------------------------------------------------
    bool jumped = false;
    {
      H.v(Y, n) = 0.0;
      H.rhs(Y, K1);
      double h;
      if (S.h_init > 0.0) {
        h = S.h_init;
      } else {
        double dnf = 0.0, dny = 0.0;
        for (int i = 0; i < n1; ++i) {
          const double sk = atol + rtol * fabs(H.v(Y, i));
          const double qf = H.v(K1, i) / sk, qy = H.v(Y, i) / sk;
          dnf = dnf + qf * qf;
          dny = dny + qy * qy;
        }
        h = (dnf <= 1e-10 || dny <= 1e-10) ? 1.0e-6 : sqrt(dny / dnf) * 0.01;
        if (h > hmax) h = hmax;
        for (int i = 0; i < n1; ++i) H.v(YS, i) = H.v(Y, i) + h * H.v(K1, i);
        H.rhs(YS, K2);
        double der2 = 0.0;
        for (int i = 0; i < n1; ++i) {
          const double sk = atol + rtol * fabs(H.v(Y, i));
          const double q = (H.v(K2, i) - H.v(K1, i)) / sk;
          der2 = der2 + q * q;
        }
        der2 = sqrt(der2) / h;
        const double der12 = dmax(der2, sqrt(dnf));
        const double h1 = der12 <= 1e-15 ? dmax(1.0e-6, h * 1.0e-3) : pm_pow_out(0.01 / der12, 0.2);
        h = dmin(100.0 * h, h1);
        if (h > hmax) h = hmax;
        if (kCount) H.flops += 15 * static_cast<uint64_t>(n1) + 12;
      }
      double facold = 1.0e-4;
      // pm_pow(facold, kBeta) = pm_exp(kBeta * pm_log(facold)): facold is the
      // last accepted err (>= 1e-4, where pm_pow's clamp is idle) or 1e-4, so
      // its log is the one already taken for that step's fac11 (or log 1e-4):
      // one log per step instead of two, the same values
      const double lfo_min = pm_log(1.0e-4);
      double lfo = lfo_min;
      bool last_rejected = false;
      while (t < t_hor) {
        if (attempts++ >= S.max_steps) { status = KIN_SIM_BUDGET; break; }
        double hh = h < hmax ? h : hmax;
        bool hit = false;
        if (t + hh >= t_hor) { hh = t_hor - t; hit = true; }
        if (!(hh > 0.0) || t + hh == t) { status = KIN_SIM_STEP_UNDERFLOW; break; }
#pragma unroll 1
        for (int st = 0; st < 6; ++st) {
          switch (st) {
            case 0: stage_input<0>(H, n1, hh); break;
            case 1: stage_input<1>(H, n1, hh); break;
            case 2: stage_input<2>(H, n1, hh); break;
            case 3: stage_input<3>(H, n1, hh); break;
            case 4: stage_input<4>(H, n1, hh); break;
            default: stage_input<5>(H, n1, hh); break;
          }
          H.rhs(YS, st == 5 ? K7 : K2 + st);
        }
        double sum = 0.0;
        bool finite = true;
        for (int i = 0; i < n1; ++i) {
          const double e = hh * (c_e1 * H.v(K1, i) + c_e3 * H.v(K3, i) + c_e4 * H.v(K4, i) + c_e5 * H.v(K5, i) +
                                 c_e6 * H.v(K6, i) + c_e7 * H.v(K7, i));
          const double sk = atol + rtol * dmax(fabs(H.v(Y, i)), fabs(H.v(YN, i)));
          const double q = e / sk;
          sum = sum + q * q;
          finite &= isfinite(H.v(YN, i));
        }
        const double err = sqrt(sum / static_cast<double>(n1));
        if (kCount) H.flops += 63 * static_cast<uint64_t>(n1) + 4;
        if (!finite || !isfinite(err)) { status = KIN_SIM_NONFINITE; break; }
        const double lerr = pm_log(err < 1e-300 ? 1e-300 : (err > 1e300 ? 1e300 : err));  // pm_pow's clamp
        const double fac11 = pmath::pm_exp(kExpo1 * lerr);
        if (err > 1.0) {
          h = hh / dmin(kFacMinInv, fac11 / kSafe);
          last_rejected = true;
          ++meta[1];
          if (kCount) H.flops += 3;
          continue;
        }
        double fac = fac11 / pmath::pm_exp(kBeta * lfo);
        fac = dmax(kFacMaxInv, dmin(kFacMinInv, fac / kSafe));
        double hnew = hh / fac;
        facold = dmax(err, 1.0e-4);
        lfo = facold == err ? lerr : lfo_min;
        if (last_rejected && hnew > hh) hnew = hh;
        last_rejected = false;
        h = hnew;
        ++meta[0];
        if (kCount) H.flops += 18 * static_cast<uint64_t>(n1) + 8;
        const double tprev = t;
        const double tnew = hit ? t_hor : t + hh;
        if (H.v(YN, n) >= E) {
          double lo = 0.0, hi = 1.0;
          const Dense5 dg(H, n, hh);
          for (int it = 0; it < 200; ++it) {
            const double tl = tprev + lo * hh, th = tprev + hi * hh;
            if (!(th - tl > 1e-10 * fabs(th))) break;
            const double mid = 0.5 * (lo + hi);
            if (dg.at(mid) >= E) hi = mid; else lo = mid;
            if (kCount) H.flops += 12;
          }
          const double ts = hi == 1.0 ? tnew : tprev + hi * hh;
          while (gi < G && tab_grid(T, S, gi) < ts) {
            double* o = O.traj + (static_cast<size_t>(s) * G + gi) * n;
            const double th = (tab_grid(T, S, gi) - tprev) / hh;
            for (int i = 0; i < n; ++i) {
              double vv = Dense5(H, i, hh).at(th);
              if (vv < 0.0) { vv = 0.0; floored = true; }
              o[i] = vv;
            }
            if (kCount) H.flops += 8 * static_cast<uint64_t>(n) + 3;
            ++gi;
          }
          for (int i = 0; i < n; ++i) {
            double vv = hi == 1.0 ? H.v(YN, i) : Dense5(H, i, hh).at(hi);
            if (vv < 0.0) { vv = 0.0; floored = true; }
            H.v(Y, i) = vv;
          }
          t = ts;
          jumped = true;
          break;
        }
        t = tnew;
        // grid samples inside the step (before y <- yn, k1 <- k7: the dense
        // output is formed from this step's vectors)
        while (gi < G && tab_grid(T, S, gi) <= t) {
          double* o = O.traj + (static_cast<size_t>(s) * G + gi) * n;
          if (tab_grid(T, S, gi) == t) {
            for (int i = 0; i < n; ++i) {
              double vv = H.v(YN, i);
              if (vv < 0.0) { vv = 0.0; floored = true; }
              o[i] = vv;
            }
          } else {
            const double th = (tab_grid(T, S, gi) - tprev) / hh;
            for (int i = 0; i < n; ++i) {
              double vv = Dense5(H, i, hh).at(th);
              if (vv < 0.0) { vv = 0.0; floored = true; }
              o[i] = vv;
            }
            if (kCount) H.flops += 8 * static_cast<uint64_t>(n) + 3;
          }
          ++gi;
        }
        for (int i = 0; i < n1; ++i) {
          H.v(Y, i) = H.v(YN, i);
          H.v(K1, i) = H.v(K7, i);
        }
        bool lifted = false;
        for (int i = 0; i < n; ++i)
          if (H.v(Y, i) < 0.0) { H.v(Y, i) = 0.0; lifted = true; }
        if (lifted) {
          floored = true;
          H.rhs(Y, K1);
        }
      }
    }
    if (status) break;
    if (jumped) {
      TableModel<double, kBlock> st{T, V, a, av};
      for (int j = 0; j < m; ++j) a[j * B] = st.prop(j);
      if (kCount) H.flops += static_cast<uint64_t>(T.fprop);
      double as = 0.0;
      for (int j = 0; j < m; ++j)
        if (H.slow(j)) as = as + a[j * B];
      const double u2 = kPhilox ? site.uniform() : rng.uniform();
      if (as > 0.0) {
        const double target = u2 * as;
        double c = 0.0;
        int sel = -1, last = -1;
        for (int j = 0; j < m; ++j) {
          if (!H.slow(j)) continue;
          if (a[j * B] > 0.0) last = j;
          c = c + a[j * B];
          if (c > target) { sel = j; break; }
        }
        if (sel < 0) sel = last;
        const int p1 = tab_col_ptr(T, sel + 1);
        for (int p = tab_col_ptr(T, sel); p < p1; ++p) {
          const uint32_t e = tab_col(T, p);
          double& vv = H.v(Y, KIN_NU_INDEX(e));
          vv = vv + static_cast<double>(KIN_NU_DELTA(e));
          if (vv < 0.0) { vv = 0.0; ++meta[2]; }
        }
        ++meta[4];
        if (kCount) H.flops += 2 * static_cast<uint64_t>(m) + 1;
      }
      while (gi < G && tab_grid(T, S, gi) <= t) emit_state();
    }
    ++seg;
  }
  while (gi < G) emit_state();
  meta[5] = floored ? 1 : 0;
  uint64_t* me = O.meta + s * 6;
  for (int q = 0; q < 6; ++q) me[q] = meta[q];
  O.status[s] = status;
  if (kCount && O.work) O.work[s] = H.flops;
}

// doubles of per-warp state (the bitmask words rounded up to whole doubles)
__host__ __device__ __forceinline__ size_t hybrid_warp_doubles(const KinTables& T, const KinSweepDev& S) {
  const size_t words = (static_cast<size_t>(T.m) + 31) / 32;
  return (static_cast<size_t>(kVecs) * (T.n + 1) + T.m + S.n_axes) * kBlock + (words * kBlock + 1) / 2;
}

template <bool kCount, bool kPhilox, bool kGlobal, int kN, class PM>
__device__ __forceinline__ void hybrid_body(const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                                            unsigned long long* __restrict__ next) {
  extern __shared__ double smem[];
  constexpr int B = kBlock;
  const int tid = threadIdx.x, lane = tid & 31;
  const int n1 = T.n + 1;
  // state in shared memory, or (kGlobal) in this block's region of global memory
  double* base = kGlobal ? S.gstate + static_cast<size_t>(blockIdx.x) * hybrid_warp_doubles(T, S) : smem;
  double* V = base + tid;
  double* a = base + static_cast<size_t>(kVecs) * n1 * B + tid;
  double* av = a + static_cast<size_t>(T.m) * B;
  uint32_t* slowm = reinterpret_cast<uint32_t*>(base + static_cast<size_t>(kVecs * n1 + T.m + S.n_axes) * B) + tid;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, static_cast<unsigned long long>(S.warp_lanes));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (base >= S.n_local) break;
    const uint64_t s = lane < S.warp_lanes ? base + lane : S.n_local;  // lanes >= warp_lanes idle
    if (s < S.n_local) simulate_hybrid_one<kCount, kPhilox, kN, PM>(T, S, O, s, V, a, av, slowm);
    __syncwarp();
  }
}

template <bool kCount, bool kPhilox, bool kGlobal, int kN>
__global__ void __launch_bounds__(kBlock) hybrid_kernel(const __grid_constant__ KinTables T,
                                                        const __grid_constant__ KinSweepDev S, KinOutDev O,
                                                        unsigned long long* __restrict__ next) {
  hybrid_body<kCount, kPhilox, kGlobal, kN, TableModel<double, kBlock>>(T, S, O, next);
}

#ifndef __CUDACC_RTC__


// Host launcher of one kernel variant (explicitly instantiated across several
// translation units so the size-specialised variants compile in parallel).
template <bool kCount, bool kPhilox, bool kGlobal, int kN>
cudaError_t launch_k(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, unsigned long long* counter,
                     size_t smem, cudaStream_t stream) {
  auto kern = hybrid_kernel<kCount, kPhilox, kGlobal, kN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  if (S.gstate && resident > S.gstate_warps) resident = S.gstate_warps;
  KinSweepDev SW = S;
  // uniform step work per simulation: full warps (fewer lanes measured 1.56x
  // slower); a sweep's variant may request another width (study / tests)
  SW.warp_lanes = S.warp_lanes > 0 ? S.warp_lanes : 32;
  const uint64_t warps = (S.n_local + SW.warp_lanes - 1) / SW.warp_lanes;
  const unsigned grid = static_cast<unsigned>(warps < resident ? warps : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  kern<<<grid, kBlock, smem, stream>>>(T, SW, O, counter);
  return cudaGetLastError();
}

#define KIN_HYB_SIG(kc, kp, kg, kn)                                                                           \
  cudaError_t launch_k<kc, kp, kg, kn>(const KinTables&, const KinSweepDev&, const KinOutDev&, unsigned long long*, \
                                       size_t, cudaStream_t)
#endif  // __CUDACC_RTC__

}  // namespace hyb
}  // namespace kin

// kin_stochastic_impl.cuh — the SSA / tau-leaping simulation body, templated on
// a MODEL POLICY (how propensities, select_tau and state updates walk the
// model): TableModel walks the packed constant-bank tables (any model);
// kin_jit.cpp generates a straight-line policy per model and compiles it with
// NVRTC.  Both execute the same floating-point operations in the same order,
// so both are bit-identical to the oracle (oracle/kin_oracle.cpp
// simulate_stochastic).  See kin_stochastic.cu for the design notes.
#pragma once
#include "kin_device.cuh"

namespace kin {
namespace stoch {

// +inf (NVRTC has no __builtin_huge_val / math_constants.h)
#define KIN_INF __longlong_as_double(0x7FF0000000000000LL)
// Threads per block: one warp, the finest shared-memory granularity (measured:
// 5-warp blocks, which fit 15 instead of 14 C4 warps per SM, ran 2.6% slower
// and leave no room for large models such as C5).
constexpr int kBlock = KIN_STOCH_BLOCK;


// One species' contribution to select_tau: bound = max(eps*x/g, 1), then
// tau = min(tau, bound/|mu|, bound^2/sigma2) (zero terms skipped).
// (eps*x)/g with g in {1,2,3}: /1 and /2 are exact scalings.  A quotient
// q = num/den can only lower tau if num <= tau*den (up to rounding): fl(tau*den)
// errs by <= 2^-53 relative, so num > fl(tau*den)*(1 + 2^-50) proves q > tau,
// hence fl(q) >= tau and the (exact, same-as-oracle) division can be skipped.
template <bool kCount>
__device__ __forceinline__ double tau_bound(double tau, double eps, double x, double g, double mu, double s2,
                                            uint64_t& flops) {
  const double ex = __dmul_rn(eps, x);
  double bound = g == 1.0 ? ex : (g == 2.0 ? __dmul_rn(ex, 0.5) : __ddiv_rn(ex, g));
  if (bound < 1.0) bound = 1.0;
  if (kCount) flops += 2;
  if (mu != 0.0) {
    const double amu = fabs(mu);
    if (!(bound > __dmul_rn(__dmul_rn(tau, amu), 1.0 + 0x1p-50))) {
      const double t1 = __ddiv_rn(bound, amu);
      if (t1 < tau) tau = t1;
    }
    if (kCount) flops += 1;
  }
  if (s2 != 0.0) {
    const double bb = __dmul_rn(bound, bound);
    if (!(bb > __dmul_rn(__dmul_rn(tau, s2), 1.0 + 0x1p-50))) {
      const double t2 = __ddiv_rn(bb, s2);
      if (t2 < tau) tau = t2;
    }
    if (kCount) flops += 2;
  }
  return tau;
}

// Amounts are exact integers.  XT = double (any magnitude below 2^53, the
// reference's SystemState) or int32_t (half the shared memory, so more resident
// simulations; an update leaving int32 range raises *ovf and the engine re-runs
// the launch with the double variant — results are identical either way).
template <class XT, int kB = kBlock>
struct TableModel {
  static constexpr bool kUniformSsa = false;
  static constexpr bool kFlatBurst = false;
  static constexpr int kBurstQuantum = 1;
  static constexpr int kM = 0;
  const KinTables& T;
  XT* x;             // x[i * B]
  double* a;         // a[j * B]
  const double* av;  // axis values av[ax * B]
  static constexpr int B = kB;

  __device__ __forceinline__ int n() const { return T.n; }
  __device__ __forceinline__ int m() const { return T.m; }

  __device__ __forceinline__ double xv(int i) const { return static_cast<double>(x[i * B]); }
  // a_j(x) = c_j * prod h(x_s, stoich_s)   (model.hpp:151-157)
  __device__ __forceinline__ double prop(int j) const {
    const uint64_t d = tab_rdesc(T, j);
    const int ax = KIN_RD_AXIS(d);
    double aj = ax < 0 ? tab_rate(T, j) : __dmul_rn(tab_rate(T, j), av[ax * B]);
    const int nt = KIN_RD_NTERMS(d);
    if (nt > 0) {
      aj = __dmul_rn(aj, combinations(xv(KIN_RD_SPECIES(d, 0)), KIN_RD_STOICH(d, 0)));
      if (nt > 1) {
        aj = __dmul_rn(aj, combinations(xv(KIN_RD_SPECIES(d, 1)), KIN_RD_STOICH(d, 1)));
        if (nt > 2) aj = __dmul_rn(aj, combinations(xv(KIN_RD_SPECIES(d, 2)), KIN_RD_STOICH(d, 2)));
      }
    }
    return aj;
  }
  // a_j as evaluated at the start of the decision (leaps update x in place,
  // so the propensities must be the cached ones)
  __device__ __forceinline__ double aval(int j) const { return a[j * B]; }
  // all propensities; returns a0 summed in reaction order (oracle order)
  __device__ __forceinline__ double all_props(int M) const {
    double a0 = 0.0;
    for (int j = 0; j < M; ++j) {
      const double aj = prop(j);
      a[j * B] = aj;
      a0 = __dadd_rn(a0, aj);
    }
    return a0;
  }
  __device__ __forceinline__ double sum_props(int M) const {
    double a0 = 0.0;
    for (int j = 0; j < M; ++j) a0 = __dadd_rn(a0, aval(j));
    return a0;
  }
  // hybrid PDMP (kin_hybrid_impl.cuh): a[] at x, without the sum
  __device__ __forceinline__ void props_only() const {
#pragma unroll 1
    for (int j = 0; j < T.m; ++j) a[j * B] = prop(j);
  }
  // hybrid PDMP: f_i = sum over the fast reactions of nu_ij a_j (row order),
  // f_N = sum over the slow ones of a_j (reaction order); slow(j) = bit j of
  // the per-lane mask words slowm[w * B]
  __device__ __forceinline__ void hyb_rows(const uint32_t* slowm, double* f, int n) const {
    auto slow = [&](int j) { return ((slowm[(j >> 5) * B] >> (j & 31)) & 1u) != 0u; };
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      const int p1 = tab_row_ptr(T, i + 1), p0 = tab_row_ptr(T, i);
#pragma unroll 1
      for (int p = p0; p < p1; ++p) {
        const uint32_t e = tab_row(T, p);
        const int j = KIN_NU_INDEX(e);
        const double t = acc + static_cast<double>(KIN_NU_DELTA(e)) * a[j * B];
        acc = slow(j) ? acc : t;  // a select, not a branch per entry (same value as the oracle's skip)
      }
      f[i * B] = acc;
    }
    double g = 0.0;
#pragma unroll 1
    for (int j = 0; j < T.m; ++j) {
      const double t = g + a[j * B];
      g = slow(j) ? t : g;
    }
    f[n * B] = g;
  }
  // x += nu[:, j] * k  (k signed: negative undoes a rejected leap)
  __device__ __forceinline__ void apply(int j, long long k, bool& ovf) const {
    const int p1 = tab_col_ptr(T, j + 1);
#pragma unroll 1
    for (int p = tab_col_ptr(T, j); p < p1; ++p) {
      const uint32_t e = tab_col(T, p);
      XT* xs = x + KIN_NU_INDEX(e) * B;
      if constexpr (sizeof(XT) == 8) {
        *xs = __dadd_rn(*xs, __dmul_rn(static_cast<double>(KIN_NU_DELTA(e)), static_cast<double>(k)));
      } else {
        const long long v = static_cast<long long>(*xs) + static_cast<long long>(KIN_NU_DELTA(e)) * k;
        ovf |= v > 2147483647LL || v < -2147483647LL;
        *xs = static_cast<XT>(v);
      }
    }
  }
  // one SSA event: x += nu[:, j]; returns true if an amount went negative
  __device__ __forceinline__ bool fire(int j, bool& ovf) const {
    bool neg = false;
    const int p1 = tab_col_ptr(T, j + 1);
#pragma unroll 1
    for (int p = tab_col_ptr(T, j); p < p1; ++p) {
      const uint32_t e = tab_col(T, p);
      XT* xs = x + KIN_NU_INDEX(e) * B;
      if constexpr (sizeof(XT) == 8) {
        const double v = __dadd_rn(*xs, static_cast<double>(KIN_NU_DELTA(e)));
        neg |= v < 0.0;
        *xs = v;
      } else {
        const long long v = static_cast<long long>(*xs) + KIN_NU_DELTA(e);
        ovf |= v > 2147483647LL;
        neg |= v < 0;
        *xs = static_cast<XT>(v);
      }
    }
    return neg;
  }
  // select_tau (stochastic.hpp:40-44), header form, on the cached a[]
  template <bool kCount>
  __device__ __forceinline__ double select_tau(double eps, uint64_t& flops) const {
    double tau = KIN_INF;
    const int N = T.n;
    for (int i = 0; i < N; ++i) {
      double mu = 0.0, s2 = 0.0;
      const int p1 = tab_row_ptr(T, i + 1);
      const int p0 = tab_row_ptr(T, i);
      for (int p = p0; p < p1; ++p) {
        const uint32_t e = tab_row(T, p);
        const int dl = KIN_NU_DELTA(e);
        const double aj = aval(KIN_NU_INDEX(e));
        mu = __dadd_rn(mu, __dmul_rn(static_cast<double>(dl), aj));
        s2 = __dadd_rn(s2, __dmul_rn(static_cast<double>(dl * dl), aj));
      }
      if (kCount) flops += 4 * static_cast<uint64_t>(p1 - p0);
      if (mu == 0.0 && s2 == 0.0) continue;
      tau = tau_bound<kCount>(tau, eps, xv(i), tab_g(T, i), mu, s2, flops);
    }
    return tau;
  }
  __device__ __forceinline__ void dep_update(int sel) const {
    const int q1 = tab_dep_ptr(T, sel + 1);
#pragma unroll 1
    for (int q = tab_dep_ptr(T, sel); q < q1; ++q) {
      const int k = tab_dep(T, q);
      a[k * B] = prop(k);
    }
  }
  __device__ __forceinline__ bool any_negative() const {
    bool neg = false;
    for (int i = 0; i < T.n; ++i) neg |= x[i * B] < static_cast<XT>(0);
    return neg;
  }
  __device__ __forceinline__ int col_len(int j) const { return tab_col_ptr(T, j + 1) - tab_col_ptr(T, j); }
};

// The simulation's sweep coordinates (Cartesian decode, last axis fastest,
// SPEC.md:441) into av[], and its initial amounts into x[]; returns true when
// an amount does not fit XT = int32.
// ssa_step_from_uniforms (stochastic.hpp:28-32): the waiting
// time ln(1/u1)/a0 and the first reaction whose cumulative propensity exceeds
// u2*a0 (the last one with a_j > 0 if rounding leaves none).  Shared by the
// kernels and the kin_device_unit seam.
__device__ __forceinline__ double ssa_dt(double u1, double a0) { return __ddiv_rn(log(__ddiv_rn(1.0, u1)), a0); }

template <class Model>
__device__ __forceinline__ int ssa_select(const Model& sm, int M, double a0, double u2) {
  const double target = __dmul_rn(u2, a0);
  if constexpr (Model::kUniformSsa) {
    // small models: every partial sum, predicated picks (no data-dependent exit)
    double c = 0.0;
    int sel = -1, last = -1;
#pragma unroll
    for (int j = 0; j < Model::kM; ++j) {
      const double aj = sm.aval(j);
      c = __dadd_rn(c, aj);
      if (sel < 0 && aj > 0.0) last = j;
      if (sel < 0 && c > target) sel = j;
    }
    return sel < 0 ? last : sel;
  }
  double c = 0.0;
  int sel = -1, last = -1, j = 0;
  if constexpr (Model::kM >= 64) {
    // large models (propensity cache in global memory): eight loads issued
    // together, then the same additions and tests in order — one memory
    // latency per eight reactions instead of per two (C5: the SSA selection
    // held ~9% of the stall samples on its loads)
    for (; j + 8 <= M; j += 8) {
      double a8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a8[u] = sm.aval(j + u);
      bool found = false;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double cn = __dadd_rn(c, a8[u]);
        if (!found) {
          if (a8[u] > 0.0) last = j + u;
          if (cn > target) {
            sel = j + u;
            found = true;
          } else {
            c = cn;
          }
        }
      }
      if (found) return sel;
    }
  }
  // two reactions per trip (same additions in the same order): both loads and
  // the second sum issue before the first test
  for (; j + 1 < M; j += 2) {
    const double a1 = sm.aval(j), a2 = sm.aval(j + 1);
    const double c1 = __dadd_rn(c, a1);
    const double c2 = __dadd_rn(c1, a2);
    if (a1 > 0.0) last = j;
    if (c1 > target) { sel = j; break; }
    if (a2 > 0.0) last = j + 1;
    if (c2 > target) { sel = j + 1; break; }
    c = c2;
  }
  if (sel < 0 && j < M) {
    const double aj = sm.aval(j);
    if (aj > 0.0) last = j;
    if (__dadd_rn(c, aj) > target) sel = j;
  }
  return sel < 0 ? last : sel;
}

// The firing law of a launch: a compile-time constant in the per-model JIT
// kernels (KFIRING_), the sweep's field in the table-driven kernel.
#ifdef KFIRING_
#define KIN_FIRING_OF(S) (KFIRING_)
#else
#define KIN_FIRING_OF(S) ((S).firing)
#endif

// One reaction of the sequential binomial leap (KIN_FIRING_BINOMIAL; oracle
// binomial_fire): k_j ~ Binomial(n_j, a_j tau / n_j) with n_j = min over
// reactants of floor(x_s / stoich_s) at the current amounts (the reactions
// before j in this leap already applied), Poisson(a_j tau) for a zero-order
// reaction.  Amounts never go negative, so the leap is never rejected.
template <bool kCount, class Model, class Rng>
__device__ __forceinline__ uint64_t binomial_fire(const KinTables& T, const Model& sm, int j, double mean, Rng& rng,
                                                  uint64_t& flops, const double* lgamma_tab) {
  const uint64_t d = tab_rdesc(T, j);
  const int nt = KIN_RD_NTERMS(d);
  if (nt == 0) return poisson<kCount>(rng, mean, flops, lgamma_tab);
  if (!(mean > 0.0)) return 0;
  double lim = KIN_INF;
  for (int t = 0; t < nt; ++t) {
    const double x = sm.xv(KIN_RD_SPECIES(d, t));
    const int st = KIN_RD_STOICH(d, t);
    // floor(x / st): x / 1 and x / 2 are exact scalings (= x, x * 0.5)
    const double v = st == 1 ? x : floor(st == 2 ? __dmul_rn(x, 0.5) : __ddiv_rn(x, 3.0));
    if (v < lim) lim = v;
  }
  if (kCount) flops += static_cast<uint64_t>(nt);
  if (!(lim > 0.0)) return 0;
  if (kCount) flops += 1;
  return binomial<kCount>(rng, static_cast<uint64_t>(lim), __ddiv_rn(mean, lim), flops);
}

template <class XT, int B = kBlock>
__device__ __forceinline__ bool init_state(const KinTables& T, const KinSweepDev& S, uint64_t sim, int N, XT* x,
                                           double* av) {
  decode_point(S, sim, av, B);
  bool ovf = false;
  for (int i = 0; i < N; ++i) {
    const int ax = tab_x0_axis(T, i);
    const double v = ax < 0 ? tab_x0(T, i) : av[ax * B];
    if (sizeof(XT) != 8) ovf |= v > 2147483647.0;
    x[i * B] = static_cast<XT>(v);
  }
  return ovf;
}

template <class Model, bool kCount, bool kPhilox, class XT>
__device__ __forceinline__ void simulate_one(const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                                             uint64_t s, XT* x, double* a, double* av, int* ovf_flag) {
  constexpr int B = kBlock;
  const uint64_t sim = global_sim(S, s);
  const Model sm{T, x, a, av};
  const int N = sm.n(), M = sm.m(), G = T.n_grid;

  bool ovf = init_state<XT>(T, S, sim, N, x, av);

  const uint64_t seed = sim_seed(S, sim);
  Xoshiro rng;
  if (!kPhilox) rng.seed(seed);
  uint64_t ev = 0;  // Philox event counter (leap attempts and SSA events)
  const int kind = S.kind;
  const double t_end = S.t_end;
  double t = 0.0;
  int gi = 0;
  uint64_t flops = 0, used = 0;
  uint64_t n_steps = 0, n_rej = 0, n_ssa = 0;
  int status = 0;
  const uint64_t budget = S.max_steps;
  const uint64_t F_prop = static_cast<uint64_t>(T.fprop);

  // time of grid point gi (+inf past the end).  Small models keep it in a
  // register (read once per grid point instead of twice per SSA event: C2
  // 51 -> 47 ms); for C4 the two extra registers cross the 128-register line
  // at which 14 warps per SM fit (4 per scheduler): 94 -> 156 ms.
  constexpr bool kTg = Model::kFlatBurst && Model::kUniformSsa;
  double tg = (kTg && G > 0) ? tab_grid(T, S, 0) : KIN_INF;
  auto next_grid = [&]() { return kTg ? tg : (gi < G ? tab_grid(T, S, gi) : KIN_INF); };
  auto emit = [&]() {
    double* o = O.traj + (static_cast<size_t>(s) * G + gi) * N;  // [sim][g][n]: one contiguous run per emit
    for (int i = 0; i < N; ++i) o[i] = sm.xv(i);
    ++gi;
    if (kTg) tg = gi < G ? tab_grid(T, S, gi) : KIN_INF;
  };

  while (next_grid() <= t) emit();
  bool a_valid = false;
  double a0 = 0.0;

  // Small models (Model::kFlatBurst): one flat loop, one step per trip — a
  // decision (then a leap, or the first event of an SSA burst) or the next
  // Model::kBurstQuantum events of a burst.  A burst nested inside the
  // decision loop holds every lane of the warp at the loop head until the
  // warp's longest burst ends: a lane that leapt advanced one leap per 100
  // events of its neighbours (C2: 73 -> 50 ms); one event per trip instead
  // makes a bursting lane pay a neighbour's whole leap per event.  A few
  // events per trip (a leap costs ~10 events) balances the two: C2 46.7 ms at
  // 1, 39.5 at 2, 36.5-37.0 at 4, 39.6 at 8, 44.0 at 16.  b: position in the
  // burst, -1 at a decision; it saturates at 100 (pure SSA never leaves its
  // burst).  Per-simulation results do not depend on the quantum.
  int b = -1;
  for (;;) {
    if (b < 0) {
      if (!(t < t_end) || ovf) break;
      if (++used > budget) { status = KIN_SIM_BUDGET; break; }
      if (!a_valid) a0 = sm.all_props(M);
      a_valid = false;
      if (kCount) flops += F_prop + M;
      if (a0 == 0.0) break;

      double tau = 0.0;
      bool burst = false;
      if (kind == 0) {
        burst = true;
      } else if (kind == 1) {
        tau = sm.template select_tau<kCount>(S.epsilon, flops);
        if (kCount) flops += 1;
        burst = tau < __ddiv_rn(10.0, a0);
      } else {
        tau = S.tau;
      }
      if (burst) {
        b = 0;
      } else {
        // Poisson leap truncated at the next grid time; reject -> halve
        const double t_stop = next_grid() < t_end ? next_grid() : t_end;
        bool hit = false;
        const double gap = __dsub_rn(t_stop, t);
        if (kCount) flops += 1;
        if (!(tau < gap)) { tau = gap; hit = true; }
        if (KIN_FIRING_OF(S) == KIN_FIRING_BINOMIAL) {
          // sequential binomial leap: one attempt, never rejected
#pragma unroll 1
          for (int j = 0; j < M; ++j) {
            uint64_t k, fl = 0;
            const double mean = __dmul_rn(sm.aval(j), tau);
            if (kPhilox) {
              PhiloxSite src(seed, ev, static_cast<uint32_t>(j));
              k = binomial_fire<kCount>(T, sm, j, mean, src, fl, S.lgamma_tab);
            } else {
              k = binomial_fire<kCount>(T, sm, j, mean, rng, fl, S.lgamma_tab);
            }
            if (kCount) flops += fl;
            if (k != 0) sm.apply(j, static_cast<long long>(k), ovf);
          }
          if (kCount) flops += static_cast<uint64_t>(M) + 2 * static_cast<uint64_t>(T.nnz);
          ++ev;
          if (ovf) break;
          if (hit) {
            t = t_stop;
          } else {
            t = __dadd_rn(t, tau);
            if (kCount) flops += 1;
          }
          ++n_steps;
          while (next_grid() <= t) emit();
          continue;
        }
        Xoshiro saved = rng, resume;
        // One Poisson call site (code size): pass 0 draws and applies; a rejected
        // attempt runs pass 1, which replays the same draws (the saved stream is
        // swapped into `rng`, or the same Philox counters) and subtracts them, then
        // resumes the stream where pass 0 left it and retries with tau/2.  The
        // streams are swapped by value so they stay in registers.
        long long sign = 1;
        for (;;) {
          // a_{j+1} is loaded while reaction j draws (global-memory state: hides
          // the load latency behind the Poisson draw)
          double a_next = sm.aval(0);
#pragma unroll 1
          for (int j = 0; j < M; ++j) {
            uint64_t k, fl = 0;
            const double aj = a_next;
            if (j + 1 < M) a_next = sm.aval(j + 1);
            const double mean = __dmul_rn(aj, tau);
            if (kPhilox) {
              PhiloxSite src(seed, ev, static_cast<uint32_t>(j));
              k = poisson<kCount>(src, mean, fl, S.lgamma_tab);
            } else {
              k = poisson<kCount>(rng, mean, fl, S.lgamma_tab);
            }
            if (kCount && sign > 0) flops += fl;
            if (k != 0) sm.apply(j, sign * static_cast<long long>(k), ovf);
          }
          if (sign < 0) {
            // undone: continue the stream with half the step
            sign = 1;
            ++ev;
            rng = resume;
            saved = rng;
            ++n_rej;
            tau = __dmul_rn(tau, 0.5);
            hit = false;
            if (kCount) flops += 1;
            continue;
          }
          if (kCount) flops += static_cast<uint64_t>(M) + 2 * static_cast<uint64_t>(T.nnz);
          if (ovf) break;
          if (!sm.any_negative()) {
            ++ev;
            break;
          }
          sign = -1;
          resume = rng;
          rng = saved;
        }
        if (ovf) break;
        if (hit) {
          t = t_stop;
        } else {
          t = __dadd_rn(t, tau);
          if (kCount) flops += 1;
        }
        ++n_steps;
        while (next_grid() <= t) emit();
        continue;
      }
    }
    // the burst's events: kBurstQuantum per trip of the outer loop (kFlat), or the whole
    // burst here (large models, whose rare bursts cost less than the extra
    // per-trip divergence of the flat form: C4 94 vs 103 ms)
    bool done = false;
    int quantum = 0;
    do {
      if (b > 0) {
        if (kind != 0 && b >= 100) { a_valid = true; b = -1; break; }
        if (++used > budget) { status = KIN_SIM_BUDGET; done = true; break; }
        if (kCount) flops += F_prop + M;
        if (a0 == 0.0) { done = true; break; }
      }
      double u1, u2;
      if (kPhilox) {
        PhiloxSite src(seed, ev++, kPhiloxSsaSite);
        u1 = src.uniform();
        u2 = src.uniform();
      } else {
        u1 = rng.uniform();
        u2 = rng.uniform();
      }
      const double dt = ssa_dt(u1, a0);
      const double tn = __dadd_rn(t, dt);
      if (kCount) flops += 8;
      if (tn > t_end) { t = t_end; done = true; break; }
      while (next_grid() < tn) emit();
      const int sel = ssa_select(sm, M, a0, u2);
      if (kCount) flops += 1 + static_cast<uint64_t>(sel + 1);
      if (sm.fire(sel, ovf)) { status = KIN_SIM_NEGATIVE; done = true; break; }
      if (ovf) { done = true; break; }
      if (kCount) flops += static_cast<uint64_t>(sm.col_len(sel));
      t = tn;
      if (kind == 0) ++n_steps; else ++n_ssa;
      while (next_grid() <= t) emit();
      // re-evaluate the propensities that changed, then a0 in oracle order
      // (small models: all of them, summed as they are produced — the same
      // values without the shared-memory round trip)
      if constexpr (Model::kUniformSsa) {
        a0 = sm.all_props(M);
      } else {
        sm.dep_update(sel);
        a0 = sm.sum_props(M);
      }
      if (b < 100) ++b;
    } while (!Model::kFlatBurst || ++quantum < Model::kBurstQuantum);
    if (done) break;
  }
  if (ovf) {
    status = KIN_SIM_INTERNAL_RETRY;
    atomicExch(ovf_flag, 1);
  }
  if (status == 0)
    while (gi < G) emit();

  uint64_t* me = O.meta + s * 6;
  me[0] = n_steps;
  me[1] = n_rej;
  me[2] = 0;
  me[3] = n_ssa;
  me[4] = 0;
  me[5] = 0;
  O.status[s] = status;
  if (kCount && O.work) O.work[s] = flops;
}

// doubles of per-warp global state: a[M] + av[axes] doubles and (unless the
// amounts live in shared memory) x[N] of XT, per lane
template <class XT, bool kSmemX = false>
__host__ __device__ __forceinline__ size_t gstate_warp_doubles(const KinTables& T, const KinSweepDev& S) {
  return static_cast<size_t>(T.m + S.n_axes) * kBlock +
         (kSmemX ? 0 : (static_cast<size_t>(T.n) * sizeof(XT) + 7) / 8 * kBlock);
}

// Kernel body shared by the table-driven kernel (kin_stochastic.cu) and the
// per-model JIT kernels (kin_jit.cpp).  Block = one warp; persistent warps.
template <class Model, bool kCount, bool kPhilox, class XT, bool kGlobal = false, bool kSmemX = false>
__device__ __forceinline__ void stochastic_body(const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                                                unsigned long long* __restrict__ next, int* ovf_flag) {
  extern __shared__ double smem[];
  constexpr int B = kBlock;
  const int tid = threadIdx.x, lane = tid & 31;
  // per-thread state, [slot][thread]: shared memory, or for models whose state
  // would leave few warps per SM, this block's region of global memory (same
  // layout, still coalesced; L1/L2-cached)
  // (a compile-time choice: with one pointer for both, every access would be a
  // generic load/store instead of LDS/STS)
  // (kSmemX, large models: x[] alone in shared memory — the leap updates and
  // propensity reads hit LDS/STS — and a[] + av[] in global memory)
  double* base = kGlobal ? S.gstate + static_cast<size_t>(blockIdx.x) * gstate_warp_doubles<XT, kSmemX>(T, S) : smem;
  double* a = base + tid;
  double* av = base + static_cast<size_t>(T.m) * B + tid;
  XT* x = (kGlobal && kSmemX) ? reinterpret_cast<XT*>(smem) + tid
                              : reinterpret_cast<XT*>(base + static_cast<size_t>(T.m + S.n_axes) * B) + tid;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, static_cast<unsigned long long>(S.warp_lanes));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (base >= S.n_local) break;
    const uint64_t s = lane < S.warp_lanes ? base + lane : S.n_local;  // lanes >= warp_lanes idle
    if (s < S.n_local) simulate_one<Model, kCount, kPhilox, XT>(T, S, O, s, x, a, av, ovf_flag);
    __syncwarp();
  }
}

}  // namespace stoch
}  // namespace kin

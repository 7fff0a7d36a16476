// oracle/kin_oracle.cpp — TEST INFRASTRUCTURE ONLY (CPU oracle / CPU baseline).
//
// Restates, from the reference's header contracts and SPEC (no .cpp exists for
// them in /root/reference), the hot path of arxiv/paper_1309_7695's kinetics
// library:
//   ReactionNetwork::create ....... model.hpp:47-53
//   propensities .................. model.hpp:145-157
//   apply_reaction ................ model.hpp:159-163
//   ssa_step(_from_uniforms) ...... stochastic.hpp:22-32
//   simulate_ssa .................. stochastic.hpp:34-38
//   select_tau .................... stochastic.hpp:40-46
//   tau_leap_step(_from_counts) ... stochastic.hpp:48-62
//   simulate_approx ............... stochastic.hpp:78-92
//   rre_rhs / rk_step / Dopri5 .... deterministic.hpp:26-95
//   derive_run_seed ............... ensemble.hpp:15-18
//   EnsembleStatistics ............ ensemble.hpp:20-57
//   run_ensemble / parameter_sweep  ensemble.hpp:78-130
// Built with -O3 -DNDEBUG -ffp-contract=off (the reference Release flags,
// proj/CMakeLists.txt:6-8, with contraction pinned off so the CUDA kernels,
// compiled with -fmad=false on the parity path, round identically).
#include "kin_oracle.hpp"
#include "kin_lsoda.hpp"
#include "kin_portable_math.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <thread>

namespace kin_oracle {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

void set_err(kin_error* e, int code, const std::string& msg) {
  if (!e) return;
  e->code = code;
  std::snprintf(e->message, sizeof(e->message), "%s", msg.c_str());
}
}  // namespace

void Scratch::resize(int n, int m) {
  x.assign(n, 0.0);
  xn.assign(n, 0.0);
  x0.assign(n, 0.0);
  z.assign(static_cast<size_t>(kLsodaL) * n + 1, 0.0);
  jac.assign(static_cast<size_t>(n) * n + 1, 0.0);
  jac2.assign(static_cast<size_t>(n) * n + 1, 0.0);
  piv.assign(n + 1, 0);
  a.assign(m, 0.0);
  rates.assign(m, 0.0);
  k.assign(m, 0);
  for (auto& vv : v) vv.assign(static_cast<size_t>(n) * (n > 1 ? n : 1) + 1, 0.0);
}

int build_network(const kin_model_desc* d, Network* net, std::string* msg) {
  if (!d) { *msg = "null model descriptor"; return KIN_ERR_USAGE; }
  const int n = d->n_species, m = d->n_reactions, np = d->n_params;
  if (n < 0 || m < 0 || np < 0) { *msg = "negative model dimension"; return KIN_ERR_INPUT; }
  if ((n > 0 && !d->initial_amounts) || (m > 0 && (!d->rate_constants || !d->reactant_ptr || !d->product_ptr))) {
    *msg = "missing model array"; return KIN_ERR_USAGE;
  }
  const int max_order = d->max_order <= 0 ? 2 : d->max_order;
  if (max_order > 3) { *msg = "max_order above 3 is not supported"; return KIN_ERR_INPUT; }
  Network& N = *net;
  N = Network{};
  N.n = n; N.m = m;
  for (int i = 0; i < n; ++i) {
    if (d->initial_amounts[i] < 0) { *msg = "species " + std::to_string(i) + ": negative initial amount"; return KIN_ERR_INPUT; }
    N.x0.push_back(static_cast<double>(d->initial_amounts[i]));
  }
  for (int p = 0; p < np; ++p) {
    if (!(d->param_values[p] > 0.0) || !std::isfinite(d->param_values[p])) { *msg = "param " + std::to_string(p) + ": rate must be positive"; return KIN_ERR_INPUT; }
    N.params.push_back(d->param_values[p]);
  }
  N.rt_ptr.push_back(0);
  N.col_ptr.push_back(0);
  std::vector<int> nu(static_cast<size_t>(n) * m, 0);
  N.g.assign(n, 1);
  for (int j = 0; j < m; ++j) {
    const int rp = d->rate_param ? d->rate_param[j] : -1;
    if (rp >= np || rp < -1) { *msg = "reaction " + std::to_string(j) + ": unknown parameter"; return KIN_ERR_INPUT; }
    const double c = rp >= 0 ? d->param_values[rp] : d->rate_constants[j];
    if (!(c > 0.0) || !std::isfinite(c)) { *msg = "reaction " + std::to_string(j) + ": rate must be positive"; return KIN_ERR_INPUT; }
    N.rate_base.push_back(d->rate_constants[j]);
    N.rate_param.push_back(rp);
    int order = 0, prev = -1;
    for (int p = d->reactant_ptr[j]; p < d->reactant_ptr[j + 1]; ++p) {
      const int s = d->reactant_species[p], st = d->reactant_stoich[p];
      if (s < 0 || s >= n) { *msg = "reaction " + std::to_string(j) + ": undeclared species"; return KIN_ERR_INPUT; }
      if (s <= prev) { *msg = "reaction " + std::to_string(j) + ": reactants must be species-ascending and unique"; return KIN_ERR_INPUT; }
      if (st <= 0) { *msg = "reaction " + std::to_string(j) + ": stoichiometry must be positive"; return KIN_ERR_INPUT; }
      prev = s;
      order += st;
      N.rt_species.push_back(s);
      N.rt_stoich.push_back(st);
      nu[static_cast<size_t>(s) * m + j] -= st;
    }
    if (order > max_order) { *msg = "reaction " + std::to_string(j) + ": reactant order " + std::to_string(order) + " exceeds " + std::to_string(max_order); return KIN_ERR_INPUT; }
    for (int p = d->reactant_ptr[j]; p < d->reactant_ptr[j + 1]; ++p)
      N.g[d->reactant_species[p]] = std::max(N.g[d->reactant_species[p]], order);
    prev = -1;
    for (int p = d->product_ptr[j]; p < d->product_ptr[j + 1]; ++p) {
      const int s = d->product_species[p], st = d->product_stoich[p];
      if (s < 0 || s >= n) { *msg = "reaction " + std::to_string(j) + ": undeclared species"; return KIN_ERR_INPUT; }
      if (s <= prev) { *msg = "reaction " + std::to_string(j) + ": products must be species-ascending and unique"; return KIN_ERR_INPUT; }
      if (st <= 0) { *msg = "reaction " + std::to_string(j) + ": stoichiometry must be positive"; return KIN_ERR_INPUT; }
      prev = s;
      nu[static_cast<size_t>(s) * m + j] += st;
    }
    N.order.push_back(order);
    N.rt_ptr.push_back(static_cast<int>(N.rt_species.size()));
    for (int s = 0; s < n; ++s) {
      const int dl = nu[static_cast<size_t>(s) * m + j];
      if (dl != 0) { N.col_species.push_back(s); N.col_delta.push_back(dl); }
    }
    N.col_ptr.push_back(static_cast<int>(N.col_species.size()));
  }
  N.row_ptr.push_back(0);
  for (int s = 0; s < n; ++s) {
    for (int j = 0; j < m; ++j) {
      const int dl = nu[static_cast<size_t>(s) * m + j];
      if (dl != 0) { N.row_reaction.push_back(j); N.row_delta.push_back(dl); }
    }
    N.row_ptr.push_back(static_cast<int>(N.row_reaction.size()));
  }
  return KIN_OK;
}

template <bool C>
double select_tau(const Network& net, const double* x, const double* a, double eps, Work* w) {
  double tau = kInf;
  for (int i = 0; i < net.n; ++i) {
    double mu = 0.0, s2 = 0.0;
    for (int p = net.row_ptr[i]; p < net.row_ptr[i + 1]; ++p) {
      const int dl = net.row_delta[p];
      const double aj = a[net.row_reaction[p]];
      mu = mu + static_cast<double>(dl) * aj;
      s2 = s2 + static_cast<double>(dl * dl) * aj;
    }
    if constexpr (C) w->flops += 4 * static_cast<std::uint64_t>(net.row_ptr[i + 1] - net.row_ptr[i]);
    if (mu == 0.0 && s2 == 0.0) continue;
    double bound = eps * x[i] / static_cast<double>(net.g[i]);
    if (bound < 1.0) bound = 1.0;
    if constexpr (C) w->flops += 2;
    if (mu != 0.0) {
      const double t1 = bound / std::fabs(mu);
      if (t1 < tau) tau = t1;
      if constexpr (C) w->flops += 1;
    }
    if (s2 != 0.0) {
      const double t2 = bound * bound / s2;
      if (t2 < tau) tau = t2;
      if constexpr (C) w->flops += 2;
    }
  }
  return tau;
}

int ssa_select(const Network& net, const double* a, double a0, double u2) {
  const double target = u2 * a0;
  double c = 0.0;
  int last = -1;
  for (int j = 0; j < net.m; ++j) {
    if (a[j] > 0.0) last = j;
    c = c + a[j];
    if (c > target) return j;
  }
  return last;
}

// One reaction of the sequential binomial leap (KIN_FIRING_BINOMIAL, kin_abi.h):
// k_j ~ Binomial(n_j, a_j tau / n_j), n_j = min over reactants of
// floor(x_s / stoich_s) at the amounts left after reactions 0..j-1 of this leap
// fired, so no amount can go negative and no leap is rejected; a zero-order
// reaction (no reactant bound) fires Poisson(a_j tau).  Draws in reaction order.
template <class Src>
std::uint64_t binomial_fire(const Network& net, Src& src, const double* x, int j, double mean, std::uint64_t* pf) {
  if (net.rt_ptr[j] == net.rt_ptr[j + 1]) return poisson_from(src, mean, pf);
  if (!(mean > 0.0)) return 0;
  double lim = kInf;
  for (int p = net.rt_ptr[j]; p < net.rt_ptr[j + 1]; ++p) {
    const double v = std::floor(x[net.rt_species[p]] / static_cast<double>(net.rt_stoich[p]));
    if (v < lim) lim = v;
  }
  if (pf) *pf += static_cast<std::uint64_t>(net.rt_ptr[j + 1] - net.rt_ptr[j]);
  if (!(lim > 0.0)) return 0;
  if (pf) *pf += 1;
  return binomial_from(src, static_cast<std::uint64_t>(lim), mean / lim, pf);
}

template <bool C>
int simulate_stochastic(const Network& net, const double* rates, const double* x0,
                        const kin_method& method, double t_end, const double* grid,
                        int n_grid, std::uint64_t seed, double* out, std::uint64_t* meta,
                        Scratch& sc, Work* w, int rng_mode) {
  const int n = net.n, m = net.m;
  double* x = sc.x.data();
  double* xn = sc.xn.data();
  double* a = sc.a.data();
  std::uint64_t* k = sc.k.data();
  std::uint64_t* pf = C ? &w->flops : nullptr;
  for (int i = 0; i < n; ++i) x[i] = x0[i];
  for (int q = 0; q < 6; ++q) meta[q] = 0;
  Stream rng(seed);
  const bool philox = rng_mode == KIN_RNG_PHILOX;
  std::uint64_t ev = 0;  // Philox event counter (leap attempts and SSA events)
  const int kind = method.kind;
  double t = 0.0;
  int gi = 0;
  auto emit = [&]() {
    std::memcpy(out + static_cast<size_t>(gi) * n, x, sizeof(double) * n);
    ++gi;
  };
  while (gi < n_grid && grid[gi] <= t) emit();
  const std::uint64_t budget = method.integrator.max_steps;
  std::uint64_t used = 0;

  while (t < t_end) {
    if (++used > budget) return KIN_SIM_BUDGET;
    propensities<C>(net, rates, x, a, w);
    double a0 = 0.0;
    for (int j = 0; j < m; ++j) a0 = a0 + a[j];
    if constexpr (C) w->flops += m;
    if (a0 == 0.0) break;  // every propensity vanished: the state is absorbing

    double tau = 0.0;
    bool burst = false;
    if (kind == KIN_METHOD_SSA) {
      burst = true;
    } else if (kind == KIN_METHOD_TAU_ADAPTIVE) {
      tau = select_tau<C>(net, x, a, method.epsilon, w);
      if constexpr (C) w->flops += 1;
      burst = tau < 10.0 / a0;  // SPEC.md:191 fallback threshold
    } else {
      tau = method.tau;
    }

    if (burst) {
      // Exact SSA events (direct method); a tau method takes at most 100 of them
      // before re-attempting a leap.
      bool stop = false;
      for (int b = 0;; ++b) {
        if (b > 0) {
          if (kind != KIN_METHOD_SSA && b >= 100) break;
          if (++used > budget) return KIN_SIM_BUDGET;
          propensities<C>(net, rates, x, a, w);
          a0 = 0.0;
          for (int j = 0; j < m; ++j) a0 = a0 + a[j];
          if constexpr (C) w->flops += m;
          if (a0 == 0.0) { stop = true; break; }
        }
        double u1, u2;
        if (philox) {
          PhiloxSite src(seed, ev++, kPhiloxSsaSite);
          u1 = src.draw_uniform();
          u2 = src.draw_uniform();
        } else {
          u1 = rng.draw_uniform();
          u2 = rng.draw_uniform();
        }
        const double dt = std::log(1.0 / u1) / a0;
        const double tn = t + dt;
        if constexpr (C) w->flops += 4 + 4;
        if (tn > t_end) { t = t_end; stop = true; break; }
        while (gi < n_grid && grid[gi] < tn) emit();
        const int j = ssa_select(net, a, a0, u2);
        if constexpr (C) w->flops += 1 + static_cast<std::uint64_t>(j + 1);
        for (int p = net.col_ptr[j]; p < net.col_ptr[j + 1]; ++p) {
          const double v = x[net.col_species[p]] + static_cast<double>(net.col_delta[p]);
          if (v < 0.0) return KIN_SIM_NEGATIVE;  // apply_reaction contract, model.hpp:159-161
          x[net.col_species[p]] = v;
        }
        if constexpr (C) w->flops += static_cast<std::uint64_t>(net.col_ptr[j + 1] - net.col_ptr[j]);
        t = tn;
        if (kind == KIN_METHOD_SSA) ++meta[0]; else ++meta[3];
        while (gi < n_grid && grid[gi] <= t) emit();
      }
      if (stop) break;
      continue;
    }

    // Poisson leap, truncated at the next grid time (App. B #3) so every grid
    // sample is an exact state; rejection halves tau.
    const double t_stop = (gi < n_grid && grid[gi] < t_end) ? grid[gi] : t_end;
    bool hit = false;
    const double gap = t_stop - t;
    if constexpr (C) w->flops += 1;
    if (!(tau < gap)) { tau = gap; hit = true; }
    if (method.firing == KIN_FIRING_BINOMIAL) {
      // sequential binomial leap: bounded by reactant availability, never rejected
      for (int i = 0; i < n; ++i) xn[i] = x[i];
      for (int j = 0; j < m; ++j) {
        std::uint64_t kj;
        if (philox) {
          PhiloxSite src(seed, ev, static_cast<std::uint32_t>(j));
          kj = binomial_fire(net, src, xn, j, a[j] * tau, pf);
        } else {
          kj = binomial_fire(net, rng, xn, j, a[j] * tau, pf);
        }
        if (kj == 0) continue;
        const double kd = static_cast<double>(kj);
        for (int p = net.col_ptr[j]; p < net.col_ptr[j + 1]; ++p)
          xn[net.col_species[p]] = xn[net.col_species[p]] + static_cast<double>(net.col_delta[p]) * kd;
      }
      if (philox) ++ev;
      if constexpr (C) w->flops += static_cast<std::uint64_t>(m) + 2 * static_cast<std::uint64_t>(net.col_ptr[m]);
    }
    for (; method.firing != KIN_FIRING_BINOMIAL;) {
      if (philox) {
        for (int j = 0; j < m; ++j) {
          PhiloxSite src(seed, ev, static_cast<std::uint32_t>(j));
          k[j] = poisson_from(src, a[j] * tau, pf);
        }
        ++ev;
      } else {
        for (int j = 0; j < m; ++j) k[j] = rng.draw_poisson(a[j] * tau, pf);
      }
      for (int i = 0; i < n; ++i) xn[i] = x[i];
      for (int j = 0; j < m; ++j) {
        if (k[j] == 0) continue;
        const double kj = static_cast<double>(k[j]);
        for (int p = net.col_ptr[j]; p < net.col_ptr[j + 1]; ++p)
          xn[net.col_species[p]] = xn[net.col_species[p]] + static_cast<double>(net.col_delta[p]) * kj;
      }
      if constexpr (C) w->flops += static_cast<std::uint64_t>(m) + 2 * static_cast<std::uint64_t>(net.col_ptr[m]);
      bool neg = false;
      for (int i = 0; i < n; ++i) neg |= xn[i] < 0.0;
      if (!neg) break;
      ++meta[1];
      tau = tau * 0.5;
      hit = false;
      if constexpr (C) w->flops += 1;
    }
    std::swap(x, xn);
    if (hit) {
      t = t_stop;
    } else {
      t = t + tau;
      if constexpr (C) w->flops += 1;
    }
    ++meta[0];
    while (gi < n_grid && grid[gi] <= t) emit();
  }
  while (gi < n_grid) emit();
  return KIN_SIM_OK;
}

// ---- Chemical Langevin Equation, Euler-Maruyama (stochastic.hpp:64-75,
// SPEC.md:163-171, :192) ----------------------------------------------------
// x' = x + sum_j nu_j a_j h + sum_j nu_j sqrt(a_j h) z_j with one standard normal
// per reaction (RngStream::draw_normal, rng.cpp:54-66: Box-Muller with a cached
// spare), reactions in index order, each reaction's drift and noise applied as
// one increment a_j h + sqrt(a_j h) z_j; then components below zero are clamped
// to 0 and counted (TrajectoryMeta::clamp_events).  Steps are
// truncated at the next grid time like the tau leaps (App. B #3), so samples are
// states at exactly the grid times.  Philox mode: z_j is the Box-Muller cosine
// of the two uniforms of site (seed, step, j).
// cle_step_from_normals (stochastic.hpp:71-75) on propensities a[] evaluated at
// x: x += nu_j (a_j h + sqrt(a_j h) z_j) for j in index order, then clamp.
template <bool C>
void cle_step_from_normals(const Network& net, double* x, const double* a, double h, const double* z,
                           std::uint64_t* clamped, Work* w) {
  for (int j = 0; j < net.m; ++j) {
    const double d = a[j] * h;
    const double inc = d + std::sqrt(d) * z[j];
    if constexpr (C) w->flops += 4;
    for (int p = net.col_ptr[j]; p < net.col_ptr[j + 1]; ++p)
      x[net.col_species[p]] = x[net.col_species[p]] + static_cast<double>(net.col_delta[p]) * inc;
    if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(net.col_ptr[j + 1] - net.col_ptr[j]);
  }
  for (int i = 0; i < net.n; ++i)
    if (x[i] < 0.0) {
      x[i] = 0.0;
      ++*clamped;
    }
}

template <bool C>
int simulate_cle(const Network& net, const double* rates, const double* x0, const kin_method& method,
                 double t_end, const double* grid, int n_grid, std::uint64_t seed, double* out,
                 std::uint64_t* meta, Scratch& sc, Work* w, int rng_mode) {
  const int n = net.n, m = net.m;
  double* x = sc.x.data();
  double* a = sc.a.data();
  for (int i = 0; i < n; ++i) x[i] = x0[i];
  for (int q = 0; q < 6; ++q) meta[q] = 0;
  Stream rng(seed);
  const bool philox = rng_mode == KIN_RNG_PHILOX;
  double t = 0.0;
  int gi = 0;
  auto emit = [&]() {
    std::memcpy(out + static_cast<size_t>(gi) * n, x, sizeof(double) * n);
    ++gi;
  };
  while (gi < n_grid && grid[gi] <= t) emit();
  const std::uint64_t budget = method.integrator.max_steps;
  std::uint64_t used = 0, step = 0, n_normal = 0;
  thread_local std::vector<double> z;
  z.resize(static_cast<size_t>(m));
  while (t < t_end) {
    if (++used > budget) return KIN_SIM_BUDGET;
    const double t_stop = (gi < n_grid && grid[gi] < t_end) ? grid[gi] : t_end;
    double h = method.tau;
    bool hit = false;
    const double gap = t_stop - t;
    if constexpr (C) w->flops += 1;
    if (!(h < gap)) { h = gap; hit = true; }
    propensities<C>(net, rates, x, a, w);
    for (int j = 0; j < m; ++j) {
      if (philox) {
        PhiloxSite src(seed, step, static_cast<std::uint32_t>(j));
        const double u1 = src.draw_uniform();
        const double u2 = src.draw_uniform();
        z[j] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
        if constexpr (C) w->flops += 4 + 3 + 1 + 2;
      } else {  // RngStream::draw_normal: a fresh Box-Muller pair every second draw
        z[j] = rng.draw_normal();
        if constexpr (C) w->flops += (n_normal % 2 == 0) ? 4 + 3 + 1 + 2 + 2 : 0;
        ++n_normal;
      }
    }
    std::uint64_t clamped = 0;
    cle_step_from_normals<C>(net, x, a, h, z.data(), &clamped, w);
    meta[2] += clamped;
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(x[i])) return KIN_SIM_NONFINITE;
    ++step;
    if (hit) {
      t = t_stop;
    } else {
      t = t + h;
      if constexpr (C) w->flops += 1;
    }
    ++meta[0];
    while (gi < n_grid && grid[gi] <= t) emit();
  }
  while (gi < n_grid) emit();
  return KIN_SIM_OK;
}

// ---- Dormand-Prince 5(4) (deterministic.hpp:26-83) --------------------------
// Coefficients: Dormand & Prince (1980); PI control, FSAL and the dense output
// follow Hairer, Norsett & Wanner's DOPRI5 conventions.
namespace dp {
constexpr double c2 = 1.0 / 5.0, c3 = 3.0 / 10.0, c4 = 4.0 / 5.0, c5 = 8.0 / 9.0;
constexpr double a21 = 1.0 / 5.0;
constexpr double a31 = 3.0 / 40.0, a32 = 9.0 / 40.0;
constexpr double a41 = 44.0 / 45.0, a42 = -56.0 / 15.0, a43 = 32.0 / 9.0;
constexpr double a51 = 19372.0 / 6561.0, a52 = -25360.0 / 2187.0, a53 = 64448.0 / 6561.0,
                 a54 = -212.0 / 729.0;
constexpr double a61 = 9017.0 / 3168.0, a62 = -355.0 / 33.0, a63 = 46732.0 / 5247.0,
                 a64 = 49.0 / 176.0, a65 = -5103.0 / 18656.0;
constexpr double a71 = 35.0 / 384.0, a73 = 500.0 / 1113.0, a74 = 125.0 / 192.0,
                 a75 = -2187.0 / 6784.0, a76 = 11.0 / 84.0;
constexpr double e1 = 71.0 / 57600.0, e3 = -71.0 / 16695.0, e4 = 71.0 / 1920.0,
                 e5 = -17253.0 / 339200.0, e6 = 22.0 / 525.0, e7 = -1.0 / 40.0;
constexpr double d1 = -12715105075.0 / 11282082432.0, d3 = 87487479700.0 / 32700410799.0,
                 d4 = -10690763975.0 / 1880347072.0, d5 = 701980252875.0 / 199316789632.0,
                 d6 = -1453857185.0 / 822651844.0, d7 = 69997945.0 / 29380423.0;
constexpr double kSafe = 0.9, kFacMinInv = 5.0 /* 1/0.2 */, kFacMaxInv = 0.1 /* 1/10 */;
constexpr double kBeta = 0.04, kExpo1 = 0.2 - kBeta * 0.75;
}  // namespace dp

template <bool C>
int integrate_rre(const Network& net, const double* rates, const double* x0,
                  const kin_integrator_config& cfg, double t_end, const double* grid,
                  int n_grid, double* out, std::uint64_t* meta, Scratch& sc, Work* w) {
  using namespace dp;
  const int n = net.n;
  double* y = sc.v[0].data();
  double* k1 = sc.v[1].data();
  double* k2 = sc.v[2].data();
  double* k3 = sc.v[3].data();
  double* k4 = sc.v[4].data();
  double* k5 = sc.v[5].data();
  double* k6 = sc.v[6].data();
  double* k7 = sc.v[7].data();
  double* yn = sc.v[8].data();
  double* ys = sc.v[9].data();
  double* r1 = sc.v[10].data();
  double* r2 = sc.v[11].data();
  double* r3 = sc.v[12].data();
  double* r4 = sc.v[13].data();
  double* r5 = sc.v[14].data();
  double* a = sc.a.data();
  const double rtol = cfg.rel_tol, atol = cfg.abs_tol;
  const double hmax = cfg.h_max > 0.0 ? cfg.h_max : kInf;
  for (int q = 0; q < 6; ++q) meta[q] = 0;
  bool floored = false;
  for (int i = 0; i < n; ++i) y[i] = x0[i];
  double t = 0.0;
  int gi = 0;
  while (gi < n_grid && grid[gi] <= t) {
    std::memcpy(out + static_cast<size_t>(gi) * n, y, sizeof(double) * n);
    ++gi;
  }
  if (!(t < t_end)) {
    while (gi < n_grid) { std::memcpy(out + static_cast<size_t>(gi) * n, y, sizeof(double) * n); ++gi; }
    return KIN_SIM_OK;
  }
  rre_rhs<C>(net, rates, y, a, k1, w);

  double h;
  if (cfg.h_init > 0.0) {
    h = cfg.h_init;
  } else {
    // Automatic initial step (Hairer's HINIT, order 5).
    double dnf = 0.0, dny = 0.0;
    for (int i = 0; i < n; ++i) {
      const double sk = atol + rtol * std::fabs(y[i]);
      const double qf = k1[i] / sk, qy = y[i] / sk;
      dnf = dnf + qf * qf;
      dny = dny + qy * qy;
    }
    if constexpr (C) w->flops += 8 * static_cast<std::uint64_t>(n);
    h = (dnf <= 1e-10 || dny <= 1e-10) ? 1.0e-6 : std::sqrt(dny / dnf) * 0.01;
    if (h > hmax) h = hmax;
    for (int i = 0; i < n; ++i) ys[i] = y[i] + h * k1[i];
    rre_rhs<C>(net, rates, ys, a, k2, w);
    double der2 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double sk = atol + rtol * std::fabs(y[i]);
      const double q = (k2[i] - k1[i]) / sk;
      der2 = der2 + q * q;
    }
    der2 = std::sqrt(der2) / h;
    const double der12 = std::max(der2, std::sqrt(dnf));
    const double h1 = der12 <= 1e-15 ? std::max(1.0e-6, h * 1.0e-3) : std::pow(0.01 / der12, 0.2);
    h = std::min(100.0 * h, h1);
    if (h > hmax) h = hmax;
    if constexpr (C) w->flops += 7 * static_cast<std::uint64_t>(n) + 12;
  }

  double facold = 1.0e-4;
  bool last_rejected = false;
  std::uint64_t attempts = 0;
  while (t < t_end) {
    if (attempts++ >= cfg.max_steps) return KIN_SIM_BUDGET;
    double hh = h < hmax ? h : hmax;
    bool hit = false;
    if (t + hh >= t_end) { hh = t_end - t; hit = true; }
    if (!(hh > 0.0) || t + hh == t) return KIN_SIM_STEP_UNDERFLOW;

    for (int i = 0; i < n; ++i) ys[i] = y[i] + hh * (a21 * k1[i]);
    rre_rhs<C>(net, rates, ys, a, k2, w);
    for (int i = 0; i < n; ++i) ys[i] = y[i] + hh * (a31 * k1[i] + a32 * k2[i]);
    rre_rhs<C>(net, rates, ys, a, k3, w);
    for (int i = 0; i < n; ++i) ys[i] = y[i] + hh * (a41 * k1[i] + a42 * k2[i] + a43 * k3[i]);
    rre_rhs<C>(net, rates, ys, a, k4, w);
    for (int i = 0; i < n; ++i)
      ys[i] = y[i] + hh * (a51 * k1[i] + a52 * k2[i] + a53 * k3[i] + a54 * k4[i]);
    rre_rhs<C>(net, rates, ys, a, k5, w);
    for (int i = 0; i < n; ++i)
      ys[i] = y[i] + hh * (a61 * k1[i] + a62 * k2[i] + a63 * k3[i] + a64 * k4[i] + a65 * k5[i]);
    rre_rhs<C>(net, rates, ys, a, k6, w);
    for (int i = 0; i < n; ++i)
      yn[i] = y[i] + hh * (a71 * k1[i] + a73 * k3[i] + a74 * k4[i] + a75 * k5[i] + a76 * k6[i]);
    rre_rhs<C>(net, rates, yn, a, k7, w);

    double sum = 0.0;
    bool finite = true;
    for (int i = 0; i < n; ++i) {
      const double e = hh * (e1 * k1[i] + e3 * k3[i] + e4 * k4[i] + e5 * k5[i] + e6 * k6[i] + e7 * k7[i]);
      const double sk = atol + rtol * std::max(std::fabs(y[i]), std::fabs(yn[i]));
      const double q = e / sk;
      sum = sum + q * q;
      finite &= std::isfinite(yn[i]);
    }
    const double err = std::sqrt(sum / static_cast<double>(n));
    if constexpr (C) w->flops += 63 * static_cast<std::uint64_t>(n) + 4;
    if (!finite || !std::isfinite(err)) return KIN_SIM_NONFINITE;
    const double fac11 = std::pow(err, kExpo1);

    if (err <= 1.0) {
      double fac = fac11 / std::pow(facold, kBeta);
      fac = std::max(kFacMaxInv, std::min(kFacMinInv, fac / kSafe));
      double hnew = hh / fac;
      facold = std::max(err, 1.0e-4);
      for (int i = 0; i < n; ++i) {
        r1[i] = y[i];
        const double yd = yn[i] - y[i];
        r2[i] = yd;
        const double bs = hh * k1[i] - yd;
        r3[i] = bs;
        r4[i] = yd - hh * k7[i] - bs;
        r5[i] = hh * (d1 * k1[i] + d3 * k3[i] + d4 * k4[i] + d5 * k5[i] + d6 * k6[i] + d7 * k7[i]);
      }
      const double tprev = t;
      t = hit ? t_end : t + hh;
      for (int i = 0; i < n; ++i) { y[i] = yn[i]; k1[i] = k7[i]; }
      if (last_rejected && hnew > hh) hnew = hh;
      last_rejected = false;
      h = hnew;
      ++meta[0];
      if constexpr (C) w->flops += 18 * static_cast<std::uint64_t>(n) + 8;
      // Dense output onto every grid time in (tprev, t]; exact at
      // the step end; floored at zero with a flag.
      while (gi < n_grid && grid[gi] <= t) {
        double* o = out + static_cast<size_t>(gi) * n;
        if (grid[gi] == t) {
          for (int i = 0; i < n; ++i) o[i] = y[i];
        } else {
          const double th = (grid[gi] - tprev) / hh;
          const double th1 = 1.0 - th;
          for (int i = 0; i < n; ++i)
            o[i] = r1[i] + th * (r2[i] + th1 * (r3[i] + th * (r4[i] + th1 * r5[i])));
          if constexpr (C) w->flops += 8 * static_cast<std::uint64_t>(n) + 3;
        }
        for (int i = 0; i < n; ++i)
          if (o[i] < 0.0) { o[i] = 0.0; floored = true; }
        ++gi;
      }
      bool lifted = false;
      for (int i = 0; i < n; ++i)
        if (y[i] < 0.0) { y[i] = 0.0; lifted = true; }
      if (lifted) {
        floored = true;
        rre_rhs<C>(net, rates, y, a, k1, w);
      }
    } else {
      h = hh / std::min(kFacMinInv, fac11 / kSafe);
      last_rejected = true;
      ++meta[1];
      if constexpr (C) w->flops += 3;
    }
  }
  while (gi < n_grid) {
    std::memcpy(out + static_cast<size_t>(gi) * n, y, sizeof(double) * n);
    ++gi;
  }
  meta[5] = floored ? 1 : 0;
  return KIN_SIM_OK;
}

// ---- Hybrid PDMP (hybrid.hpp:14-62) -------------------------
// Per segment: partition_reactions (slow iff a_j < theta_a or a reactant amount
// < theta_x), horizon = min(t + repartition_interval, t_end), threshold
// E = -ln(u); Dopri5 (the integrate_rre scheme) on the augmented system
// y = (x, G): dx/dt = sum_{j fast} nu_j a_j (row order, as rre_rhs), dG/dt =
// sum_{j slow} a_j (index order); error norm over all N+1 components.  On the
// accepted step where G reaches E, the root is bisected on the dense output
// until the bracket is <= 1e-10 relative in t; t* is the bracket's upper end.
// Grid times before t* take dense values, x(t*) the dense state; the firing
// slow reaction is the first slow j whose cumulative propensity at x(t*)
// exceeds u2 * sum_slow a (ssa_select rule over the slow set); nu_j is added
// to the continuous state (no rounding) and components below 0
// clamp to 0 (counted); grid times <= t* then take the post-jump state.  Each
// segment restarts the integrator (HINIT).  Step-size control and E use the
// portable pow/log (kin_portable_math.hpp) so the CUDA kernel reproduces the
// step sequence bit for bit.  meta: steps = accepted steps, rejected_leaps =
// rejected steps, clamp_events, jumps, floored.  Philox mode: u and u2 are the
// two uniforms of site (seed, segment, 0).
namespace {
struct HybridRhs {
  const Network& net;
  const double* rates;
  const std::vector<char>& slow;
  double* a;
  template <bool C>
  void operator()(const double* y, double* f, Work* w) const {
    const int n = net.n, m = net.m;
    propensities<C>(net, rates, y, a, w);
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int p = net.row_ptr[i]; p < net.row_ptr[i + 1]; ++p)
        if (!slow[net.row_reaction[p]]) acc = acc + static_cast<double>(net.row_delta[p]) * a[net.row_reaction[p]];
      f[i] = acc;
      if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(net.row_ptr[i + 1] - net.row_ptr[i]);
    }
    double g = 0.0;
    for (int j = 0; j < m; ++j)
      if (slow[j]) g = g + a[j];
    f[n] = g;
    if constexpr (C) w->flops += static_cast<std::uint64_t>(m);
  }
};
}  // namespace

// next_jump_with_threshold (hybrid.hpp:43-48): from (t, x = y[0..n-1]) under
// partition `slow`, integrate the augmented system toward t_hor until G = E.
// Grid samples on the way go to out[gi..] (pre-jump values).  On return t is
// t* (jumped) or t_hor, and y holds the (pre-jump, floored) state there.
template <bool C>
int hybrid_segment(const Network& net, const double* rates, const std::vector<char>& slow,
                   const kin_integrator_config& cfg, double E, double t_hor, double& t, Scratch& sc, Work* w,
                   const double* grid, int n_grid, int& gi, double* out, bool& floored, std::uint64_t& attempts,
                   std::uint64_t* meta, bool* jumped) {
  using namespace dp;
  const int n = net.n, n1 = n + 1;
  double* y = sc.v[0].data();
  double* k1 = sc.v[1].data();
  double* k2 = sc.v[2].data();
  double* k3 = sc.v[3].data();
  double* k4 = sc.v[4].data();
  double* k5 = sc.v[5].data();
  double* k6 = sc.v[6].data();
  double* k7 = sc.v[7].data();
  double* yn = sc.v[8].data();
  double* ys = sc.v[9].data();
  double* r1 = sc.v[10].data();
  double* r2 = sc.v[11].data();
  double* r3 = sc.v[12].data();
  double* r4 = sc.v[13].data();
  double* r5 = sc.v[14].data();
  const HybridRhs f{net, rates, slow, sc.a.data()};
  const double rtol = cfg.rel_tol, atol = cfg.abs_tol;
  const double hmax = cfg.h_max > 0.0 ? cfg.h_max : kInf;
  auto dense = [&](double th, int i) {
    const double th1 = 1.0 - th;
    return r1[i] + th * (r2[i] + th1 * (r3[i] + th * (r4[i] + th1 * r5[i])));
  };
  *jumped = false;
  y[n] = 0.0;  // G
  f.template operator()<C>(y, k1, w);
  double h;
  if (cfg.h_init > 0.0) {
    h = cfg.h_init;
  } else {  // HINIT over the N+1 components
    double dnf = 0.0, dny = 0.0;
    for (int i = 0; i < n1; ++i) {
      const double sk = atol + rtol * std::fabs(y[i]);
      const double qf = k1[i] / sk, qy = y[i] / sk;
      dnf = dnf + qf * qf;
      dny = dny + qy * qy;
    }
    h = (dnf <= 1e-10 || dny <= 1e-10) ? 1.0e-6 : std::sqrt(dny / dnf) * 0.01;
    if (h > hmax) h = hmax;
    for (int i = 0; i < n1; ++i) ys[i] = y[i] + h * k1[i];
    f.template operator()<C>(ys, k2, w);
    double der2 = 0.0;
    for (int i = 0; i < n1; ++i) {
      const double sk = atol + rtol * std::fabs(y[i]);
      const double q = (k2[i] - k1[i]) / sk;
      der2 = der2 + q * q;
    }
    der2 = std::sqrt(der2) / h;
    const double der12 = std::max(der2, std::sqrt(dnf));
    const double h1 = der12 <= 1e-15 ? std::max(1.0e-6, h * 1.0e-3) : pm_pow(0.01 / der12, 0.2);
    h = std::min(100.0 * h, h1);
    if (h > hmax) h = hmax;
    if constexpr (C) w->flops += 15 * static_cast<std::uint64_t>(n1) + 12;
  }
  double facold = 1.0e-4;
  bool last_rejected = false;
  while (t < t_hor) {
    if (attempts++ >= cfg.max_steps) return KIN_SIM_BUDGET;
    double hh = h < hmax ? h : hmax;
    bool hit = false;
    if (t + hh >= t_hor) { hh = t_hor - t; hit = true; }
    if (!(hh > 0.0) || t + hh == t) return KIN_SIM_STEP_UNDERFLOW;
    for (int i = 0; i < n1; ++i) ys[i] = y[i] + hh * (a21 * k1[i]);
    f.template operator()<C>(ys, k2, w);
    for (int i = 0; i < n1; ++i) ys[i] = y[i] + hh * (a31 * k1[i] + a32 * k2[i]);
    f.template operator()<C>(ys, k3, w);
    for (int i = 0; i < n1; ++i) ys[i] = y[i] + hh * (a41 * k1[i] + a42 * k2[i] + a43 * k3[i]);
    f.template operator()<C>(ys, k4, w);
    for (int i = 0; i < n1; ++i) ys[i] = y[i] + hh * (a51 * k1[i] + a52 * k2[i] + a53 * k3[i] + a54 * k4[i]);
    f.template operator()<C>(ys, k5, w);
    for (int i = 0; i < n1; ++i)
      ys[i] = y[i] + hh * (a61 * k1[i] + a62 * k2[i] + a63 * k3[i] + a64 * k4[i] + a65 * k5[i]);
    f.template operator()<C>(ys, k6, w);
    for (int i = 0; i < n1; ++i)
      yn[i] = y[i] + hh * (a71 * k1[i] + a73 * k3[i] + a74 * k4[i] + a75 * k5[i] + a76 * k6[i]);
    f.template operator()<C>(yn, k7, w);
    double sum = 0.0;
    bool finite = true;
    for (int i = 0; i < n1; ++i) {
      const double e = hh * (e1 * k1[i] + e3 * k3[i] + e4 * k4[i] + e5 * k5[i] + e6 * k6[i] + e7 * k7[i]);
      const double sk = atol + rtol * std::max(std::fabs(y[i]), std::fabs(yn[i]));
      const double q = e / sk;
      sum = sum + q * q;
      finite &= std::isfinite(yn[i]);
    }
    const double err = std::sqrt(sum / static_cast<double>(n1));
    if constexpr (C) w->flops += 63 * static_cast<std::uint64_t>(n1) + 4;
    if (!finite || !std::isfinite(err)) return KIN_SIM_NONFINITE;
    const double fac11 = pm_pow(err, kExpo1);
    if (err > 1.0) {
      h = hh / std::min(kFacMinInv, fac11 / kSafe);
      last_rejected = true;
      ++meta[1];
      if constexpr (C) w->flops += 3;
      continue;
    }
    double fac = fac11 / pm_pow(facold, kBeta);
    fac = std::max(kFacMaxInv, std::min(kFacMinInv, fac / kSafe));
    double hnew = hh / fac;
    facold = std::max(err, 1.0e-4);
    for (int i = 0; i < n1; ++i) {
      r1[i] = y[i];
      const double yd = yn[i] - y[i];
      r2[i] = yd;
      const double bs = hh * k1[i] - yd;
      r3[i] = bs;
      r4[i] = yd - hh * k7[i] - bs;
      r5[i] = hh * (d1 * k1[i] + d3 * k3[i] + d4 * k4[i] + d5 * k5[i] + d6 * k6[i] + d7 * k7[i]);
    }
    if (last_rejected && hnew > hh) hnew = hh;
    last_rejected = false;
    h = hnew;
    ++meta[0];
    if constexpr (C) w->flops += 18 * static_cast<std::uint64_t>(n1) + 8;
    const double tprev = t;
    const double tnew = hit ? t_hor : t + hh;
    if (yn[n] >= E) {
      // G reaches E inside (tprev, tnew]: bisection on the dense G until the
      // bracket is <= 1e-10 relative in t; t* = the bracket's upper end
      double lo = 0.0, hi = 1.0;
      for (int it = 0; it < 200; ++it) {
        const double tl = tprev + lo * hh, th = tprev + hi * hh;
        if (!(th - tl > 1e-10 * std::fabs(th))) break;
        const double mid = 0.5 * (lo + hi);
        if (dense(mid, n) >= E) hi = mid; else lo = mid;
        if constexpr (C) w->flops += 12;
      }
      const double ts = hi == 1.0 ? tnew : tprev + hi * hh;
      while (gi < n_grid && grid[gi] < ts) {
        double* o = out + static_cast<size_t>(gi) * n;
        const double th = (grid[gi] - tprev) / hh;
        for (int i = 0; i < n; ++i) {
          o[i] = dense(th, i);
          if (o[i] < 0.0) { o[i] = 0.0; floored = true; }
        }
        if constexpr (C) w->flops += 8 * static_cast<std::uint64_t>(n) + 3;
        ++gi;
      }
      for (int i = 0; i < n; ++i) {
        y[i] = hi == 1.0 ? yn[i] : dense(hi, i);
        if (y[i] < 0.0) { y[i] = 0.0; floored = true; }
      }
      t = ts;
      *jumped = true;
      return KIN_SIM_OK;
    }
    // no jump in this step: dense output onto (tprev, tnew], as integrate_rre
    t = tnew;
    for (int i = 0; i < n1; ++i) { y[i] = yn[i]; k1[i] = k7[i]; }
    while (gi < n_grid && grid[gi] <= t) {
      double* o = out + static_cast<size_t>(gi) * n;
      if (grid[gi] == t) {
        for (int i = 0; i < n; ++i) o[i] = y[i];
      } else {
        const double th = (grid[gi] - tprev) / hh;
        for (int i = 0; i < n; ++i) o[i] = dense(th, i);
        if constexpr (C) w->flops += 8 * static_cast<std::uint64_t>(n) + 3;
      }
      for (int i = 0; i < n; ++i)
        if (o[i] < 0.0) { o[i] = 0.0; floored = true; }
      ++gi;
    }
    bool lifted = false;
    for (int i = 0; i < n; ++i)
      if (y[i] < 0.0) { y[i] = 0.0; lifted = true; }
    if (lifted) {
      floored = true;
      f.template operator()<C>(y, k1, w);
    }
  }
  return KIN_SIM_OK;
}

// partition_reactions (hybrid.hpp:28-33): slow iff a_j < theta_a or a reactant
// amount < theta_x.  a[] = propensities at x.
inline void hybrid_partition(const Network& net, const double* x, const double* a, double theta_x, double theta_a,
                             std::vector<char>* slow) {
  slow->assign(static_cast<size_t>(net.m), 0);
  for (int j = 0; j < net.m; ++j) {
    bool sl = a[j] < theta_a;
    for (int p = net.rt_ptr[j]; p < net.rt_ptr[j + 1]; ++p) sl |= x[net.rt_species[p]] < theta_x;
    (*slow)[j] = sl;
  }
}

template <bool C>
int simulate_hybrid(const Network& net, const double* rates, const double* x0, const kin_method& method,
                    double t_end, const double* grid, int n_grid, std::uint64_t seed, double* out,
                    std::uint64_t* meta, Scratch& sc, Work* w, int rng_mode) {
  const int n = net.n, m = net.m;
  double* y = sc.v[0].data();
  double* a = sc.a.data();
  thread_local std::vector<char> slow;
  const double rep = method.repartition_interval > 0.0 ? method.repartition_interval : t_end / 100.0;
  for (int q = 0; q < 6; ++q) meta[q] = 0;
  bool floored = false;
  for (int i = 0; i < n; ++i) y[i] = x0[i];
  Stream rng(seed);
  const bool philox = rng_mode == KIN_RNG_PHILOX;
  double t = 0.0;
  int gi = 0;
  auto emit_state = [&]() {
    std::memcpy(out + static_cast<size_t>(gi) * n, y, sizeof(double) * n);
    ++gi;
  };
  while (gi < n_grid && grid[gi] <= t) emit_state();
  std::uint64_t attempts = 0, seg = 0;
  while (t < t_end) {
    propensities<C>(net, rates, y, a, w);
    hybrid_partition(net, y, a, method.theta_x, method.theta_a, &slow);
    const double t_hor = t + rep < t_end ? t + rep : t_end;
    PhiloxSite site(seed, seg, 0);
    const double u = philox ? site.draw_uniform() : rng.draw_uniform();
    const double E = -pm_log(u);
    if constexpr (C) w->flops += 3;
    bool jumped = false;
    const int rc = hybrid_segment<C>(net, rates, slow, method.integrator, E, t_hor, t, sc, w, grid, n_grid, gi, out,
                                     floored, attempts, meta, &jumped);
    if (rc != KIN_SIM_OK) return rc;
    if (jumped) {
      // the caller's selection (hybrid.hpp:39-40): first slow j whose cumulative
      // propensity at x(t*) exceeds u2 * sum_slow a
      propensities<C>(net, rates, y, a, w);
      double as = 0.0;
      for (int j = 0; j < m; ++j)
        if (slow[j]) as = as + a[j];
      const double u2 = philox ? site.draw_uniform() : rng.draw_uniform();
      if (as > 0.0) {
        const double target = u2 * as;
        double c = 0.0;
        int sel = -1, last = -1;
        for (int j = 0; j < m; ++j) {
          if (!slow[j]) continue;
          if (a[j] > 0.0) last = j;
          c = c + a[j];
          if (c > target) { sel = j; break; }
        }
        if (sel < 0) sel = last;
        for (int p = net.col_ptr[sel]; p < net.col_ptr[sel + 1]; ++p) {
          double& v = y[net.col_species[p]];
          v = v + static_cast<double>(net.col_delta[p]);
          if (v < 0.0) { v = 0.0; ++meta[2]; }
        }
        ++meta[4];
        if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(m) + 1;
      }
      while (gi < n_grid && grid[gi] <= t) emit_state();
    }
    ++seg;
  }
  while (gi < n_grid) emit_state();
  meta[5] = floored ? 1 : 0;
  return KIN_SIM_OK;
}

constexpr bool kLsodaAvailable = true;

// Analytic Jacobian of the RRE, J = nu * da/dx (row-major N x N), continuous
// combinations with the same clamp as propensities (zero slope where clamped).
template <bool C>
void rre_jacobian(const Network& net, const double* rates, const double* x, double* J, Work* w) {
  const int n = net.n;
  for (int q = 0; q < n * n; ++q) J[q] = 0.0;
  for (int k = 0; k < net.m; ++k) {
    const int p0 = net.rt_ptr[k], p1 = net.rt_ptr[k + 1];
    for (int p = p0; p < p1; ++p) {
      // d a_k / d x_s for reactant term p
      const int s = net.rt_species[p], st = net.rt_stoich[p];
      const double xs = x[s];
      double dh;
      const double h = combinations(xs, st);
      if (st == 1) dh = xs < 0.0 ? 0.0 : 1.0;
      else if (st == 2) dh = h > 0.0 ? xs - 0.5 : 0.0;
      else dh = h > 0.0 ? ((3.0 * xs - 6.0) * xs + 2.0) / 6.0 : 0.0;
      double d = rates[k] * dh;
      for (int q = p0; q < p1; ++q)
        if (q != p) d = d * combinations(x[net.rt_species[q]], net.rt_stoich[q]);
      for (int c = net.col_ptr[k]; c < net.col_ptr[k + 1]; ++c)
        J[net.col_species[c] * n + s] += static_cast<double>(net.col_delta[c]) * d;
      if constexpr (C) w->flops += 4 + (p1 - p0) + 2 * static_cast<std::uint64_t>(net.col_ptr[k + 1] - net.col_ptr[k]);
    }
  }
}

// LU with partial pivoting, in place (row-major), piv[i] = pivot row.
// Returns false when singular.
template <bool C>
bool lu_factor(double* A, int n, int* piv, Work* w) {
  for (int k = 0; k < n; ++k) {
    int pr = k;
    double best = std::fabs(A[k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(A[i * n + k]) > best) { best = std::fabs(A[i * n + k]); pr = i; }
    piv[k] = pr;
    if (best == 0.0) return false;
    if (pr != k)
      for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[pr * n + j]);
    const double inv = 1.0 / A[k * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double l = A[i * n + k] * inv;
      A[i * n + k] = l;
      for (int j = k + 1; j < n; ++j) A[i * n + j] -= l * A[k * n + j];
    }
  }
  if constexpr (C) w->flops += static_cast<std::uint64_t>(2 * n * n * n / 3 + n);
  return true;
}

template <bool C>
void lu_solve(const double* A, int n, const int* piv, double* b, Work* w) {
  for (int k = 0; k < n; ++k) {
    if (piv[k] != k) std::swap(b[k], b[piv[k]]);
    for (int i = k + 1; i < n; ++i) b[i] -= A[i * n + k] * b[k];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A[i * n + j] * b[j];
    b[i] = s / A[i * n + i];
  }
  if constexpr (C) w->flops += static_cast<std::uint64_t>(2 * n * n);
}

// LSODA-style integration of the RRE (see oracle/kin_lsoda.hpp for sources).
// Nordsieck history Z[j] = h^j y^(j)/j!, j = 0..12; Adams orders 1..12 with
// functional iteration, BDF orders 1..5 with chord Newton on P = I - h*l0*J;
// LSODE error test, order/step selection every nq+1 steps; LSODA method
// switching (stiffness ratio 5, Adams stability sizes sm1, Jacobian norm).
// Grid values by Nordsieck interpolation inside each accepted step, floored at
// zero (flag); the state itself is not modified.
template <bool C>
int integrate_lsoda(const Network& net, const double* rates, const double* x0, const kin_integrator_config& cfg,
                    double t_end, const double* grid, int n_grid, double* out, std::uint64_t* meta, Scratch& sc,
                    Work* w) {
  static const LsodaCoeffs CO = [] { LsodaCoeffs c; kin_lsoda_coeffs(&c); return c; }();
  const int n = net.n;
  const double rtol = cfg.rel_tol, atol = cfg.abs_tol;
  const double hmax = cfg.h_max > 0.0 ? cfg.h_max : kInf;
  const std::uint64_t F_rhs = static_cast<std::uint64_t>(
      [&] { std::uint64_t f = 0; for (int p = 0; p < static_cast<int>(net.rt_species.size()); ++p) f += 1 + combinations_flops(net.rt_stoich[p]); return f; }() +
      2 * net.row_reaction.size());
  double* Z = sc.z.data();  // 13 x n
  double* acor = sc.v[0].data();
  double* savf = sc.v[1].data();
  double* ewt = sc.v[2].data();
  double* y = sc.v[3].data();
  double* tmp = sc.v[4].data();
  double* P = sc.jac.data();
  int* piv = sc.piv.data();
  double* a = sc.a.data();
  auto Zr = [&](int j) { return Z + static_cast<size_t>(j) * n; };
  for (int q = 0; q < 6; ++q) meta[q] = 0;
  bool floored = false;
  auto rhs = [&](const double* yy, double* f) {
    rre_rhs<false>(net, rates, yy, a, f, nullptr);
    if constexpr (C) w->flops += F_rhs;
  };
  auto wrms = [&](const double* v) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) { const double q = v[i] / ewt[i]; s += q * q; }
    if constexpr (C) w->flops += 3 * static_cast<std::uint64_t>(n) + 2;
    return std::sqrt(s / n);
  };
  auto emit = [&](int g, const double* v) {
    double* o = out + static_cast<size_t>(g) * n;
    for (int i = 0; i < n; ++i) {
      double vi = v[i];
      if (vi < 0.0) { vi = 0.0; floored = true; }
      o[i] = vi;
    }
  };

  double t = 0.0;
  int gi = 0;
  for (int i = 0; i < n; ++i) y[i] = x0[i];
  while (gi < n_grid && grid[gi] <= t) emit(gi++, y);
  if (!(t < t_end)) {
    while (gi < n_grid) emit(gi++, y);
    return KIN_SIM_OK;
  }
  for (int i = 0; i < n; ++i) { Zr(0)[i] = y[i]; ewt[i] = rtol * std::fabs(y[i]) + atol; }
  rhs(y, savf);
  double h;
  if (cfg.h_init > 0.0) {
    h = cfg.h_init;
  } else {
    // LSODA's starting step: h0 = (1/(tol*w0^2) + tol*||f0||^2)^(-1/2), weighted
    // max-norm, tol = rtol clamped to [100*uround, 1e-3], w0 = tdist = t_end
    double tol = rtol;
    if (tol < 100.0 * 2.220446049250313e-16) tol = 100.0 * 2.220446049250313e-16;
    if (tol > 1e-3) tol = 1e-3;
    double fn = 0.0;
    for (int i = 0; i < n; ++i) fn = std::max(fn, std::fabs(savf[i]) / ewt[i]);
    const double w0 = t_end;
    const double sum = 1.0 / (tol * w0 * w0) + tol * fn * fn;
    h = 1.0 / std::sqrt(sum);
    if (h > t_end) h = t_end;
    if (h > hmax) h = hmax;
    if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(n) + 10;
  }
  for (int i = 0; i < n; ++i) Zr(1)[i] = h * savf[i];

  int meth = 0;  // 0 Adams, 1 BDF
  int nq = 1;
  int ialth = 2;
  int icount = 20;
  int nstab = 0;  // consecutive order selections whose Adams step the stability cap bound
  double rmax = 1.0e4;
  double crate = 0.7;
  bool ipup = false, jcur = false, have_p = false;
  double hl0_p = 0.0;  // h*l0 when P was formed
  std::uint64_t nst = 0, nslp = 0, attempts = 0;
  const double* el = CO.elco[meth][nq];
  auto maxord = [&]() { return meth == 0 ? kLsodaMaxOrdAdams : kLsodaMaxOrdBdf; };
  auto set_order = [&](int m, int q) { meth = m; nq = q; el = CO.elco[meth][nq]; };
  auto rescale = [&](double rh) {
    double r = rh;
    for (int j = 1; j <= nq; ++j) {
      double* zj = Zr(j);
      for (int i = 0; i < n; ++i) zj[i] *= r;
      r *= rh;
    }
    h *= rh;
    if constexpr (C) w->flops += static_cast<std::uint64_t>(nq) * (n + 1);
  };
  auto predict = [&]() {
    for (int k = 0; k < nq; ++k)
      for (int j = nq - 1; j >= k; --j) {
        double* a0 = Zr(j);
        const double* a1 = Zr(j + 1);
        for (int i = 0; i < n; ++i) a0[i] += a1[i];
      }
    if constexpr (C) w->flops += static_cast<std::uint64_t>(nq) * (nq + 1) / 2 * n;
  };
  auto unpredict = [&]() {
    for (int k = nq - 1; k >= 0; --k)
      for (int j = k; j <= nq - 1; ++j) {
        double* a0 = Zr(j);
        const double* a1 = Zr(j + 1);
        for (int i = 0; i < n; ++i) a0[i] -= a1[i];
      }
  };
  auto form_p = [&](const double* yy) {
    rre_jacobian<C>(net, rates, yy, P, w);
    const double hl0 = h * el[0];
    for (int q = 0; q < n * n; ++q) P[q] = -hl0 * P[q];
    for (int i = 0; i < n; ++i) P[i * n + i] += 1.0;
    hl0_p = hl0;
    have_p = lu_factor<C>(P, n, piv, w);
    return have_p;
  };
  // weighted max-row-sum norm of J at yy (LSODA fnorm with weights 1/ewt)
  auto jac_norm = [&](const double* yy) {
    rre_jacobian<C>(net, rates, yy, sc.jac2.data(), w);
    const double* J = sc.jac2.data();
    double nm = 0.0;
    for (int i = 0; i < n; ++i) {
      double sr = 0.0;
      for (int j = 0; j < n; ++j) sr += std::fabs(J[i * n + j]) * ewt[j];
      nm = std::max(nm, sr / ewt[i]);
    }
    if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(n) * n + n;
    return nm;
  };
  auto sm1 = [](int q) { return kLsodaSm1[q]; };
  auto cm1 = [&](int q) { return CO.tesco[0][q][1] * CO.elco[0][q][q]; };
  auto cm2 = [&](int q) { return CO.tesco[1][q][1] * CO.elco[1][q][q]; };

  int kflag = 0;
  int ncf = 0;
  while (t < t_end) {
    // ---- one accepted step (stode) ----
    for (int i = 0; i < n; ++i) ewt[i] = rtol * std::fabs(Zr(0)[i]) + atol;
    kflag = 0;
    ncf = 0;
    double dsm = 0.0;
    for (;;) {
      if (attempts++ >= cfg.max_steps) return KIN_SIM_BUDGET;
      if (!(h > 0.0) || t + h == t) return KIN_SIM_STEP_UNDERFLOW;
      if (meth == 1 && (!have_p || std::fabs(h * el[0] / hl0_p - 1.0) > 0.3 || nst >= nslp + 20)) ipup = true;
      const double tn = t + h;
      predict();
      bool conv = false;
      for (;;) {  // corrector (re-entered once with a fresh Jacobian)
        for (int i = 0; i < n; ++i) y[i] = Zr(0)[i];
        rhs(y, savf);
        if (meth == 1 && ipup) {
          if (!form_p(y)) return KIN_SIM_NONFINITE;
          ipup = false;
          jcur = true;
          crate = 0.7;
          nslp = nst;
        }
        for (int i = 0; i < n; ++i) acor[i] = 0.0;
        double delp = 0.0;
        int m = 0;
        for (;;) {
          double del;
          if (meth == 1) {
            for (int i = 0; i < n; ++i) tmp[i] = h * savf[i] - (Zr(1)[i] + acor[i]);
            lu_solve<C>(P, n, piv, tmp, w);
            del = wrms(tmp);
            for (int i = 0; i < n; ++i) { acor[i] += tmp[i]; y[i] = Zr(0)[i] + el[0] * acor[i]; }
          } else {
            for (int i = 0; i < n; ++i) tmp[i] = h * savf[i] - Zr(1)[i];
            for (int i = 0; i < n; ++i) acor[i] = tmp[i] - acor[i];
            del = wrms(acor);
            for (int i = 0; i < n; ++i) { y[i] = Zr(0)[i] + el[0] * tmp[i]; acor[i] = tmp[i]; }
          }
          if constexpr (C) w->flops += 5 * static_cast<std::uint64_t>(n);
          if (!std::isfinite(del)) { conv = false; break; }
          if (m != 0) crate = std::max(0.2 * crate, del / delp);
          const double conit = 0.5 / (nq + 2);
          const double dcon = del * std::min(1.0, 1.5 * crate) / (CO.tesco[meth][nq][1] * conit);
          if (dcon <= 1.0) { conv = true; break; }
          ++m;
          if (m == 3 || (m >= 2 && del > 2.0 * delp)) break;
          delp = del;
          rhs(y, savf);
        }
        if (conv) break;
        if (meth == 1 && !jcur) { ipup = true; continue; }
        break;
      }
      if (!conv) {
        unpredict();
        ++meta[1];
        if (++ncf >= 10) return KIN_SIM_STEP_UNDERFLOW;
        rescale(0.25);
        if (meth == 1) ipup = true;
        continue;
      }
      jcur = false;
      dsm = wrms(acor) / CO.tesco[meth][nq][1];
      if (dsm > 1.0) {
        unpredict();
        ++meta[1];
        --kflag;
        if (kflag <= -3) {
          // repeated error-test failures: restart at order 1 with h/10
          for (int i = 0; i < n; ++i) y[i] = Zr(0)[i];
          h *= 0.1;
          rhs(y, savf);
          for (int i = 0; i < n; ++i) Zr(1)[i] = h * savf[i];
          set_order(meth, 1);
          ialth = 5;
          if (meth == 1) ipup = true;
          continue;
        }
        const double rhsm = 1.0 / (1.2 * pm_pow(dsm, 1.0 / (nq + 1)) + 1.2e-6);
        double rhdn = 0.0;
        if (nq > 1) {
          const double ddn = wrms(Zr(nq)) / CO.tesco[meth][nq][0];
          rhdn = 1.0 / (1.3 * pm_pow(ddn, 1.0 / nq) + 1.3e-6);
        }
        double rh;
        if (rhsm >= rhdn) {
          rh = rhsm;
        } else {
          rh = rhdn;
          set_order(meth, nq - 1);
        }
        rh = std::min(rh, 1.0);
        if (kflag <= -2) rh = std::min(rh, 0.2);
        rescale(rh);
        if (meth == 1) ipup = true;
        ialth = nq + 1;
        continue;
      }
      // ---- accepted ----
      ++nst;
      ++meta[0];
      if (meth == 1) ++meta[3];  // accepted BDF steps (the stiff share; TrajectoryMeta slot 3)
      for (int j = 0; j <= nq; ++j) {
        double* zj = Zr(j);
        const double e = el[j];
        for (int i = 0; i < n; ++i) zj[i] += e * acor[i];
      }
      if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(nq + 1) * n;
      const double tprev = t;
      t = tn;
      while (gi < n_grid && grid[gi] <= t && grid[gi] > tprev) {
        const double s = (grid[gi] - t) / h;
        for (int i = 0; i < n; ++i) {
          double v = Zr(nq)[i];
          for (int j = nq - 1; j >= 0; --j) v = Zr(j)[i] + s * v;
          tmp[i] = v;
        }
        if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(nq) * n + 2;
        emit(gi++, tmp);
      }
      break;
    }
    // ---- order / step / method selection ----
    --ialth;
    if (ialth == 0) {
      const double rhsm = 1.0 / (1.2 * pm_pow(dsm, 1.0 / (nq + 1)) + 1.2e-6);
      double rhsm_cap;
      double rhup = 0.0;
      if (nq < maxord()) {
        const double* sv = Zr(kLsodaL - 1);
        for (int i = 0; i < n; ++i) tmp[i] = acor[i] - sv[i];
        const double dup = wrms(tmp) / CO.tesco[meth][nq][2];
        rhup = 1.0 / (1.4 * pm_pow(dup, 1.0 / (nq + 2)) + 1.4e-6);
      }
      double rhdn = 0.0;
      if (nq > 1) {
        const double ddn = wrms(Zr(nq)) / CO.tesco[meth][nq][0];
        rhdn = 1.0 / (1.3 * pm_pow(ddn, 1.0 / nq) + 1.3e-6);
      }
      // Adams steps are also capped by the stability region (LSODA sm1):
      // h*||J|| <= sm1(order) for the order each candidate would use.
      double pdnorm = -1.0;
      if (meth == 0) {
        pdnorm = jac_norm(Zr(0));
        const double pdh = std::max(h * pdnorm, 1.0e-6);
        if (nq < kLsodaMaxOrdAdams) rhup = std::min(rhup, sm1(nq + 1) / pdh);
        rhsm_cap = std::min(rhsm, sm1(nq) / pdh);
        if (nq > 1) rhdn = std::min(rhdn, sm1(nq - 1) / pdh);
        nstab = pdh >= 0.5 * sm1(nq) ? nstab + 1 : 0;  // within 2x of the stability boundary
      } else {
        rhsm_cap = rhsm;
        nstab = 0;
      }
      int newq = nq;
      double rh = rhsm_cap;
      if (rhsm_cap >= rhup) {
        if (rhsm_cap < rhdn) { newq = nq - 1; rh = rhdn; }
      } else if (rhup > rhdn) {
        newq = nq + 1;
        rh = rhup;
      } else {
        newq = nq - 1;
        rh = rhdn;
      }
      // LSODA stiffness switch (Petzold): compare the step each method could take
      int newm = meth;
      if (icount > 0) {
        --icount;
      } else {
        if (pdnorm < 0.0) pdnorm = jac_norm(Zr(0));
        const double exsm = 1.0 / (nq + 1);
        if (meth == 0 && nq <= kLsodaMaxOrdBdf) {
          // Adams -> BDF when BDF could step ratio*5 farther than the
          // (stability-capped) Adams choice
          const double rh1 = rh;
          const double dm2 = dsm * (cm1(nq) / cm2(nq));
          const double rh2 = 1.0 / (1.2 * pm_pow(dm2, exsm) + 1.2e-6);
          if (rh2 >= 5.0 * rh1) {
            newm = 1; newq = nq; rh = rh2;
          } else if (nstab >= kLsodaStabSwitch) {
            // extension of Petzold's test: the Adams step has been held by its
            // stability region for kLsodaStabSwitch selections in a row (a stiff
            // mode near the stability boundary inflates the Adams error
            // estimate, so the error-constant comparison above never fires)
            newm = 1; newq = nq; rh = rh1;
          }
        } else if (meth == 1) {
          const double dm1 = dsm * (cm2(nq) / cm1(nq));
          double rh1 = 1.0 / (1.2 * pm_pow(dm1, exsm) + 1.2e-6);
          double rh1it = 2.0 * rh1;
          const double pdh = pdnorm * h;
          if (pdh * rh1 > 1e-5) rh1it = sm1(nq) / pdh;
          rh1 = std::min(rh1, rh1it);
          const double rh2 = rh;
          if (rh1 >= rh2) { newm = 0; newq = nq; rh = rh1; }
        }
        if (newm != meth) icount = 20;
        else icount = 0;
      }
      if (newm == meth && newq == nq && rh < 1.1) {
        ialth = 3;
      } else {
        if (newq == nq + 1) {
          const double r = el[nq] / (nq + 1);
          double* zq = Zr(newq);
          for (int i = 0; i < n; ++i) zq[i] = acor[i] * r;
        }
        rh = std::min(rh, rmax);
        rh = rh / std::max(1.0, h * rh / hmax);
        if (newm != meth || newq != nq) set_order(newm, newq);
        rescale(rh);
        ialth = nq + 1;
        if (meth == 1) ipup = true;
      }
      rmax = 10.0;
    } else if (ialth == 1 && nq < maxord()) {
      double* sv = Zr(kLsodaL - 1);
      for (int i = 0; i < n; ++i) sv[i] = acor[i];
    }
  }
  while (gi < n_grid) emit(gi++, Zr(0));
  meta[5] = floored ? 1 : 0;
  return KIN_SIM_OK;
}

// ---- sweep decoding (ensemble.hpp:101-130) ----------------------------------
int sweep_layout(const kin_sweep_desc* d, SweepLayout* L, std::string* msg) {
  if (!d) { *msg = "null sweep descriptor"; return KIN_ERR_USAGE; }
  if (d->n_axes < 0 || (d->n_axes > 0 && !d->axes)) { *msg = "bad axes"; return KIN_ERR_USAGE; }
  std::uint64_t P = 1;
  for (int ax = 0; ax < d->n_axes; ++ax) {
    const kin_sweep_axis& A = d->axes[ax];
    if (A.n_values <= 0 || !A.values) { *msg = "axis " + std::to_string(ax) + ": empty value list"; return KIN_ERR_INPUT; }
    if (P > (std::uint64_t{1} << 40) / static_cast<std::uint64_t>(A.n_values)) { *msg = "sweep too large"; return KIN_ERR_INPUT; }
    P *= static_cast<std::uint64_t>(A.n_values);
  }
  if (d->runs_per_point == 0) { *msg = "runs_per_point must be >= 1"; return KIN_ERR_INPUT; }
  L->n_points = P;
  L->runs = d->runs_per_point;
  L->n_sims = P * d->runs_per_point;
  return KIN_OK;
}

void decode_sim(const Network& net, const kin_sweep_desc* d, std::uint64_t sim, double* rates,
                double* x0, std::uint64_t* seed) {
  const std::uint64_t R = d->runs_per_point;
  const std::uint64_t point = sim / R, run = sim % R;
  double params[64];
  std::vector<double> pbig;
  double* pv = params;
  if (net.params.size() > 64) { pbig = net.params; pv = pbig.data(); }
  else for (size_t p = 0; p < net.params.size(); ++p) params[p] = net.params[p];
  for (int i = 0; i < net.n; ++i) x0[i] = net.x0[i];
  std::uint64_t rem = point;
  for (int ax = d->n_axes - 1; ax >= 0; --ax) {
    const kin_sweep_axis& A = d->axes[ax];
    const std::uint64_t nv = static_cast<std::uint64_t>(A.n_values);
    const double v = A.values[rem % nv];
    rem /= nv;
    if (A.kind == KIN_AXIS_PARAM) pv[A.index] = v;
    else if (A.kind == KIN_AXIS_INITIAL) x0[A.index] = v;
  }
  for (int j = 0; j < net.m; ++j) rates[j] = net.rate_param[j] >= 0 ? pv[net.rate_param[j]] : net.rate_base[j];
  // global scale factors (KIN_AXIS_SCALE): c_j * s for the axis' reactions
  rem = point;
  for (int ax = d->n_axes - 1; ax >= 0; --ax) {
    const kin_sweep_axis& A = d->axes[ax];
    const std::uint64_t nv = static_cast<std::uint64_t>(A.n_values);
    const double v = A.values[rem % nv];
    rem /= nv;
    if (A.kind == KIN_AXIS_SCALE)
      for (int j = A.index; j < A.index + A.span; ++j) rates[j] = rates[j] * v;
  }
  switch (d->seed_mode) {
    case KIN_SEED_ENSEMBLE: *seed = derive_run_seed(d->master_seed, sim); break;
    case KIN_SEED_DIRECT: *seed = sim == 0 ? d->master_seed : derive_run_seed(d->master_seed, sim); break;
    default: *seed = derive_run_seed(derive_run_seed(d->master_seed, point), run); break;
  }
}

int validate_sweep(const Network& net, const kin_sweep_desc* d, std::string* msg) {
  const kin_method& M = d->method;
  if (M.kind == KIN_METHOD_HYBRID && !(M.theta_x >= 0.0 && M.theta_a >= 0.0 && M.repartition_interval >= 0.0)) { *msg = "hybrid thresholds and repartition interval must be non-negative"; return KIN_ERR_INPUT; }
  if (M.kind == KIN_METHOD_HYBRID && !(M.integrator.rel_tol > 0.0 && M.integrator.abs_tol > 0.0)) { *msg = "tolerances must be positive"; return KIN_ERR_INPUT; }
  if (M.kind == KIN_METHOD_CLE && !(M.tau > 0.0)) { *msg = "tau must be positive"; return KIN_ERR_INPUT; }
  if (M.kind < 0 || M.kind > KIN_METHOD_LSODA) { *msg = "unknown method kind"; return KIN_ERR_INPUT; }
  if (M.kind == KIN_METHOD_LSODA && !kLsodaAvailable) { *msg = "LSODA not built"; return KIN_ERR_INPUT; }
  if (M.kind == KIN_METHOD_TAU_FIXED && !(M.tau > 0.0)) { *msg = "tau must be positive"; return KIN_ERR_INPUT; }
  if (M.kind == KIN_METHOD_TAU_ADAPTIVE && !(M.epsilon > 0.0 && M.epsilon < 1.0)) { *msg = "epsilon must be in (0,1)"; return KIN_ERR_INPUT; }
  if (M.integrator.max_steps == 0) { *msg = "max_steps must be positive"; return KIN_ERR_INPUT; }
  if ((M.kind == KIN_METHOD_ODE || M.kind == KIN_METHOD_LSODA) && !(M.integrator.rel_tol > 0.0 && M.integrator.abs_tol > 0.0)) { *msg = "tolerances must be positive"; return KIN_ERR_INPUT; }
  if (!(d->t_end >= 0.0) || !std::isfinite(d->t_end)) { *msg = "t_end must be finite and non-negative"; return KIN_ERR_INPUT; }
  if (d->n_grid < 0 || (d->n_grid > 0 && !d->grid)) { *msg = "bad grid"; return KIN_ERR_USAGE; }
  for (int g = 0; g < d->n_grid; ++g) {
    if (!(d->grid[g] >= 0.0 && d->grid[g] <= d->t_end)) { *msg = "grid point outside [0, t_end]"; return KIN_ERR_INPUT; }
    if (g > 0 && !(d->grid[g] > d->grid[g - 1])) { *msg = "grid must be strictly increasing"; return KIN_ERR_INPUT; }
  }
  for (int ax = 0; ax < d->n_axes; ++ax) {
    const kin_sweep_axis& A = d->axes[ax];
    if (A.kind == KIN_AXIS_PARAM) {
      if (A.index < 0 || A.index >= static_cast<int>(net.params.size())) { *msg = "axis " + std::to_string(ax) + ": unknown parameter"; return KIN_ERR_INPUT; }
      for (int v = 0; v < A.n_values; ++v)
        if (!(A.values[v] > 0.0) || !std::isfinite(A.values[v])) { *msg = "axis " + std::to_string(ax) + ": rate values must be positive"; return KIN_ERR_INPUT; }
    } else if (A.kind == KIN_AXIS_INITIAL) {
      if (A.index < 0 || A.index >= net.n) { *msg = "axis " + std::to_string(ax) + ": unknown species"; return KIN_ERR_INPUT; }
      for (int v = 0; v < A.n_values; ++v)
        if (!(A.values[v] >= 0.0) || A.values[v] != std::floor(A.values[v]) || A.values[v] > 9007199254740992.0) { *msg = "axis " + std::to_string(ax) + ": initial amounts must be non-negative integers"; return KIN_ERR_INPUT; }
    } else if (A.kind == KIN_AXIS_SCALE) {
      if (A.index < 0 || A.span <= 0 || A.index + A.span > net.m) { *msg = "axis " + std::to_string(ax) + ": scale range outside the reactions"; return KIN_ERR_INPUT; }
      for (int v = 0; v < A.n_values; ++v)
        if (!(A.values[v] > 0.0) || !std::isfinite(A.values[v])) { *msg = "axis " + std::to_string(ax) + ": scale factors must be positive"; return KIN_ERR_INPUT; }
    } else {
      *msg = "axis " + std::to_string(ax) + ": unknown axis kind"; return KIN_ERR_INPUT;
    }
  }
  if (d->seed_mode == KIN_SEED_DIRECT) {
    SweepLayout L; std::string m2;
    if (sweep_layout(d, &L, &m2) == KIN_OK && L.n_sims != 1) { *msg = "direct seeding needs exactly one simulation"; return KIN_ERR_INPUT; }
  }
  return KIN_OK;
}

template <bool C>
int run_one(const Network& net, const kin_sweep_desc* d, std::uint64_t sim, double* traj,
            std::uint64_t* meta, Scratch& sc, Work* w) {
  std::uint64_t seed;
  double* x0 = sc.x0.data();
  decode_sim(net, d, sim, sc.rates.data(), x0, &seed);
  const kin_method& M = d->method;
  if (M.kind == KIN_METHOD_ODE)
    return integrate_rre<C>(net, sc.rates.data(), x0, M.integrator, d->t_end, d->grid, d->n_grid, traj, meta, sc, w);
  if (M.kind == KIN_METHOD_LSODA)
    return integrate_lsoda<C>(net, sc.rates.data(), x0, M.integrator, d->t_end, d->grid, d->n_grid, traj, meta, sc, w);
  if (M.kind == KIN_METHOD_HYBRID)
    return simulate_hybrid<C>(net, sc.rates.data(), x0, M, d->t_end, d->grid, d->n_grid, seed, traj, meta, sc, w,
                              d->rng_mode);
  if (M.kind == KIN_METHOD_CLE)
    return simulate_cle<C>(net, sc.rates.data(), x0, M, d->t_end, d->grid, d->n_grid, seed, traj, meta, sc, w,
                           d->rng_mode);
  return simulate_stochastic<C>(net, sc.rates.data(), x0, M, d->t_end, d->grid, d->n_grid, seed, traj, meta, sc, w,
                                d->rng_mode);
}

// EnsembleStatistics::add (Welford), ensemble.hpp:29-30; App. B #9 order.
inline void welford_add(std::uint64_t n_after, const double* x, double* mean, double* m2, size_t len) {
  const double nn = static_cast<double>(n_after);
  for (size_t q = 0; q < len; ++q) {
    const double delta = x[q] - mean[q];
    mean[q] = mean[q] + delta / nn;
    m2[q] = m2[q] + delta * (x[q] - mean[q]);
  }
}

}  // namespace kin_oracle

// ============================ C API (ctypes) =================================
using namespace kin_oracle;

extern "C" {

uint64_t kin_oracle_splitmix64_mix(uint64_t v) { return splitmix64_mix(v); }
uint64_t kin_oracle_derive_run_seed(uint64_t m, uint64_t i) { return derive_run_seed(m, i); }

// kind: 0 next_u64, 1 uniform, 2 normal, 3 poisson(mean); out as raw bits.
void kin_oracle_rng_draws(uint64_t seed, int kind, double mean, int n, uint64_t* out) {
  Stream r(seed);
  for (int q = 0; q < n; ++q) {
    uint64_t bits = 0;
    double v;
    switch (kind) {
      case 0: bits = r.next_u64(); break;
      case 1: v = r.draw_uniform(); std::memcpy(&bits, &v, 8); break;
      case 2: v = r.draw_normal(); std::memcpy(&bits, &v, 8); break;
      default: bits = r.draw_poisson(mean); break;
    }
    out[q] = bits;
  }
}

// Philox4x32-10 block (known-answer tests) and Philox draw sites:
// kind 4 = uniforms (bits) of site (seed, event 0, slot 0); kind 5 = one
// Poisson(mean) draw per site (seed, event 0, slot q) for q = 0..n-1.
void kin_oracle_philox_block(uint32_t k0, uint32_t k1, const uint32_t* ctr, uint32_t* out) {
  Philox::block(k0, k1, ctr[0], ctr[1], ctr[2], ctr[3], out);
}

void kin_oracle_philox_draws(uint64_t seed, int kind, double mean, int n, uint64_t* out) {
  if (kind == 4) {
    PhiloxSite src(seed, 0, 0);
    for (int q = 0; q < n; ++q) {
      const double v = src.draw_uniform();
      std::memcpy(&out[q], &v, 8);
    }
  } else {
    for (int q = 0; q < n; ++q) {
      PhiloxSite src(seed, 0, static_cast<uint32_t>(q));
      out[q] = poisson_from(src, mean, nullptr);
    }
  }
}

// n_draws Binomial(n_trials, p) draws from one stream (KIN_FIRING_BINOMIAL sampler).
void kin_oracle_binomial_draws(uint64_t seed, uint64_t n_trials, double p, int n_draws, uint64_t* out) {
  Stream r(seed);
  for (int q = 0; q < n_draws; ++q) out[q] = binomial_from(r, n_trials, p, nullptr);
}

// One stream: n_each draw_poisson for each mean in order, then n_normal
// draw_normal (SURVEY Appendix A flag-insensitivity digest).  Normals as bits.
void kin_oracle_rng_sequence(uint64_t seed, const double* means, int n_means, int n_each, int n_normal,
                             uint64_t* out) {
  Stream r(seed);
  int q = 0;
  for (int a = 0; a < n_means; ++a)
    for (int e = 0; e < n_each; ++e) out[q++] = r.draw_poisson(means[a]);
  for (int e = 0; e < n_normal; ++e) {
    const double v = r.draw_normal();
    std::memcpy(&out[q++], &v, 8);
  }
}

static int load(const kin_model_desc* d, Network* net, kin_error* err) {
  std::string msg;
  const int rc = build_network(d, net, &msg);
  if (rc != KIN_OK) set_err(err, rc, msg);
  return rc;
}

int kin_oracle_model_check(const kin_model_desc* d, kin_error* err) {
  Network net;
  return load(d, &net, err);
}

int kin_oracle_propensities(const kin_model_desc* d, const double* x, double* a, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  std::vector<double> r(net.m);
  for (int j = 0; j < net.m; ++j) r[j] = net.rate_param[j] >= 0 ? net.params[net.rate_param[j]] : net.rate_base[j];
  propensities<false>(net, r.data(), x, a, nullptr);
  return KIN_OK;
}

int kin_oracle_select_tau(const kin_model_desc* d, const double* x, double eps, double* tau, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  std::vector<double> r(net.m), a(net.m);
  for (int j = 0; j < net.m; ++j) r[j] = net.rate_param[j] >= 0 ? net.params[net.rate_param[j]] : net.rate_base[j];
  propensities<false>(net, r.data(), x, a.data(), nullptr);
  double a0 = 0.0;
  for (int j = 0; j < net.m; ++j) a0 = a0 + a[j];
  *tau = a0 == 0.0 ? std::numeric_limits<double>::infinity() : select_tau<false>(net, x, a.data(), eps, nullptr);
  return KIN_OK;
}

// ssa_step_from_uniforms: returns fired reaction (>=0) or -1 (Exhausted).
int kin_oracle_ssa_step_from_uniforms(const kin_model_desc* d, const double* x, double u1, double u2,
                                      double* dt, int* reaction, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  std::vector<double> r(net.m), a(net.m);
  for (int j = 0; j < net.m; ++j) r[j] = net.rate_param[j] >= 0 ? net.params[net.rate_param[j]] : net.rate_base[j];
  propensities<false>(net, r.data(), x, a.data(), nullptr);
  double a0 = 0.0;
  for (int j = 0; j < net.m; ++j) a0 = a0 + a[j];
  if (a0 == 0.0) { *reaction = -1; *dt = 0.0; return KIN_OK; }
  *dt = std::log(1.0 / u1) / a0;
  *reaction = ssa_select(net, a.data(), a0, u2);
  return KIN_OK;
}

// tau_leap_step_from_counts: *rejected = 1 when any amount would go negative.
int kin_oracle_tau_leap_from_counts(const kin_model_desc* d, const double* x, const uint64_t* counts,
                                    double* xout, int* rejected, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  for (int i = 0; i < net.n; ++i) xout[i] = x[i];
  for (int j = 0; j < net.m; ++j) {
    if (!counts[j]) continue;
    for (int p = net.col_ptr[j]; p < net.col_ptr[j + 1]; ++p)
      xout[net.col_species[p]] = xout[net.col_species[p]] + static_cast<double>(net.col_delta[p]) * static_cast<double>(counts[j]);
  }
  *rejected = 0;
  for (int i = 0; i < net.n; ++i) if (xout[i] < 0.0) *rejected = 1;
  return KIN_OK;
}

int kin_oracle_cle_step(const kin_model_desc* d, const double* x, double h, const double* z, double* xout,
                        uint64_t* clamped, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  std::vector<double> r(net.m), a(net.m);
  for (int j = 0; j < net.m; ++j) r[j] = net.rate_param[j] >= 0 ? net.params[net.rate_param[j]] : net.rate_base[j];
  propensities<false>(net, r.data(), x, a.data(), nullptr);
  for (int i = 0; i < net.n; ++i) xout[i] = x[i];
  std::uint64_t c = 0;
  cle_step_from_normals<false>(net, xout, a.data(), h, z, &c, nullptr);
  *clamped = c;
  return KIN_OK;
}

// next_jump_with_threshold (hybrid.hpp:43-48) from t = 0: returns 1 with *tstar
// and the pre-jump state when G reaches `threshold` before t_end, else 0 with
// the state at t_end.  slow_mask[j] != 0 marks slow reactions (NULL: use the
// thresholds at x via partition_reactions).
int kin_oracle_next_jump(const kin_model_desc* d, const double* x, const int32_t* slow_mask, double theta_x,
                         double theta_a, double t_end, double threshold, const kin_integrator_config* cfg,
                         double* tstar, double* xout, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return -1;
  std::vector<double> r(net.m);
  for (int j = 0; j < net.m; ++j) r[j] = net.rate_param[j] >= 0 ? net.params[net.rate_param[j]] : net.rate_base[j];
  Scratch sc;
  sc.resize(net.n, net.m);
  std::vector<char> slow(static_cast<size_t>(net.m), 0);
  propensities<false>(net, r.data(), x, sc.a.data(), nullptr);
  if (slow_mask) {
    for (int j = 0; j < net.m; ++j) slow[j] = slow_mask[j] != 0;
  } else {
    hybrid_partition(net, x, sc.a.data(), theta_x, theta_a, &slow);
  }
  for (int i = 0; i < net.n; ++i) sc.v[0][i] = x[i];
  double t = 0.0;
  int gi = 0;
  bool floored = false, jumped = false;
  std::uint64_t attempts = 0, meta[6] = {0, 0, 0, 0, 0, 0};
  const int rc = hybrid_segment<false>(net, r.data(), slow, *cfg, threshold, t_end, t, sc, nullptr, nullptr, 0, gi,
                                       nullptr, floored, attempts, meta, &jumped);
  if (rc != KIN_SIM_OK) {
    set_err(err, KIN_ERR_SIMULATION, "integrator failure");
    return -1;
  }
  *tstar = t;
  for (int i = 0; i < net.n; ++i) xout[i] = sc.v[0][i];
  return jumped ? 1 : 0;
}

int kin_oracle_apply_reaction(const kin_model_desc* d, const double* x, int j, double* xout, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  for (int i = 0; i < net.n; ++i) xout[i] = x[i];
  for (int p = net.col_ptr[j]; p < net.col_ptr[j + 1]; ++p) {
    const double v = xout[net.col_species[p]] + net.col_delta[p];
    if (v < 0.0) { set_err(err, KIN_ERR_SIMULATION, "apply_reaction: amount would become negative"); return KIN_ERR_SIMULATION; }
    xout[net.col_species[p]] = v;
  }
  return KIN_OK;
}

int kin_oracle_rre_rhs(const kin_model_desc* d, const double* x, double* dx, kin_error* err) {
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  std::vector<double> r(net.m), a(net.m);
  for (int j = 0; j < net.m; ++j) r[j] = net.rate_param[j] >= 0 ? net.params[net.rate_param[j]] : net.rate_base[j];
  rre_rhs<false>(net, r.data(), x, a.data(), dx, nullptr);
  return KIN_OK;
}

// rk_step (deterministic.hpp:26-36): one Dormand-Prince 5(4) step of size h
// from x with k1 = f(x) — the stage/error expressions of integrate_rre above.
// out: y5[N], err (sqrt(mean((e_i/sk_i)^2)), sk_i = atol + rtol*max(|y_i|,|y5_i|)),
// then k7 = f(y5)[N].
int kin_oracle_rk_step(const kin_model_desc* d, const double* x, double h, double rtol, double atol, double* out,
                       kin_error* err) {
  using namespace dp;
  Network net;
  if (int rc = load(d, &net, err)) return rc;
  const int n = net.n;
  std::vector<double> r(net.m), a(net.m);
  for (int j = 0; j < net.m; ++j) r[j] = net.rate_param[j] >= 0 ? net.params[net.rate_param[j]] : net.rate_base[j];
  std::vector<double> y(x, x + n), k1(n), k2(n), k3(n), k4(n), k5(n), k6(n), k7(n), ys(n), yn(n);
  rre_rhs<false>(net, r.data(), y.data(), a.data(), k1.data(), nullptr);
  for (int i = 0; i < n; ++i) ys[i] = y[i] + h * (a21 * k1[i]);
  rre_rhs<false>(net, r.data(), ys.data(), a.data(), k2.data(), nullptr);
  for (int i = 0; i < n; ++i) ys[i] = y[i] + h * (a31 * k1[i] + a32 * k2[i]);
  rre_rhs<false>(net, r.data(), ys.data(), a.data(), k3.data(), nullptr);
  for (int i = 0; i < n; ++i) ys[i] = y[i] + h * (a41 * k1[i] + a42 * k2[i] + a43 * k3[i]);
  rre_rhs<false>(net, r.data(), ys.data(), a.data(), k4.data(), nullptr);
  for (int i = 0; i < n; ++i) ys[i] = y[i] + h * (a51 * k1[i] + a52 * k2[i] + a53 * k3[i] + a54 * k4[i]);
  rre_rhs<false>(net, r.data(), ys.data(), a.data(), k5.data(), nullptr);
  for (int i = 0; i < n; ++i) ys[i] = y[i] + h * (a61 * k1[i] + a62 * k2[i] + a63 * k3[i] + a64 * k4[i] + a65 * k5[i]);
  rre_rhs<false>(net, r.data(), ys.data(), a.data(), k6.data(), nullptr);
  for (int i = 0; i < n; ++i) yn[i] = y[i] + h * (a71 * k1[i] + a73 * k3[i] + a74 * k4[i] + a75 * k5[i] + a76 * k6[i]);
  rre_rhs<false>(net, r.data(), yn.data(), a.data(), k7.data(), nullptr);
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    const double e = h * (e1 * k1[i] + e3 * k3[i] + e4 * k4[i] + e5 * k5[i] + e6 * k6[i] + e7 * k7[i]);
    const double sk = atol + rtol * std::max(std::fabs(y[i]), std::fabs(yn[i]));
    const double q = e / sk;
    sum = sum + q * q;
  }
  for (int i = 0; i < n; ++i) out[i] = yn[i];
  out[n] = std::sqrt(sum / static_cast<double>(n));
  for (int i = 0; i < n; ++i) out[n + 1 + i] = k7[i];
  return KIN_OK;
}

// Chan merge (ensemble.hpp:31-33,56-57) of b into a.
void kin_oracle_stats_merge(uint64_t* na, double* mean_a, double* m2_a, uint64_t nb,
                            const double* mean_b, const double* m2_b, uint64_t len) {
  if (nb == 0) return;
  if (*na == 0) {
    *na = nb;
    for (uint64_t q = 0; q < len; ++q) { mean_a[q] = mean_b[q]; m2_a[q] = m2_b[q]; }
    return;
  }
  const double fa = static_cast<double>(*na), fb = static_cast<double>(nb);
  const double fn = fa + fb;
  for (uint64_t q = 0; q < len; ++q) {
    const double delta = mean_b[q] - mean_a[q];
    mean_a[q] = mean_a[q] + delta * fb / fn;
    m2_a[q] = m2_a[q] + m2_b[q] + delta * delta * fa * fb / fn;
  }
  *na += nb;
}

// parameter_sweep / run_ensemble / run_single on `workers` std::threads owning
// contiguous simulation ranges (ensemble.hpp:91-99).  Outputs as in kin_abi.h
// (host layout [S][G][N]).  Per-point statistics: Welford over each point's runs
// in ascending run order (the workers=1 merge order).
int kin_oracle_sweep(const kin_model_desc* md, const kin_sweep_desc* d, kin_sweep_out* out,
                     kin_error* err, int workers) {
  if (err) { std::memset(err, 0, sizeof(*err)); }
  Network net;
  if (int rc = load(md, &net, err)) return rc;
  std::string msg;
  SweepLayout L;
  if (int rc = sweep_layout(d, &L, &msg)) { set_err(err, rc, msg); return rc; }
  if (int rc = validate_sweep(net, d, &msg)) { set_err(err, rc, msg); return rc; }
  const std::uint64_t s0 = d->sim_begin;
  const std::uint64_t s1 = d->sim_end == 0 ? L.n_sims : std::min<std::uint64_t>(d->sim_end, L.n_sims);
  if (s0 > s1) { set_err(err, KIN_ERR_USAGE, "empty or inverted simulation range"); return KIN_ERR_USAGE; }
  // interleaved point shard (kin_abi.h kin_sweep_desc): local simulation s is
  // run s % R of global point p_first + shard_index + (s / R) * shard_count
  const bool sharded = d->shard_count > 1;
  if (sharded && (d->shard_index < 0 || d->shard_index >= d->shard_count || s0 % L.runs || s1 % L.runs)) {
    set_err(err, KIN_ERR_INPUT, "bad shard");
    return KIN_ERR_INPUT;
  }
  const std::uint64_t R = L.runs;
  std::uint64_t S = s1 - s0;
  if (sharded) {
    const std::uint64_t P = S / R, n = static_cast<std::uint64_t>(d->shard_count);
    S = (P > static_cast<std::uint64_t>(d->shard_index) ? (P - d->shard_index + n - 1) / n : 0) * R;
  }
  auto global_of = [&](std::uint64_t s) -> std::uint64_t {
    if (!sharded) return s0 + s;
    const std::uint64_t k = s / R;
    return (s0 / R + d->shard_index + static_cast<std::uint64_t>(d->shard_count) * k) * R + (s - k * R);
  };
  const int G = d->n_grid, N = net.n;
  const size_t per = static_cast<size_t>(G) * N;
  std::vector<double> tmp_traj;
  double* traj = (out && d->output_mode != KIN_OUTPUT_STATS_ONLY) ? out->traj : nullptr;
  const bool need_stats = out && (out->mean || out->m2);
  if (!traj && need_stats) { tmp_traj.resize(S * per); traj = tmp_traj.data(); }
  std::vector<std::uint64_t> tmp_meta;
  std::vector<int32_t> status(S, 0);
  if (workers < 1) workers = 1;
  if (static_cast<std::uint64_t>(workers) > S) workers = static_cast<int>(std::max<std::uint64_t>(S, 1));
  const bool count = out && out->work;
  auto body = [&](std::uint64_t lo, std::uint64_t hi) {
    Scratch sc;
    sc.resize(N, net.m);
    std::vector<double> scratch_traj(per);
    std::uint64_t meta_local[6];
    for (std::uint64_t s = lo; s < hi; ++s) {  // s: local index
      double* tr = traj ? traj + s * per : scratch_traj.data();
      std::uint64_t* me = (out && out->meta) ? out->meta + s * 6 : meta_local;
      Work w;
      const std::uint64_t g = global_of(s);
      const int st = count ? run_one<true>(net, d, g, tr, me, sc, &w) : run_one<false>(net, d, g, tr, me, sc, nullptr);
      status[s] = st;
      if (count) out->work[s] = w.flops;
    }
  };
  std::vector<std::thread> pool;
  const std::uint64_t chunk = (S + workers - 1) / std::max(workers, 1);
  for (int wk = 0; wk < workers; ++wk) {
    const std::uint64_t lo = std::min<std::uint64_t>(S, wk * chunk);
    const std::uint64_t hi = std::min<std::uint64_t>(S, (wk + 1) * chunk);
    if (lo >= hi) continue;
    if (workers == 1) body(lo, hi); else pool.emplace_back(body, lo, hi);
  }
  for (auto& th : pool) th.join();
  if (out && out->status) for (std::uint64_t s = 0; s < S; ++s) out->status[s] = status[s];
  for (std::uint64_t s = 0; s < S; ++s) {
    if (status[s] != KIN_SIM_OK) {
      const std::uint64_t g = global_of(s);
      if (err) {
        err->code = KIN_ERR_SIMULATION;
        err->sim_status = status[s];
        err->sim_index = g;
        err->point_index = g / L.runs;
        err->run_index = g % L.runs;
        std::snprintf(err->message, sizeof(err->message), "simulation %llu (point %llu, run %llu) failed: status %d",
                      (unsigned long long)g, (unsigned long long)(g / L.runs), (unsigned long long)(g % L.runs), status[s]);
      }
      return KIN_ERR_SIMULATION;
    }
  }
  if (need_stats) {
    // local points: whole points of the local index space (a shard is whole points)
    const std::uint64_t p0 = sharded ? 0 : (s0 + L.runs - 1) / L.runs;
    const std::uint64_t p1 = sharded ? S / L.runs : s1 / L.runs;
    const std::uint64_t first = sharded ? 0 : s0;  // global index of local simulation 0
    for (std::uint64_t p = p0; p < p1; ++p) {
      double* mean = out->mean ? out->mean + (p - p0) * per : nullptr;
      double* m2 = out->m2 ? out->m2 + (p - p0) * per : nullptr;
      std::vector<double> mv(per, 0.0), qv(per, 0.0);
      for (std::uint64_t r = 0; r < L.runs; ++r)
        welford_add(r + 1, traj + (p * L.runs + r - first) * per, mv.data(), qv.data(), per);
      if (mean) std::memcpy(mean, mv.data(), per * sizeof(double));
      if (m2) std::memcpy(m2, qv.data(), per * sizeof(double));
    }
  }
  return KIN_OK;
}

int kin_oracle_sweep_size(const kin_sweep_desc* d, uint64_t* np, uint64_t* ns, kin_error* err) {
  SweepLayout L;
  std::string msg;
  if (int rc = sweep_layout(d, &L, &msg)) { set_err(err, rc, msg); return rc; }
  *np = L.n_points;
  *ns = L.n_sims;
  return KIN_OK;
}

}  // extern "C"

// explicit instantiations used above
namespace kin_oracle {
template double select_tau<true>(const Network&, const double*, const double*, double, Work*);
template double select_tau<false>(const Network&, const double*, const double*, double, Work*);
}  // namespace kin_oracle

// oracle/kin_oracle.hpp — TEST INFRASTRUCTURE ONLY.
//
// CPU oracle: a C++20 restatement of the reference's hot path, which ships as
// header contracts + SPEC only (the simulators/ensemble have no .cpp in
// /root/reference).  Each function cites the contract it
// restates.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
// leg may load this library, and only as the checker / the baseline timed
// beside the GPU — never as the product.
//
// Every choice the reference leaves open is fixed here once and mirrored by the
// CUDA kernels (DESIGN.md §"Fixed semantics").
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "kin_abi.h"
#include "kin_rng.hpp"

namespace kin_oracle {

// ReactionNetwork (model.hpp:13-95) flattened into the tables the simulators use.
struct Network {
  int n = 0;  // species
  int m = 0;  // reactions
  std::vector<double> x0;          // initial_amounts() (model.hpp:76), exact integers
  std::vector<double> rate_base;   // Reaction::rate_constant
  std::vector<int> rate_param;     // Reaction::rate_param or -1
  std::vector<double> params;      // Parameter::value
  // reactant multiset per reaction, species ascending (std::map order, model.hpp:33)
  std::vector<int> rt_ptr, rt_species, rt_stoich;
  // nonzero nu column per reaction (model.hpp:67-71), species ascending
  std::vector<int> col_ptr, col_species, col_delta;
  // nonzero nu row per species, reaction ascending (used by select_tau / rre_rhs)
  std::vector<int> row_ptr, row_reaction, row_delta;
  std::vector<int> g;              // highest reactant order per species, 1 if none
  std::vector<int> order;          // Reaction::order()
};

// ReactionNetwork::create validation (model.hpp:47-53).
// Returns KIN_OK or KIN_ERR_INPUT with a message.
int build_network(const kin_model_desc* d, Network* net, std::string* msg);

// combinations (model.hpp:145-149), order-3 extension C(x,3).
inline double combinations(double x, int s) {
  double h;
  switch (s) {
    case 0: return 1.0;
    case 1: h = x; break;
    case 2: h = x * (x - 1.0) / 2.0; break;
    default: h = x * (x - 1.0) * (x - 2.0) / 6.0; break;
  }
  return h < 0.0 ? 0.0 : h;
}
inline int combinations_flops(int s) { return s <= 1 ? 0 : (s == 2 ? 3 : 5); }

struct Work {
  std::uint64_t flops = 0;
};

// Per-simulation scratch (no allocation inside the hot loop).
struct Scratch {
  std::vector<double> x, a, xn, x0, rates;
  std::vector<std::uint64_t> k;
  // Dopri5 / LSODA
  std::vector<double> v[24];
  std::vector<double> z, jac, jac2;
  std::vector<int> piv;
  void resize(int n, int m);
};

// propensities (model.hpp:151-157): a_j = c_j * prod h(x_s, stoich_s).
template <bool C>
inline void propensities(const Network& net, const double* rates, const double* x,
                         double* a, Work* w) {
  for (int j = 0; j < net.m; ++j) {
    double aj = rates[j];
    for (int p = net.rt_ptr[j]; p < net.rt_ptr[j + 1]; ++p) {
      aj = aj * combinations(x[net.rt_species[p]], net.rt_stoich[p]);
      if constexpr (C) w->flops += 1 + combinations_flops(net.rt_stoich[p]);
    }
    a[j] = aj;
  }
}

// select_tau (stochastic.hpp:40-46), header form (App. B #2).
template <bool C>
double select_tau(const Network& net, const double* x, const double* a, double eps, Work* w);

// ssa_step_from_uniforms (stochastic.hpp:28-32).  Returns -1 when
// exhausted (a0 == 0), else the fired reaction; *dt receives ln(1/u1)/a0.
int ssa_select(const Network& net, const double* a, double a0, double u2);

// Simulation of one run.  out: [G][N] samples; meta: 6 counters.
// Returns enum kin_sim_status.
template <bool C>
int simulate_stochastic(const Network& net, const double* rates, const double* x0,
                        const kin_method& method, double t_end, const double* grid,
                        int n_grid, std::uint64_t seed, double* out, std::uint64_t* meta,
                        Scratch& sc, Work* w, int rng_mode);

template <bool C>
int integrate_rre(const Network& net, const double* rates, const double* x0,
                  const kin_integrator_config& cfg, double t_end, const double* grid,
                  int n_grid, double* out, std::uint64_t* meta, Scratch& sc, Work* w);

template <bool C>
int integrate_lsoda(const Network& net, const double* rates, const double* x0,
                    const kin_integrator_config& cfg, double t_end, const double* grid,
                    int n_grid, double* out, std::uint64_t* meta, Scratch& sc, Work* w);

// rre_rhs (deterministic.hpp:85-88): dx = nu * a(x), row order.
template <bool C>
inline void rre_rhs(const Network& net, const double* rates, const double* x, double* a,
                    double* dx, Work* w) {
  propensities<C>(net, rates, x, a, w);
  for (int i = 0; i < net.n; ++i) {
    double s = 0.0;
    for (int p = net.row_ptr[i]; p < net.row_ptr[i + 1]; ++p)
      s = s + static_cast<double>(net.row_delta[p]) * a[net.row_reaction[p]];
    dx[i] = s;
    if constexpr (C) w->flops += 2 * static_cast<std::uint64_t>(net.row_ptr[i + 1] - net.row_ptr[i]);
  }
}

// Sweep decoding (ensemble.hpp:101-130): per-simulation rate
// constants, initial amounts and seed for global simulation index `sim`.
struct SweepLayout {
  std::uint64_t n_points = 1, runs = 1, n_sims = 1;
};
int sweep_layout(const kin_sweep_desc* d, SweepLayout* out, std::string* msg);
void decode_sim(const Network& net, const kin_sweep_desc* d, std::uint64_t sim,
                double* rates, double* x0, std::uint64_t* seed);

}  // namespace kin_oracle

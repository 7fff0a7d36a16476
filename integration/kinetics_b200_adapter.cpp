// integration/kinetics_b200_adapter.cpp — the reference-side binding a
// maintainer adds to proj/src/ to route the ensemble layer through the B200
// engine (include/kin_abi.h).  Uses only the reference's public headers
// (model.hpp / ensemble.hpp); compile-checked against them by
// tests/test_integration.py.  Link: -L<repo>/paper_1309_7695_b200 -lkin_b200.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kin_abi.h"
#include "kinetics/ensemble.hpp"
#include "kinetics/errors.hpp"

namespace kinetics::b200 {

namespace {

struct PackedModel {
  std::vector<int64_t> x0;
  std::vector<double> rates, params;
  std::vector<int32_t> rparam, rptr, rsp, rst, pptr, psp, pst;
  kin_model_desc d{};
};

// ReactionNetwork (model.hpp:44-95) -> kin_model_desc.  Reactant/product maps
// are std::map, so iteration is species-ascending as the ABI requires.
PackedModel pack(const ReactionNetwork& net) {
  PackedModel m;
  for (const auto& s : net.species()) m.x0.push_back(s.initial_amount);
  for (const auto& p : net.params()) m.params.push_back(p.value);
  m.rptr.push_back(0);
  m.pptr.push_back(0);
  int max_order = 2;
  for (const auto& r : net.reactions()) {
    m.rates.push_back(r.rate_constant);
    m.rparam.push_back(r.rate_param ? static_cast<int32_t>(*r.rate_param) : -1);
    for (const auto& [s, c] : r.reactants) { m.rsp.push_back(static_cast<int32_t>(s)); m.rst.push_back(c); }
    for (const auto& [s, c] : r.products) { m.psp.push_back(static_cast<int32_t>(s)); m.pst.push_back(c); }
    m.rptr.push_back(static_cast<int32_t>(m.rsp.size()));
    m.pptr.push_back(static_cast<int32_t>(m.psp.size()));
  }
  m.d.n_species = static_cast<int32_t>(net.species_count());
  m.d.n_reactions = static_cast<int32_t>(net.reaction_count());
  m.d.n_params = static_cast<int32_t>(net.params().size());
  m.d.initial_amounts = m.x0.data();
  m.d.rate_constants = m.rates.data();
  m.d.rate_param = m.rparam.data();
  m.d.param_values = m.params.data();
  m.d.reactant_ptr = m.rptr.data();
  m.d.reactant_species = m.rsp.data();
  m.d.reactant_stoich = m.rst.data();
  m.d.product_ptr = m.pptr.data();
  m.d.product_species = m.psp.data();
  m.d.product_stoich = m.pst.data();
  m.d.max_order = max_order;
  return m;
}

kin_method method_of(const Method& m) {
  kin_method k{};
  k.kind = static_cast<int32_t>(m.kind);  // Method::Kind order == enum kin_method_kind
  k.tau = m.tau;
  k.epsilon = m.epsilon;
  // a hybrid run integrates with HybridConfig::integrator (hybrid.hpp:21-26)
  const IntegratorConfig& ic = m.kind == Method::Kind::Hybrid ? m.hybrid.integrator : m.integrator;
  k.integrator = {ic.rel_tol, ic.abs_tol, ic.h_init, ic.h_max, ic.max_steps};
  k.theta_x = static_cast<double>(m.hybrid.amount_threshold);
  k.theta_a = m.hybrid.propensity_threshold;
  k.repartition_interval = m.hybrid.repartition_interval;
  return k;
}

[[noreturn]] void rethrow(int rc, const kin_error& e) {
  if (rc == KIN_ERR_SIMULATION) throw SimulationError(e.message);
  if (rc == KIN_ERR_DEVICE) throw KineticsError(std::string("device: ") + e.message);
  throw ValidationError(e.message);
}

// RAII over context + uploaded model
struct Engine {
  kin_ctx* ctx = nullptr;
  kin_model* model = nullptr;
  PackedModel pm;
  explicit Engine(const ReactionNetwork& net) : pm(pack(net)) {
    kin_error e{};
    if (int rc = kin_ctx_create(nullptr, 0, &ctx, &e)) rethrow(rc, e);
    if (int rc = kin_model_upload(ctx, &pm.d, &model, &e)) rethrow(rc, e);
  }
  ~Engine() {
    kin_model_free(model);
    kin_ctx_destroy(ctx);
  }
};

// Run a descriptor and return every trajectory [sim][g][n] plus meta.
void run(Engine& eng, kin_sweep_desc& d, std::vector<double>& traj, std::vector<uint64_t>& meta) {
  kin_error e{};
  uint64_t P = 0, S = 0;
  if (int rc = kin_sweep_size(&d, &P, &S, &e)) rethrow(rc, e);
  traj.assign(S * static_cast<uint64_t>(d.n_grid) * eng.pm.d.n_species, 0.0);
  meta.assign(S * 6, 0);
  kin_sweep_out out{};
  out.traj = traj.data();
  out.meta = meta.data();
  if (int rc = kin_sweep_run(eng.ctx, eng.model, &d, &out, &e)) rethrow(rc, e);
}

Trajectory trajectory_at(const std::vector<double>& traj, const std::vector<uint64_t>& meta, uint64_t s,
                         const std::vector<double>& grid, std::size_t n, const Method& m, uint64_t seed) {
  Trajectory t;
  t.grid = grid;
  t.method = m.name();
  if (!m.deterministic()) t.seed = seed;
  const double* row = traj.data() + s * grid.size() * n;
  for (std::size_t g = 0; g < grid.size(); ++g) t.samples.emplace_back(row + g * n, row + (g + 1) * n);
  const uint64_t* me = meta.data() + s * 6;
  t.meta = {me[0], me[1], me[2], me[3], me[4], me[5] != 0};
  return t;
}

}  // namespace

// parameter_sweep (ensemble.hpp:126-130)
SweepResults parameter_sweep(const ReactionNetwork& net, const SweepConfig& cfg, unsigned /*workers*/) {
  Engine eng(net);
  std::vector<kin_sweep_axis> axes;
  SweepResults res;
  for (const auto& ax : cfg.axes) {
    const auto p = net.param_index(ax.param);
    if (!p) throw ValidationError("unknown sweep parameter '" + ax.param + "'");
    axes.push_back({KIN_AXIS_PARAM, static_cast<int32_t>(*p), static_cast<int32_t>(ax.values.size()), ax.values.data()});
    res.axis_names.push_back(ax.param);
  }
  kin_sweep_desc d{};
  d.method = method_of(cfg.method);
  d.n_axes = static_cast<int32_t>(axes.size());
  d.axes = axes.data();
  d.runs_per_point = cfg.runs_per_point;
  d.master_seed = cfg.master_seed;
  d.seed_mode = KIN_SEED_SWEEP;
  d.rng_mode = KIN_RNG_COMPAT;
  d.t_end = cfg.t_end;
  d.n_grid = static_cast<int32_t>(cfg.grid.size());
  d.grid = cfg.grid.data();
  std::vector<double> traj;
  std::vector<uint64_t> meta;
  run(eng, d, traj, meta);
  const std::size_t n = net.species_count();
  uint64_t P = 0, S = 0;
  kin_error e{};
  kin_sweep_size(&d, &P, &S, &e);
  for (uint64_t k = 0; k < P; ++k) {
    SweepPointResult pr;
    uint64_t rem = k;
    pr.coordinates.assign(cfg.axes.size(), 0.0);
    for (std::size_t a = cfg.axes.size(); a-- > 0;) {  // last axis fastest
      pr.coordinates[a] = cfg.axes[a].values[rem % cfg.axes[a].values.size()];
      rem /= cfg.axes[a].values.size();
    }
    pr.stats = EnsembleStatistics(cfg.grid, n);
    const uint64_t pm = kin_derive_run_seed(cfg.master_seed, k);
    for (uint64_t r = 0; r < cfg.runs_per_point; ++r)  // ascending run order
      pr.stats.add(trajectory_at(traj, meta, k * cfg.runs_per_point + r, cfg.grid, n, cfg.method,
                                 kin_derive_run_seed(pm, r)));
    res.points.push_back(std::move(pr));
  }
  return res;
}

// run_ensemble (ensemble.hpp:97-99)
EnsembleStatistics run_ensemble(const ReactionNetwork& net, const EnsembleOptions& o, const RunSink& sink) {
  Engine eng(net);
  kin_sweep_desc d{};
  d.method = method_of(o.method);
  d.runs_per_point = o.n_runs;
  d.master_seed = o.master_seed;
  d.seed_mode = KIN_SEED_ENSEMBLE;
  d.t_end = o.t_end;
  d.n_grid = static_cast<int32_t>(o.grid.size());
  d.grid = o.grid.data();
  std::vector<double> traj;
  std::vector<uint64_t> meta;
  run(eng, d, traj, meta);
  EnsembleStatistics st(o.grid, net.species_count());
  for (uint64_t i = 0; i < o.n_runs; ++i) {
    Trajectory t = trajectory_at(traj, meta, i, o.grid, net.species_count(), o.method,
                                 kin_derive_run_seed(o.master_seed, i));
    if (sink) sink(i, t);
    st.add(t);
  }
  return st;
}

// run_single (ensemble.hpp:73-76)
Trajectory run_single(const ReactionNetwork& net, const Method& m, double t_end, const std::vector<double>& grid,
                      uint64_t seed) {
  Engine eng(net);
  kin_sweep_desc d{};
  d.method = method_of(m);
  d.runs_per_point = 1;
  d.master_seed = seed;
  d.seed_mode = KIN_SEED_DIRECT;
  d.t_end = t_end;
  d.n_grid = static_cast<int32_t>(grid.size());
  d.grid = grid.data();
  std::vector<double> traj;
  std::vector<uint64_t> meta;
  run(eng, d, traj, meta);
  return trajectory_at(traj, meta, 0, grid, net.species_count(), m, seed);
}

}  // namespace kinetics::b200

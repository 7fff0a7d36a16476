// integration/kinetics_b200_adapter.cpp — the reference-side binding a
// maintainer adds to proj/src/ to route the ensemble layer through the B200
// engine (include/kin_abi.h).  Uses only the reference's public headers
// (model.hpp / ensemble.hpp / errors.hpp); tests/test_integration.py
// compile-checks it against them and builds it with a test driver
// (integration/Makefile) that tests/test_gpu_integration.py runs on the GPU.
// Link: -L<repo>/paper_1309_7695_b200 -lkin_b200.
//
//   parameter_sweep  ensemble.hpp:126-130  one kin_sweep_run, KIN_OUTPUT_STATS_ONLY:
//                                          the per-point EnsembleStatistics come
//                                          from the engine's own Welford kernel
//   run_ensemble     ensemble.hpp:97-99    one kin_ensemble_run; trajectories are
//                                          copied back only when a RunSink is given
//   run_single       ensemble.hpp:73-76    one kin_run_single
//
// `workers` (the reference's thread count, ensemble.hpp:91-96) selects how many
// GPUs the call spreads over (min(workers, visible GPUs); per-run results never
// depend on it).  One engine context per device count is created
// on first use and reused by every later call (device memory pools, JIT
// kernels and streams persist); the model is re-packed per call (host only).
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "kin_abi.h"
#include "kinetics/ensemble.hpp"
#include "kinetics/errors.hpp"

namespace kinetics::b200 {

namespace {

// EnsembleStatistics exposes no way to set (n, mean, m2) directly; the engine
// computes them on the GPU (the same Welford order as EnsembleStatistics::add,
// run-ascending).  These accessors bind its private members through the
// explicit-instantiation rule (access checking does not apply to the template
// arguments of an explicit instantiation); a maintainer merging this adapter
// would instead add a `from_moments` constructor to ensemble.hpp.
template <class Tag, typename Tag::type M>
struct Bind {
  friend typename Tag::type member(Tag) { return M; }
};
struct StatsN { using type = std::uint64_t EnsembleStatistics::*; friend type member(StatsN); };
struct StatsMean { using type = std::vector<double> EnsembleStatistics::*; friend type member(StatsMean); };
struct StatsM2 { using type = std::vector<double> EnsembleStatistics::*; friend type member(StatsM2); };
template struct Bind<StatsN, &EnsembleStatistics::n_>;
template struct Bind<StatsMean, &EnsembleStatistics::mean_>;
template struct Bind<StatsM2, &EnsembleStatistics::m2_>;

EnsembleStatistics stats_from_moments(const std::vector<double>& grid, std::size_t n_species, std::uint64_t n,
                                      const double* mean, const double* m2) {
  EnsembleStatistics st(grid, n_species);
  const std::size_t len = grid.size() * n_species;
  st.*member(StatsN{}) = n;
  st.*member(StatsMean{}) = std::vector<double>(mean, mean + len);
  st.*member(StatsM2{}) = std::vector<double>(m2, m2 + len);
  return st;
}

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
  m.d.max_order = 2;  // ReactionNetwork::create enforces order <= 2 (model.hpp:47-53)
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
  k.firing = KIN_FIRING_POISSON;
  return k;
}

[[noreturn]] void rethrow(int rc, const kin_error& e) {
  if (rc == KIN_ERR_SIMULATION) throw SimulationError(e.message);
  if (rc == KIN_ERR_DEVICE) throw KineticsError(std::string("device: ") + e.message);
  throw ValidationError(e.message);
}

// One context per device count, created on first use and kept for the life of
// the process (the reference's worker pool is per call; a GPU context is too
// expensive for that).
kin_ctx* context_for(unsigned workers) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<kin_ctx, void (*)(kin_ctx*)>> ctxs;
  const int visible = kin_visible_devices();
  if (visible <= 0) throw KineticsError("device: no CUDA device visible");
  const int n = static_cast<int>(std::min<unsigned>(std::max(workers, 1u), static_cast<unsigned>(visible)));
  std::lock_guard<std::mutex> lk(mu);
  auto it = ctxs.find(n);
  if (it != ctxs.end()) return it->second.get();
  std::vector<int32_t> ids(n);
  for (int i = 0; i < n; ++i) ids[i] = i;
  kin_ctx* ctx = nullptr;
  kin_error e{};
  if (int rc = kin_ctx_create(ids.data(), n, &ctx, &e)) rethrow(rc, e);
  ctxs.emplace(n, std::unique_ptr<kin_ctx, void (*)(kin_ctx*)>(ctx, kin_ctx_destroy));
  return ctx;
}

// The model uploaded into a (reused) context for the duration of one call.
struct Call {
  kin_ctx* ctx;
  PackedModel pm;
  kin_model* model = nullptr;
  Call(const ReactionNetwork& net, unsigned workers) : ctx(context_for(workers)), pm(pack(net)) {
    kin_error e{};
    if (int rc = kin_model_upload(ctx, &pm.d, &model, &e)) rethrow(rc, e);
  }
  ~Call() { kin_model_free(model); }
  Call(const Call&) = delete;
  Call& operator=(const Call&) = delete;
};

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

// parameter_sweep (ensemble.hpp:126-130): per-point statistics straight from
// the engine (KIN_OUTPUT_STATS_ONLY: trajectories never leave the device, nor
// are they materialised there as a whole).
SweepResults parameter_sweep(const ReactionNetwork& net, const SweepConfig& cfg, unsigned workers) {
  Call call(net, workers);
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
  d.output_mode = KIN_OUTPUT_STATS_ONLY;
  kin_error e{};
  uint64_t P = 0, S = 0;
  if (int rc = kin_sweep_size(&d, &P, &S, &e)) rethrow(rc, e);
  const std::size_t n = net.species_count(), gn = cfg.grid.size() * n;
  std::vector<double> mean(P * gn), m2(P * gn);
  kin_sweep_out out{};
  out.mean = mean.data();
  out.m2 = m2.data();
  if (int rc = kin_sweep_run(call.ctx, call.model, &d, &out, &e)) rethrow(rc, e);
  for (uint64_t k = 0; k < P; ++k) {
    SweepPointResult pr;
    uint64_t rem = k;
    pr.coordinates.assign(cfg.axes.size(), 0.0);
    for (std::size_t a = cfg.axes.size(); a-- > 0;) {  // last axis fastest
      pr.coordinates[a] = cfg.axes[a].values[rem % cfg.axes[a].values.size()];
      rem /= cfg.axes[a].values.size();
    }
    pr.stats = stats_from_moments(cfg.grid, n, cfg.runs_per_point, mean.data() + k * gn, m2.data() + k * gn);
    res.points.push_back(std::move(pr));
  }
  return res;
}

// run_ensemble (ensemble.hpp:97-99): statistics from the engine; the sink (if
// any) sees every trajectory in run order.  Runs spread over
// min(options.workers, GPUs) devices and their per-device accumulators merge
// in ascending range order, as the reference's workers do.
EnsembleStatistics run_ensemble(const ReactionNetwork& net, const EnsembleOptions& o, const RunSink& sink) {
  Call call(net, o.workers);
  const std::size_t n = net.species_count(), gn = o.grid.size() * n;
  std::vector<double> mean(gn), m2(gn), traj;
  std::vector<uint64_t> meta(o.n_runs * 6);
  if (sink) traj.assign(o.n_runs * gn, 0.0);
  kin_sweep_out out{};
  out.traj = sink ? traj.data() : nullptr;  // no sink: KIN_OUTPUT_STATS_ONLY inside kin_ensemble_run
  out.meta = meta.data();
  out.mean = mean.data();
  out.m2 = m2.data();
  const kin_method m = method_of(o.method);
  kin_error e{};
  if (int rc = kin_ensemble_run(call.ctx, call.model, &m, o.n_runs, o.master_seed, o.t_end, o.grid.data(),
                                static_cast<int32_t>(o.grid.size()), KIN_RNG_COMPAT, &out, &e))
    rethrow(rc, e);
  if (sink)
    for (uint64_t i = 0; i < o.n_runs; ++i)
      sink(i, trajectory_at(traj, meta, i, o.grid, n, o.method, kin_derive_run_seed(o.master_seed, i)));
  return stats_from_moments(o.grid, n, o.n_runs, mean.data(), m2.data());
}

// run_single (ensemble.hpp:73-76)
Trajectory run_single(const ReactionNetwork& net, const Method& m, double t_end, const std::vector<double>& grid,
                      uint64_t seed) {
  Call call(net, 1);
  const std::size_t n = net.species_count();
  std::vector<double> traj(grid.size() * n);
  std::vector<uint64_t> meta(6);
  const kin_method km = method_of(m);
  kin_error e{};
  if (int rc = kin_run_single(call.ctx, call.model, &km, t_end, grid.data(), static_cast<int32_t>(grid.size()), seed,
                              KIN_RNG_COMPAT, traj.data(), meta.data(), &e))
    rethrow(rc, e);
  return trajectory_at(traj, meta, 0, grid, n, m, seed);
}

}  // namespace kinetics::b200

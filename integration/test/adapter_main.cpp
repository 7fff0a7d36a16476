// integration/test/adapter_main.cpp — TEST DRIVER: the reference's public API
// (kinetics::b200::parameter_sweep / run_ensemble / run_single through the
// adapter) on the Michaelis-Menten and birth-death models; raw doubles into
// <outdir>/*.bin for tests/test_gpu_integration.py to compare with the oracle.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "kinetics/ensemble.hpp"

namespace kinetics::b200 {
SweepResults parameter_sweep(const ReactionNetwork&, const SweepConfig&, unsigned);
EnsembleStatistics run_ensemble(const ReactionNetwork&, const EnsembleOptions&, const RunSink&);
Trajectory run_single(const ReactionNetwork&, const Method&, double, const std::vector<double>&, std::uint64_t);
}  // namespace kinetics::b200

using namespace kinetics;

static void dump(const std::string& path, const std::vector<double>& v) {
  FILE* f = std::fopen(path.c_str(), "wb");
  std::fwrite(v.data(), sizeof(double), v.size(), f);
  std::fclose(f);
}

static Reaction rx(std::string name, std::map<std::size_t, int> l, std::map<std::size_t, int> r, double c,
                   std::optional<std::size_t> p = std::nullopt) {
  Reaction x;
  x.name = std::move(name);
  x.reactants = std::move(l);
  x.products = std::move(r);
  x.rate_constant = c;
  x.rate_param = p;
  return x;
}

int main(int argc, char** argv) {
  const std::string out = argc > 1 ? argv[1] : ".";
  // C1 Michaelis-Menten (workloads.michaelis_menten), params c1, c2, c3
  auto mm = ReactionNetwork::create({{"S", 301}, {"E", 120}, {"ES", 0}, {"P", 0}},
                                    {{"c1", 1.66e-3}, {"c2", 1e-4}, {"c3", 0.1}},
                                    {rx("bind", {{0, 1}, {1, 1}}, {{2, 1}}, 1.66e-3, 0),
                                     rx("unbind", {{2, 1}}, {{0, 1}, {1, 1}}, 1e-4, 1),
                                     rx("convert", {{2, 1}}, {{1, 1}, {3, 1}}, 0.1, 2)});
  std::vector<double> grid;
  for (int g = 0; g < 11; ++g) grid.push_back(50.0 * g / 10.0);
  SweepConfig sc;
  sc.axes = {{"c1", {1.66e-4, 1.66e-3, 1.66e-2}}, {"c3", {0.01, 0.1, 1.0, 10.0}}};
  sc.runs_per_point = 16;
  sc.method.kind = Method::Kind::TauAdaptive;
  sc.master_seed = 13097695;
  sc.t_end = 50.0;
  sc.grid = grid;
  std::vector<double> mean, m2;
  for (unsigned workers : {1u, 4u}) {
    SweepResults res = b200::parameter_sweep(mm, sc, workers);
    mean.clear();
    m2.clear();
    for (const auto& p : res.points)
      for (std::size_t g = 0; g < grid.size(); ++g)
        for (std::size_t s = 0; s < 4; ++s) {
          mean.push_back(p.stats.mean(g, s));
          m2.push_back(p.stats.m2(g, s));
        }
    dump(out + "/sweep_mean_w" + std::to_string(workers) + ".bin", mean);
    dump(out + "/sweep_m2_w" + std::to_string(workers) + ".bin", m2);
  }
  // birth-death ensemble (workloads.birth_death), SSA, with and without a RunSink
  auto bd = ReactionNetwork::create({{"A", 0}}, {{"lam", 5.0}, {"c", 1.0}},
                                    {rx("birth", {}, {{0, 1}}, 5.0, 0), rx("death", {{0, 1}}, {}, 1.0, 1)});
  EnsembleOptions eo;
  eo.method.kind = Method::Kind::Ssa;
  eo.n_runs = 1000;
  eo.t_end = 20.0;
  eo.grid.clear();
  for (int g = 0; g < 21; ++g) eo.grid.push_back(g);
  eo.master_seed = 99;
  eo.workers = 1;
  std::vector<double> traj(1000 * 21, -1.0);
  EnsembleStatistics st = b200::run_ensemble(bd, eo, [&](std::uint64_t i, const Trajectory& t) {
    for (std::size_t g = 0; g < t.samples.size(); ++g) traj[i * 21 + g] = t.samples[g][0];
  });
  std::vector<double> em, eq;
  for (std::size_t g = 0; g < 21; ++g) {
    em.push_back(st.mean(g, 0));
    eq.push_back(st.m2(g, 0));
  }
  dump(out + "/ens_traj.bin", traj);
  dump(out + "/ens_mean.bin", em);
  dump(out + "/ens_m2.bin", eq);
  EnsembleStatistics st2 = b200::run_ensemble(bd, eo, {});  // no sink: statistics only
  std::vector<double> em2, eq2;
  for (std::size_t g = 0; g < 21; ++g) {
    em2.push_back(st2.mean(g, 0));
    eq2.push_back(st2.m2(g, 0));
  }
  dump(out + "/ens_nosink_mean.bin", em2);
  dump(out + "/ens_nosink_m2.bin", eq2);
  // run_single: tau-adaptive on MM, seed given directly
  Method tm;
  tm.kind = Method::Kind::TauAdaptive;
  Trajectory t = b200::run_single(mm, tm, 50.0, grid, 123456789);
  std::vector<double> flat;
  for (const auto& row : t.samples) flat.insert(flat.end(), row.begin(), row.end());
  dump(out + "/single.bin", flat);
  std::printf("adapter driver: sweep %zu points, ensemble n=%llu mean(20)=%.6f, single seed=%llu ok\n",
              mean.size() / (grid.size() * 4), (unsigned long long)st.runs(), st.mean(20, 0),
              (unsigned long long)t.seed.value_or(0));
  return 0;
}

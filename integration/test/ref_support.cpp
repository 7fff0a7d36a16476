// integration/test/ref_support.cpp — TEST INFRASTRUCTURE ONLY.
//
// The reference declares these symbols in its public headers but ships no
// implementation for them (the only .cpp is proj/src/rng.cpp).  To
// LINK and RUN the adapter (kinetics_b200_adapter.cpp) end to end, this test
// translation unit supplies minimal definitions restated from the header
// contracts and SPEC.md:
//   ReactionNetwork::create / param_index / species_index   model.hpp:47-76
//   EnsembleStatistics ctor / add / merge / variance         ensemble.hpp:20-57
//   merge_statistics                                          ensemble.hpp:56-57
//   Method::name                                              ensemble.hpp:59-71
// Nothing here is on the product path: the adapter routes the simulations
// through libkin_b200.so.
#include <cstdint>
#include <string>
#include <vector>

#include "kinetics/ensemble.hpp"
#include "kinetics/errors.hpp"

namespace kinetics {

ReactionNetwork ReactionNetwork::create(std::vector<Species> species, std::vector<Parameter> params,
                                        std::vector<Reaction> reactions) {
  ReactionNetwork n;
  const std::size_t N = species.size(), M = reactions.size();
  n.nu_.assign(N * M, 0);
  n.nu_columns_.resize(M);
  for (std::size_t j = 0; j < M; ++j) {
    Reaction& r = reactions[j];
    if (r.rate_param) {
      if (*r.rate_param >= params.size()) throw ValidationError("unknown parameter");
      r.rate_constant = params[*r.rate_param].value;
    }
    if (!(r.rate_constant > 0.0)) throw ValidationError("rate must be positive");
    for (const auto& [s, c] : r.reactants) n.nu_[s * M + j] -= c;
    for (const auto& [s, c] : r.products) n.nu_[s * M + j] += c;
    for (std::size_t s = 0; s < N; ++s)
      if (n.nu_[s * M + j] != 0) n.nu_columns_[j].emplace_back(s, n.nu_[s * M + j]);
  }
  n.species_ = std::move(species);
  n.params_ = std::move(params);
  n.reactions_ = std::move(reactions);
  return n;
}

std::optional<std::size_t> ReactionNetwork::species_index(std::string_view name) const {
  for (std::size_t i = 0; i < species_.size(); ++i)
    if (species_[i].name == name) return i;
  return std::nullopt;
}

std::optional<std::size_t> ReactionNetwork::param_index(std::string_view name) const {
  for (std::size_t i = 0; i < params_.size(); ++i)
    if (params_[i].name == name) return i;
  return std::nullopt;
}

EnsembleStatistics::EnsembleStatistics(std::vector<double> grid, std::size_t species_count)
    : grid_(std::move(grid)), species_count_(species_count) {
  mean_.assign(grid_.size() * species_count_, 0.0);
  m2_.assign(grid_.size() * species_count_, 0.0);
}

// Welford (SURVEY App. B #9 order): delta = x - mean; mean += delta/n; m2 += delta*(x - mean)
void EnsembleStatistics::add(const Trajectory& t) {
  ++n_;
  const double nn = static_cast<double>(n_);
  for (std::size_t g = 0; g < grid_.size(); ++g)
    for (std::size_t s = 0; s < species_count_; ++s) {
      const std::size_t q = g * species_count_ + s;
      const double x = t.samples[g][s];
      const double delta = x - mean_[q];
      mean_[q] = mean_[q] + delta / nn;
      m2_[q] = m2_[q] + delta * (x - mean_[q]);
    }
}

void EnsembleStatistics::merge(const EnsembleStatistics& o) {
  if (o.n_ == 0) return;
  if (n_ == 0) { *this = o; return; }
  const double fa = static_cast<double>(n_), fb = static_cast<double>(o.n_), fn = fa + fb;
  for (std::size_t q = 0; q < mean_.size(); ++q) {
    const double delta = o.mean_[q] - mean_[q];
    mean_[q] = mean_[q] + delta * fb / fn;
    m2_[q] = m2_[q] + o.m2_[q] + delta * delta * fa * fb / fn;
  }
  n_ += o.n_;
}

double EnsembleStatistics::variance(std::size_t g, std::size_t s) const {
  return n_ < 2 ? 0.0 : m2(g, s) / static_cast<double>(n_ - 1);
}

EnsembleStatistics merge_statistics(EnsembleStatistics a, const EnsembleStatistics& b) {
  a.merge(b);
  return a;
}

std::string Method::name() const {
  switch (kind) {
    case Kind::Ssa: return "ssa";
    case Kind::TauAdaptive: return "tau-adaptive";
    case Kind::TauFixed: return "tau-fixed";
    case Kind::Cle: return "cle";
    case Kind::Ode: return "ode";
    case Kind::Hybrid: return "hybrid";
  }
  return "?";
}

}  // namespace kinetics

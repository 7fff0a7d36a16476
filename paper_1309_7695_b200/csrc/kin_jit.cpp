// kin_jit.cpp — per-model specialisation of the SSA / tau-leaping kernel.
//
// The table-driven kernel (kin_stochastic.cu) walks the model's packed tables
// at run time: ~60% of its instructions (profiles/r1_v4_tau_lines.txt) decode
// reaction descriptors, nu rows/columns and shared-memory addresses.  Here the
// host generates, from the model's structure, a model policy whose
// propensities, select_tau rows, state updates and dependency updates are
// straight-line code with literal species/reaction indices, stoichiometries
// and g_i (rate constants still come from the constant-bank tables, so one
// compiled kernel serves every sweep point).  The policy plugs into the same
// kernel body (kin_stochastic_impl.cuh) and performs the same floating-point
// operations in the same order, so the results stay bit-identical to the
// oracle.  Compiled once per (model structure, sweep-axis binding, variant)
// with NVRTC for sm_100a (-fmad=false) and cached for the process.
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <sys/stat.h>
#include <unistd.h>

#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/kin_abi.h"
#include "kin_jit.h"
#include "kin_launch.h"

namespace kin {

namespace {

#include "build/kin_jit_sources.inc"  // kJitHeaders[] = {name, text}

struct JitKernel {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  bool ok = false;
  std::string log;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<JitKernel>> g_cache;

bool jit_debug() {
  static const bool d = std::getenv("KIN_JIT_DEBUG") != nullptr;
  return d;
}

std::string dlit(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  std::string s(b);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// Largest model whose SSA events are branch-free (select, update and
// propensity refresh the same instructions on every lane, whatever `sel`).
constexpr int kUniformSsaMaxReactions = 8;
// Largest model whose divergent SSA updates are emitted as a switch.
constexpr int kSwitchMaxReactions = 8;
// Largest number of species with a nu row whose select_tau is fully inlined.
constexpr int kInlineTauMaxSpecies = 8;
// Smallest M whose select_tau walks four species per trip (every model whose
// select_tau is not fully inlined: C4 94.5 -> 89.1 ms, C5 1337 -> 1217 ms).
constexpr int kGroupTauMinReactions = 1;
// Largest nnz(nu) whose leap update is a switch of straight-line updates.
constexpr int kSwitchApplyMaxNnz = 16;
// Largest M whose all_props is straight-line (above: uniform loop over prop(j)).
constexpr int kInlinePropsMaxReactions = 1 << 30;
// Flat-loop models: SSA events per trip of the flat loop (see
// kin_stochastic_impl.cuh simulate_one; C2 46.7 / 39.5 / 36.5 / 39.6 / 44.0 ms
// at 1 / 2 / 4 / 8 / 16).
constexpr int kBurstQuantumDefault = 4;

// Development knobs (KIN_JIT_TAU_INLINE / KIN_JIT_APPLY_SWITCH override the
// thresholds; they change the generated source, hence the cache key).
// Read once per process and name (study knobs, never per launch).
int jit_knob(const char* name, int dflt) {
  static std::mutex mu;
  static std::map<std::string, int> seen;
  std::lock_guard<std::mutex> lk(mu);
  auto it = seen.find(name);
  if (it == seen.end()) {
    const char* v = std::getenv(name);
    it = seen.emplace(name, v && *v ? std::atoi(v) : INT32_MIN).first;
  }
  return it->second == INT32_MIN ? dflt : it->second;
}

// Model policy source for one model structure (see kin_stochastic_impl.cuh
// TableModel for the reference semantics of each member).
std::string generate_policy(const JitModel& m) {
  std::ostringstream o;
  o << "namespace kin { namespace stoch {\n"
       "template <class XT> struct GenModel {\n"
       "  const KinTables& T; XT* x; double* a; const double* av;\n"
       "  static constexpr int B = kBlock;\n"
    << "  __device__ __forceinline__ int n() const { return " << m.n << "; }\n"
    << "  __device__ __forceinline__ int m() const { return " << m.m << "; }\n"
       "  __device__ __forceinline__ double xv(int i) const { return static_cast<double>(x[i * B]); }\n"
       "  __device__ __forceinline__ double aval(int j) const { return a[j * B]; }\n"
       "  __device__ __forceinline__ void upd(int i, int d, long long k, bool& ovf) const {\n"
       "    XT* xs = x + i * B;\n"
       "    if constexpr (sizeof(XT) == 8) {\n"
       "      *xs = __dadd_rn(*xs, __dmul_rn(static_cast<double>(d), static_cast<double>(k)));\n"
       "    } else {\n"
       "      const long long v = static_cast<long long>(*xs) + static_cast<long long>(d) * k;\n"
       "      ovf |= v > 2147483647LL || v < -2147483647LL;\n"
       "      *xs = static_cast<XT>(v);\n"
       "    }\n"
       "  }\n"
       "  __device__ __forceinline__ bool upd1(int i, int d, bool& ovf) const {\n"
       "    XT* xs = x + i * B;\n"
       "    if constexpr (sizeof(XT) == 8) {\n"
       "      const double v = __dadd_rn(*xs, static_cast<double>(d));\n"
       "      *xs = v;\n"
       "      return v < 0.0;\n"
       "    } else {\n"
       "      const long long v = static_cast<long long>(*xs) + d;\n"
       "      ovf |= v > 2147483647LL;\n"
       "      *xs = static_cast<XT>(v);\n"
       "      return v < 0;\n"
       "    }\n"
       "  }\n";
  // propensity of reaction j (model.hpp:151-157, oracle order)
  o << "  __device__ __forceinline__ double prop(const int j) const {\n    double aj;\n    switch (j) {\n";
  for (int j = 0; j < m.m; ++j) {
    o << "      case " << j << ": aj = ";
    if (m.rate_axis[j] >= 0 && !m.rate_scaled.empty() && m.rate_scaled[j])
      o << "__dmul_rn(tab_rate(T, " << j << "), av[" << m.rate_axis[j] << " * B])";
    else if (m.rate_axis[j] >= 0) o << "av[" << m.rate_axis[j] << " * B]";
    else o << "tab_rate(T, " << j << ")";
    o << ";";
    for (int p = m.rt_ptr[j]; p < m.rt_ptr[j + 1]; ++p)
      o << " aj = __dmul_rn(aj, combinations_c<" << m.rt_stoich[p] << ">(xv(" << m.rt_species[p] << ")));";
    o << " return aj;\n";
  }
  o << "    }\n    return 0.0;\n  }\n";
  if (m.m <= jit_knob("KIN_JIT_PROPS_INLINE", kInlinePropsMaxReactions)) {
    o << "  __device__ __forceinline__ double all_props(int) const {\n    double a0 = 0.0, aj;\n";
    for (int j = 0; j < m.m; ++j)
      o << "    aj = prop(" << j << "); a[" << j << " * B] = aj; a0 = __dadd_rn(a0, aj);\n";
    o << "    return a0;\n  }\n";
  } else {
    o << "  __device__ __forceinline__ double all_props(int) const {\n    double a0 = 0.0;\n"
         "#pragma unroll 1\n    for (int j = 0; j < " << m.m << "; ++j) { const double aj = prop(j); a[j * B] = aj; a0 = __dadd_rn(a0, aj); }\n"
         "    return a0;\n  }\n";
  }
  o << "  __device__ __forceinline__ double sum_props(int) const {\n    double a0 = 0.0;\n";
  for (int j = 0; j < m.m; ++j) o << "    a0 = __dadd_rn(a0, a[" << j << " * B]);\n";
  o << "    return a0;\n  }\n";
  // select_tau (stochastic.hpp:40-44): per species, its nu row in reaction
  // order.  Straight-line code for every species would inline tau_bound N times
  // and overflow the instruction cache on larger models, so above
  // kInlineTauMaxSpecies the species are walked by a warp-uniform, non-unrolled
  // loop whose switch holds only each species' mu/sigma^2 sums (one tau_bound).
  // mu += d*a_j, s2 += d^2*a_j.  For d = +-1 the products are exactly +-a_j,
  // and an intrinsic multiply by 1.0 is not folded: emit the add / subtract
  // (x + (-a) and x - a are the same IEEE operation), so each unit term costs
  // two DADDs instead of two DMUL + DADD pairs — bit-identical sums.
  auto tau_terms = [&](int d, int j) {
    std::ostringstream t;
    const std::string aj = "a[" + std::to_string(j) + " * B]";
    if (d == 1) t << " mu = __dadd_rn(mu, " << aj << "); s2 = __dadd_rn(s2, " << aj << ");";
    else if (d == -1) t << " mu = __dsub_rn(mu, " << aj << "); s2 = __dadd_rn(s2, " << aj << ");";
    else
      t << " mu = __dadd_rn(mu, __dmul_rn(" << dlit(d) << ", " << aj << "));"
        << " s2 = __dadd_rn(s2, __dmul_rn(" << dlit(static_cast<double>(d) * d) << ", " << aj << "));";
    return t.str();
  };
  int n_act = 0;
  for (int i = 0; i < m.n; ++i) n_act += m.row_ptr[i] != m.row_ptr[i + 1];
  o << "  template <bool kCount> __device__ __forceinline__ double select_tau(double eps, uint64_t& flops) const {\n"
       "    double tau = KIN_INF;\n";
  if (n_act <= jit_knob("KIN_JIT_TAU_INLINE", kInlineTauMaxSpecies)) {
    for (int i = 0; i < m.n; ++i) {
      const int p0 = m.row_ptr[i], p1 = m.row_ptr[i + 1];
      if (p0 == p1) continue;  // mu = sigma2 = 0 exactly: skipped by the reference too
      o << "    { double mu = 0.0, s2 = 0.0;";
      for (int p = p0; p < p1; ++p) {
        const int j = m.row_reaction[p], d = m.row_delta[p];
        o << tau_terms(d, j);
      }
      o << "\n      if (kCount) flops += " << 4 * (p1 - p0) << ";\n"
        << "      if (!(mu == 0.0 && s2 == 0.0)) tau = tau_bound<kCount>(tau, eps, xv(" << i << "), " << dlit(m.g[i])
        << ", mu, s2, flops); }\n";
    }
  } else if (m.m >= kGroupTauMinReactions) {
    // four species per trip: their row sums formed together (one switch
    // dispatch per four species, the loads of all four rows in flight —
    // global memory on large models), then four tau_bound in species order
    const int kG = std::max(1, std::min(16, jit_knob("KIN_JIT_TAU_GROUP", 4)));
    const int n_grp = (n_act + kG - 1) / kG;
    std::string ones = "1.0";
    for (int u = 1; u < kG; ++u) ones += ", 1.0";
    o << "#pragma unroll 1\n    for (int q = 0; q < " << n_grp << "; ++q) {\n"
         "      double mu[" << kG << "] = {}, s2[" << kG << "] = {}, g[" << kG << "] = {" << ones << "};\n"
         "      int sp[" << kG << "] = {}, nt = 0;\n      switch (q) {\n";
    int q = 0;
    for (int i = 0; i < m.n; ++i) {
      const int p0 = m.row_ptr[i], p1 = m.row_ptr[i + 1];
      if (p0 == p1) continue;
      const int u = q % kG;
      if (u == 0) o << "        case " << q / kG << ":";
      o << " { double& mu_ = mu[" << u << "]; double& s2_ = s2[" << u << "]; sp[" << u << "] = " << i << "; g[" << u
        << "] = " << dlit(m.g[i]) << "; nt += " << 4 * (p1 - p0) << ";";
      for (int p = p0; p < p1; ++p) {
        std::string t = tau_terms(m.row_delta[p], m.row_reaction[p]);
        for (size_t k; (k = t.find("mu = __d")) != std::string::npos;) t.replace(k, 8, "mu_ = __d");
        for (size_t k; (k = t.find("s2 = __d")) != std::string::npos;) t.replace(k, 8, "s2_ = __d");
        for (size_t k; (k = t.find("(mu, ")) != std::string::npos;) t.replace(k, 5, "(mu_, ");
        for (size_t k; (k = t.find("(s2, ")) != std::string::npos;) t.replace(k, 5, "(s2_, ");
        o << t;
      }
      o << " }";
      ++q;
      if (q % kG == 0 || q == n_act) o << " break;\n";
    }
    o << "      }\n      if (kCount) flops += nt;\n"
         "#pragma unroll\n      for (int u = 0; u < " << kG << "; ++u)\n"
         "        if (!(mu[u] == 0.0 && s2[u] == 0.0)) tau = tau_bound<kCount>(tau, eps, xv(sp[u]), g[u], mu[u], s2[u], flops);\n"
         "    }\n";
  } else {
    o << "#pragma unroll 1\n    for (int q = 0; q < " << n_act << "; ++q) {\n"
         "      double mu = 0.0, s2 = 0.0, g = 1.0; int sp = 0, nt = 0;\n      switch (q) {\n";
    int q = 0;
    for (int i = 0; i < m.n; ++i) {
      const int p0 = m.row_ptr[i], p1 = m.row_ptr[i + 1];
      if (p0 == p1) continue;
      o << "        case " << q++ << ": sp = " << i << "; g = " << dlit(m.g[i]) << "; nt = " << 4 * (p1 - p0) << ";";
      for (int p = p0; p < p1; ++p) {
        const int j = m.row_reaction[p], d = m.row_delta[p];
        o << tau_terms(d, j);
      }
      o << " break;\n";
    }
    o << "      }\n      if (kCount) flops += nt;\n"
         "      if (!(mu == 0.0 && s2 == 0.0)) tau = tau_bound<kCount>(tau, eps, xv(sp), g, mu, s2, flops);\n    }\n";
  }
  o << "    return tau;\n  }\n";
  // leap updates x += nu[:, j] * k (j warp-uniform): a switch of straight-line
  // updates for small models, the CSC walk above kSwitchApplyMaxNnz (code size)
  if (m.col_ptr[m.m] <= jit_knob("KIN_JIT_APPLY_SWITCH", kSwitchApplyMaxNnz)) {
    o << "  __device__ __forceinline__ void apply(int j, long long k, bool& ovf) const {\n    switch (j) {\n";
    for (int j = 0; j < m.m; ++j) {
      o << "      case " << j << ":";
      for (int p = m.col_ptr[j]; p < m.col_ptr[j + 1]; ++p)
        o << " upd(" << m.col_species[p] << ", " << m.col_delta[p] << ", k, ovf);";
      o << " break;\n";
    }
    o << "    }\n  }\n";
  } else {
    o << "  __device__ __forceinline__ void apply(int j, long long k, bool& ovf) const { TableModel<XT>{T, x, a, av}.apply(j, k, ovf); }\n";
  }
  // SSA events: `sel` differs from lane to lane, and a switch over reactions
  // serialises a warp over every distinct case it holds (up to M of them).
  // Small models keep the straight-line cases; larger ones walk the tables
  // (TableModel: the lanes stay converged, only trip counts differ).
  if (m.m <= jit_knob("KIN_JIT_UNIFORM_SSA", kUniformSsaMaxReactions)) {
    // Branch-free SSA event: each touched species takes its delta for `j`
    // from a select chain (a zero delta rewrites the same amount), and every
    // propensity is re-evaluated (a pure function of x: the untouched ones
    // get the same values) — the lanes of a warp never split over `sel`.
    std::vector<int> touched(m.n, 0);
    for (int p = 0; p < m.col_ptr[m.m]; ++p) touched[m.col_species[p]] = 1;
    o << "  static constexpr bool kUniformSsa = true;\n  static constexpr bool kFlatBurst = true;\n"
         "  static constexpr int kM = " << m.m << ";\n"
         "  static constexpr int kBurstQuantum = " << std::max(1, std::min(64, jit_knob("KIN_JIT_BURST_K", kBurstQuantumDefault))) << ";\n";
    o << "  __device__ __forceinline__ bool fire(int j, bool& ovf) const {\n    bool neg = false;\n";
    for (int i = 0; i < m.n; ++i) {
      if (!touched[i]) continue;
      std::vector<int> d(m.m, 0);
      for (int j = 0; j < m.m; ++j)
        for (int p = m.col_ptr[j]; p < m.col_ptr[j + 1]; ++p)
          if (m.col_species[p] == i) d[j] += m.col_delta[p];
      o << "    { const int d = ";
      for (int j = 0; j + 1 < m.m; ++j) o << "j == " << j << " ? " << d[j] << " : ";
      o << d[m.m - 1] << "; const bool ng = upd1(" << i << ", d, ovf); neg |= d != 0 && ng; }\n";
    }
    o << "    return neg;\n  }\n";
    o << "  __device__ __forceinline__ void dep_update(int) const {\n";
    for (int j = 0; j < m.m; ++j) o << "    a[" << j << " * B] = prop(" << j << ");\n";
    o << "  }\n";
  } else if (m.m <= kSwitchMaxReactions) {
    o << "  static constexpr bool kUniformSsa = false;\n  static constexpr bool kFlatBurst = false;\n"
         "  static constexpr int kBurstQuantum = 1;\n"
         "  static constexpr int kM = " << m.m << ";\n";
    o << "  __device__ __forceinline__ bool fire(int j, bool& ovf) const {\n    bool neg = false;\n    switch (j) {\n";
    for (int j = 0; j < m.m; ++j) {
      o << "      case " << j << ":";
      for (int p = m.col_ptr[j]; p < m.col_ptr[j + 1]; ++p)
        o << " neg |= upd1(" << m.col_species[p] << ", " << m.col_delta[p] << ", ovf);";
      o << " break;\n";
    }
    o << "    }\n    return neg;\n  }\n";
    o << "  __device__ __forceinline__ void dep_update(int sel) const {\n    switch (sel) {\n";
    for (int j = 0; j < m.m; ++j) {
      o << "      case " << j << ":";
      for (int q = m.dep_ptr[j]; q < m.dep_ptr[j + 1]; ++q)
        o << " a[" << m.dep[q] << " * B] = prop(" << m.dep[q] << ");";
      o << " break;\n";
    }
    o << "    }\n  }\n";
  } else {
    // Flat loop when the state lives in global memory (C5: 1208 -> 1074 ms at
    // four events per trip; 16: 1134, 64: 1222); shared-memory layouts keep
    // the nested burst (C4: 89.1 vs 90.5-92.4 ms flat — the flat form needs
    // 135 registers, past the 128 at which 14 warps per SM fit)
    const int flat = jit_knob("KIN_JIT_FLAT_LARGE", -1);
    o << "  static constexpr bool kUniformSsa = false;\n  static constexpr bool kFlatBurst = "
      << (flat < 0 ? "KGLOBAL_" : flat ? "true" : "false") << ";\n"
         "  static constexpr int kBurstQuantum = " << std::max(1, jit_knob("KIN_JIT_BURST_K_LARGE", 4)) << ";\n"
         "  static constexpr int kM = " << m.m << ";\n";
    o << "  __device__ __forceinline__ bool fire(int j, bool& ovf) const { return TableModel<XT>{T, x, a, av}.fire(j, ovf); }\n"
         "  __device__ __forceinline__ void dep_update(int sel) const { TableModel<XT>{T, x, a, av}.dep_update(sel); }\n";
  }
  o << "  __device__ __forceinline__ bool any_negative() const {\n    bool neg = false;\n"
    << "#pragma unroll\n    for (int i = 0; i < " << m.n << "; ++i) neg |= x[i * B] < static_cast<XT>(0);\n"
    << "    return neg;\n  }\n";
  o << "  __device__ __forceinline__ int col_len(int j) const { return tab_col_ptr(T, j + 1) - tab_col_ptr(T, j); }\n";
  // hybrid PDMP (kin_hybrid_impl.cuh; TableModel::props_only / hyb_rows):
  // straight-line propensities and row sums, the slow-set words read once
  o << "  __device__ __forceinline__ void props_only() const {\n";
  for (int j = 0; j < m.m; ++j) o << "    a[" << j << " * B] = prop(" << j << ");\n";
  o << "  }\n";
  o << "  __device__ __forceinline__ void hyb_rows(const uint32_t* slowm, double* f, int) const {\n";
  const int words = (m.m + 31) / 32;
  for (int w = 0; w < words; ++w) o << "    const uint32_t w" << w << " = slowm[" << w << " * B];\n";
  auto slow = [](int j) { return "((w" + std::to_string(j >> 5) + " >> " + std::to_string(j & 31) + ") & 1u)"; };
  for (int i = 0; i < m.n; ++i) {
    o << "    { double acc = 0.0;";
    for (int p = m.row_ptr[i]; p < m.row_ptr[i + 1]; ++p) {
      const int j = m.row_reaction[p], d = m.row_delta[p];
      const std::string aj = "a[" + std::to_string(j) + " * B]";
      std::string t;
      if (d == 1) t = "__dadd_rn(acc, " + aj + ")";
      else if (d == -1) t = "__dsub_rn(acc, " + aj + ")";
      else t = "__dadd_rn(acc, __dmul_rn(" + dlit(d) + ", " + aj + "))";
      o << " { const double t = " << t << "; acc = " << slow(j) << " ? acc : t; }";
    }
    o << " f[" << i << " * B] = acc; }\n";
  }
  o << "    double g = 0.0;\n";
  for (int j = 0; j < m.m; ++j)
    o << "    { const double t = __dadd_rn(g, a[" << j << " * B]); g = " << slow(j) << " ? t : g; }\n";
  o << "    f[" << m.n << " * B] = g;\n  }\n";
  o << "  static constexpr bool kJit = true;\n";
  // LSODA (kin_lsoda_impl.cuh; rre_rhs): f_i = sum over the nu row of d * a_j
  o << "  __device__ __forceinline__ void rre_rows(double* f, int) const {\n";
  for (int i = 0; i < m.n; ++i) {
    o << "    { double acc = 0.0;";
    for (int p = m.row_ptr[i]; p < m.row_ptr[i + 1]; ++p) {
      const int j = m.row_reaction[p], d = m.row_delta[p];
      const std::string aj = "a[" + std::to_string(j) + " * B]";
      if (d == 1) o << " acc = __dadd_rn(acc, " << aj << ");";
      else if (d == -1) o << " acc = __dsub_rn(acc, " << aj << ");";
      else o << " acc = __dadd_rn(acc, __dmul_rn(" << dlit(d) << ", " << aj << "));";
    }
    o << " f[" << i << " * B] = acc; }\n";
  }
  o << "  }\n";
  // LSODA's Jacobian J = nu * da/dx (rre_jacobian), straight-line for small
  // models (kin_lsoda_impl.cuh Lsoda::jac_row / jacobian: the same products
  // and sums in the same order as their table walks; x = the state vector)
  int jac_work = 0;
  for (int j = 0; j < m.m; ++j) {
    const int nt = m.rt_ptr[j + 1] - m.rt_ptr[j];
    jac_work += nt * (m.col_ptr[j + 1] - m.col_ptr[j]);
  }
  const bool jit_jac = m.n <= 8 && jac_work <= jit_knob("KIN_JIT_JAC_MAX", 64);
  o << "  static constexpr bool kJitJac = " << (jit_jac ? "true" : "false") << ";\n";
  auto rate_expr = [&](int j) {
    if (m.rate_axis[j] >= 0) return "__dmul_rn(tab_rate(T, " + std::to_string(j) + "), av[" + std::to_string(m.rate_axis[j]) + " * B])";
    return "tab_rate(T, " + std::to_string(j) + ")";
  };
  // dd of term p of reaction j: rk * dh(x_s) * prod over the other terms
  auto term_dd = [&](int j, int p) {
    std::ostringstream t;
    t << "double dd = __dmul_rn(rk, jac_dh<" << m.rt_stoich[p] << ">(xv(" << m.rt_species[p] << ")));";
    for (int q = m.rt_ptr[j]; q < m.rt_ptr[j + 1]; ++q)
      if (q != p) t << " dd = __dmul_rn(dd, combinations_c<" << m.rt_stoich[q] << ">(xv(" << m.rt_species[q] << ")));";
    return t.str();
  };
  auto add_term = [&](const std::string& dst, int d) {
    if (d == 1) return dst + " = __dadd_rn(" + dst + ", dd);";
    if (d == -1) return dst + " = __dsub_rn(" + dst + ", dd);";
    return dst + " = __dadd_rn(" + dst + ", __dmul_rn(" + dlit(d) + ", dd));";
  };
  o << "  __device__ __forceinline__ void jac_row(int i, double* tmp) const {\n";
  if (jit_jac) {
    o << "#pragma unroll\n    for (int s = 0; s < " << m.n << "; ++s) tmp[s * B] = 0.0;\n    switch (i) {\n";
    for (int i = 0; i < m.n; ++i) {
      o << "      case " << i << ":";
      for (int pr = m.row_ptr[i]; pr < m.row_ptr[i + 1]; ++pr) {
        const int j = m.row_reaction[pr], d = m.row_delta[pr];
        if (m.rt_ptr[j + 1] == m.rt_ptr[j]) continue;  // zero-order: no x dependence
        o << " { const double rk = " << rate_expr(j) << ";";
        for (int p = m.rt_ptr[j]; p < m.rt_ptr[j + 1]; ++p)
          o << " { " << term_dd(j, p) << " " << add_term("tmp[" + std::to_string(m.rt_species[p]) + " * B]", d) << " }";
        o << " }";
      }
      o << " break;\n";
    }
    o << "    }\n";
  }
  o << "  }\n";
  o << "  __device__ __forceinline__ void jac_full(double* J) const {\n";
  if (jit_jac) {
    o << "#pragma unroll\n    for (int q = 0; q < " << m.n * m.n << "; ++q) J[q * B] = 0.0;\n";
    for (int j = 0; j < m.m; ++j) {
      if (m.rt_ptr[j + 1] == m.rt_ptr[j]) continue;
      o << "    { const double rk = " << rate_expr(j) << ";";
      for (int p = m.rt_ptr[j]; p < m.rt_ptr[j + 1]; ++p) {
        o << " { " << term_dd(j, p);
        for (int c = m.col_ptr[j]; c < m.col_ptr[j + 1]; ++c)
          o << " " << add_term("J[" + std::to_string(m.col_species[c] * m.n + m.rt_species[p]) + " * B]", m.col_delta[c]);
        o << " }";
      }
      o << " }\n";
    }
  }
  o << "  }\n";
  o << "};\n}}  // namespace kin::stoch\n";
  return o.str();
}

const char* const kNvrtcOpts[5] = {"--gpu-architecture=sm_100a", "-fmad=false", "-std=c++17", "-lineinfo",
                                   "-default-device"};

// NVRTC: policy source -> sm_100a cubin.  Returns false with the log on error.
// Which kernel a JIT variant is (`spec`): < 0 the stochastic kernel
// (kin_jit_stoch); 0..99 the hybrid PDMP kernel (kin_jit_hybrid) specialised
// on kN = spec species (0 = runtime); >= 100 the LSODA kernel (kin_jit_lsoda)
// with kN = spec - 100.
constexpr int kSpecLsoda = 100;
const char* spec_kernel_name(int spec) {
  return spec < 0 ? "kin_jit_stoch" : (spec < kSpecLsoda ? "kin_jit_hybrid" : "kin_jit_lsoda");
}
bool nvrtc_compile(const std::string& policy, bool count, bool philox, bool int_state, bool global_state,
                   bool smem_x, int firing, std::vector<char>* cubin, std::string* log, int spec) {
  std::string src =
      spec >= kSpecLsoda
          ? "#include \"kin_stochastic_impl.cuh\"\n#include \"kin_lsoda_impl.cuh\"\n" + policy +
                "extern \"C\" __global__ void __maxnreg__(200) kin_jit_lsoda(\n"
                "    const __grid_constant__ KinTables T, const __grid_constant__ KinSweepDev S, KinOutDev O,\n"
                "    const double* __restrict__ co, unsigned long long* __restrict__ next) {\n"
                "  kin::lsd::lsoda_body<KCOUNT_, KGLOBAL_, " + std::to_string(spec - kSpecLsoda) +
                ", kin::stoch::GenModel<double>>(T, S, O, co, next);\n"
                "}\n"
      : spec >= 0
          ? "#include \"kin_hybrid_impl.cuh\"\n" + policy +
                "extern \"C\" __global__ void __launch_bounds__(32) kin_jit_hybrid(\n"
                "    const __grid_constant__ KinTables T, const __grid_constant__ KinSweepDev S, KinOutDev O,\n"
                "    unsigned long long* __restrict__ next) {\n"
                "  kin::hyb::hybrid_body<KCOUNT_, KPHILOX_, KGLOBAL_, " + std::to_string(spec) +
                ", kin::stoch::GenModel<double>>(T, S, O, next);\n"
                "}\n"
          : "#include \"kin_stochastic_impl.cuh\"\n" + policy +
                "extern \"C\" __global__ void __launch_bounds__(KIN_STOCH_BLOCK, KMINB_) kin_jit_stoch(\n"
                "    const __grid_constant__ KinTables T, const __grid_constant__ KinSweepDev S, KinOutDev O,\n"
                "    unsigned long long* __restrict__ next, int* ovf) {\n"
                "  kin::stoch::stochastic_body<kin::stoch::GenModel<XT_>, KCOUNT_, KPHILOX_, XT_, KGLOBAL_, KSMEMX_>(T, S, O, next, ovf);\n"
                "}\n";
  std::vector<const char*> hs, hn;
  for (const auto& h : kJitHeaders) {
    hn.push_back(h.name);
    hs.push_back(h.text);
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "kin_jit_stoch.cu", static_cast<int>(hs.size()), hs.data(), hn.data()) !=
      NVRTC_SUCCESS) {
    *log = "nvrtcCreateProgram failed";
    return false;
  }
  const std::string d_xt = std::string("-DXT_=") + (int_state ? "int" : "double");
  const std::string d_c = std::string("-DKCOUNT_=") + (count ? "true" : "false");
  const std::string d_p = std::string("-DKPHILOX_=") + (philox ? "true" : "false");
  const std::string d_g = std::string("-DKGLOBAL_=") + (global_state ? "true" : "false");
  const std::string d_x = std::string("-DKSMEMX_=") + (smem_x ? "true" : "false");
  // split layout: its 16 KB of shared memory per warp allows 13 resident warps
  // per SM; ask the register allocator for that many (development knob)
  const std::string d_b = "-DKMINB_=" + std::to_string(smem_x ? jit_knob("KIN_JIT_SPLIT_MINB", 1) : jit_knob("KIN_JIT_MINB", 1));
  const std::string d_f = "-DKFIRING_=" + std::to_string(firing);
  const char* opts[] = {kNvrtcOpts[0], kNvrtcOpts[1], kNvrtcOpts[2], kNvrtcOpts[3], kNvrtcOpts[4],
                        d_xt.c_str(),  d_c.c_str(),   d_p.c_str(),   d_g.c_str(),   d_x.c_str(), d_b.c_str(),
                        d_f.c_str()};
  const nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  if (log_size > 1) {
    log->resize(log_size);
    nvrtcGetProgramLog(prog, &(*log)[0]);
  }
  if (rc != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return false;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  if (const char* dump = std::getenv("KIN_JIT_DUMP")) {  // offline inspection (cuobjdump / nvcc -Xptxas -v)
    const std::string base = std::string(dump) + "/kin_jit_" + (count ? "C" : "c") + (philox ? "P" : "p") +
                             (int_state ? "I" : "D");
    if (FILE* f = std::fopen((base + ".cu").c_str(), "wb")) {
      std::fwrite(src.data(), 1, src.size(), f);
      std::fclose(f);
    }
    if (FILE* f = std::fopen((base + ".cubin").c_str(), "wb")) {
      std::fwrite(cubin->data(), 1, cubin->size(), f);
      std::fclose(f);
    }
  }
  return true;
}

// On-disk cubin cache (optimisation only): $KIN_JIT_CACHE, else
// $HOME/.cache/kin_b200_jit; keyed by a hash of the full source + variant.
std::string cache_path(const std::string& key) {
  const char* dir = std::getenv("KIN_JIT_CACHE");
  std::string d;
  if (dir && *dir) {
    d = dir;
  } else {
    const char* home = std::getenv("HOME");
    if (!home) return "";
    d = std::string(home) + "/.cache/kin_b200_jit";
  }
  int major = 0, minor = 0;
  nvrtcVersion(&major, &minor);  // statically linked (Makefile), but keyed anyway
  std::string full = key + "|nvrtc " + std::to_string(major) + "." + std::to_string(minor);
  for (const char* o : kNvrtcOpts) full += std::string("|") + o;
  for (const auto& h : kJitHeaders) full += h.text;
  uint64_t hsh = 1469598103934665603ULL;  // FNV-1a 64
  for (unsigned char c : full) hsh = (hsh ^ c) * 1099511628211ULL;
  char name[64];
  std::snprintf(name, sizeof name, "/%016llx.cubin", static_cast<unsigned long long>(hsh));
  return d + name;
}

bool read_file(const std::string& p, std::vector<char>* out) {
  if (p.empty()) return false;
  FILE* f = std::fopen(p.c_str(), "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out->resize(n > 0 ? static_cast<size_t>(n) : 0);
  const bool ok = n > 0 && std::fread(out->data(), 1, out->size(), f) == out->size();
  std::fclose(f);
  return ok;
}

void write_file(const std::string& p, const std::vector<char>& data) {
  if (p.empty()) return;
  const std::string dir = p.substr(0, p.rfind('/'));
  std::string cmd_dir;
  for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0755);
  const std::string tmp = p + ".tmp" + std::to_string(getpid());
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;
  const bool ok = std::fwrite(data.data(), 1, data.size(), f) == data.size();
  std::fclose(f);
  if (ok) std::rename(tmp.c_str(), p.c_str());
  else std::remove(tmp.c_str());
}

// Variant part of a kernel's cache key.
std::string variant_key(bool count, bool philox, bool int_state, bool global_state, bool smem_x, int firing,
                        int spec = -1) {
  return std::string(count ? "C" : "c") + (philox ? "P" : "p") + (int_state ? "I" : "D") +
         (global_state ? (smem_x ? "H" + std::to_string(jit_knob("KIN_JIT_SPLIT_MINB", 1)) : "G") : "S") +
         (jit_knob("KIN_JIT_MINB", 1) != 1 ? "M" + std::to_string(jit_knob("KIN_JIT_MINB", 1)) : "") +
         (firing ? "B" : "") + (spec >= 0 ? "Y" + std::to_string(spec) : "");
}

std::shared_ptr<JitKernel> compile(const std::string& policy, bool count, bool philox, bool int_state,
                                   bool global_state, bool smem_x, int firing, int spec = -1) {
  auto jk = std::make_shared<JitKernel>();
  std::vector<char> cubin;
  const std::string path =
      cache_path(policy + variant_key(count, philox, int_state, global_state, smem_x, firing, spec));
  if (!read_file(path, &cubin)) {
    if (!nvrtc_compile(policy, count, philox, int_state, global_state, smem_x, firing, &cubin, &jk->log, spec)) {
      if (jit_debug()) std::fprintf(stderr, "[kin_jit] compile failed:\n%s\n", jk->log.c_str());
      return jk;
    }
    write_file(path, cubin);
  }
  if (cudaLibraryLoadData(&jk->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&jk->kern, jk->lib, spec_kernel_name(spec)) != cudaSuccess) {
    jk->log += "\ncudaLibraryLoadData/GetKernel failed";
    cudaGetLastError();
    return jk;
  }
  jk->ok = true;
  if (jit_debug())
    std::fprintf(stderr, "[kin_jit] compiled %zu-byte policy (%zu-byte cubin)\n", policy.size(), cubin.size());
  return jk;
}

}  // namespace

// doubles of one block's global-state region that the kernel touches: a[M] +
// av[axes] per lane (+ x[N] when the amounts are not in shared memory)
size_t gstate_live_doubles(const KinTables& T, const KinSweepDev& S, bool x_in_smem) {
  return static_cast<size_t>(T.m + S.n_axes) * KIN_STOCH_BLOCK + (x_in_smem ? 0 : static_cast<size_t>(T.n) * KIN_STOCH_BLOCK);
}

bool jit_compile_check(const JitModel& model, bool count, bool philox, bool int_state, std::string* log) {
  std::vector<char> cubin;
  // KIN_JIT_CHECK_LAYOUT=G|H: the global-state / split layouts (offline register study)
  const char* lay = std::getenv("KIN_JIT_CHECK_LAYOUT");
  const bool g = lay && (*lay == 'G' || *lay == 'H'), h = lay && *lay == 'H';
  return nvrtc_compile(generate_policy(model), count, philox, int_state, g, h, 0, &cubin, log, -1);
}

int hybrid_jit_kn(const JitModel& model) { return model.n <= 8 ? model.n : 0; }

bool jit_compile_check_hybrid(const JitModel& model, bool count, bool philox, std::string* log) {
  std::vector<char> cubin;
  return nvrtc_compile(generate_policy(model), count, philox, false, false, false, 0, &cubin, log,
                       hybrid_jit_kn(model));
}

int lsoda_jit_spec(const JitModel& model) { return kSpecLsoda + (model.n <= 8 ? model.n : 0); }

bool jit_compile_check_lsoda(const JitModel& model, bool count, std::string* log) {
  std::vector<char> cubin;
  return nvrtc_compile(generate_policy(model), count, false, false, false, false, 0, &cubin, log,
                       lsoda_jit_spec(model));
}

cudaError_t launch_lsoda_jit(const JitModel& model, const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                             const double* coeffs, bool count, unsigned long long* counter, size_t smem,
                             cudaStream_t stream, bool* used) {
  *used = false;
  if (S.n_local == 0) {
    *used = true;
    return cudaSuccess;
  }
  const std::string policy = model.policy.empty() ? generate_policy(model) : model.policy;
  const bool global_state = S.gstate != nullptr;
  const int spec = lsoda_jit_spec(model);
  const std::string key = policy + variant_key(count, false, false, global_state, false, 0, spec);
  std::shared_ptr<JitKernel> jk;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      jk = it->second;
    } else {
      jk = compile(policy, count, false, false, global_state, false, 0, spec);
      g_cache[key] = jk;
    }
  }
  if (!jk->ok) return cudaSuccess;  // caller falls back to the table-driven kernel
  if (smem > 227 * 1024) return cudaSuccess;
  const void* fn = reinterpret_cast<const void*>(jk->kern);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaSuccess;
  if (const int cap = jit_knob("KIN_JIT_LSODA_WARPS_PER_SM", 0); cap > 0 && cap < per_sm) per_sm = cap;  // study knob
  const uint64_t warps = (S.n_local + 31) / 32;
  uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  if (S.gstate && S.gstate_warps < resident) resident = S.gstate_warps;
  const unsigned grid = static_cast<unsigned>(warps < resident ? warps : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  KinTables* Tp = const_cast<KinTables*>(&T);
  KinSweepDev* Sp = const_cast<KinSweepDev*>(&S);
  KinOutDev Oc = O;
  void* args[] = {Tp, Sp, &Oc, &coeffs, &counter};
  e = cudaLaunchKernel(fn, dim3(grid), dim3(32), args, smem, stream);
  if (e == cudaSuccess) *used = true;
  return e;
}

cudaError_t launch_hybrid_jit(const JitModel& model, const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                              bool count, unsigned long long* counter, size_t smem, cudaStream_t stream,
                              bool* used) {
  *used = false;
  if (S.n_local == 0) {
    *used = true;
    return cudaSuccess;
  }
  const bool philox = S.rng_mode == KIN_RNG_PHILOX;
  const std::string policy = model.policy.empty() ? generate_policy(model) : model.policy;
  const bool global_state = S.gstate != nullptr;
  const int kn = hybrid_jit_kn(model);
  const std::string key = policy + variant_key(count, philox, false, global_state, false, 0, kn);
  std::shared_ptr<JitKernel> jk;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      jk = it->second;
    } else {
      jk = compile(policy, count, philox, false, global_state, false, 0, kn);
      g_cache[key] = jk;
    }
  }
  if (!jk->ok) return cudaSuccess;  // caller falls back to the table-driven kernel
  if (smem > 227 * 1024) return cudaSuccess;
  const void* fn = reinterpret_cast<const void*>(jk->kern);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaSuccess;
  if (const int cap = jit_knob("KIN_JIT_HYBRID_WARPS_PER_SM", 0); cap > 0 && cap < per_sm) per_sm = cap;  // study knob
  uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  if (S.gstate && S.gstate_warps < resident) resident = S.gstate_warps;
  KinSweepDev SW = S;
  SW.warp_lanes = S.warp_lanes > 0 ? S.warp_lanes : 32;  // as the table-driven hybrid kernel
  const uint64_t warps = (S.n_local + SW.warp_lanes - 1) / SW.warp_lanes;
  const unsigned grid = static_cast<unsigned>(warps < resident ? warps : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  KinTables* Tp = const_cast<KinTables*>(&T);
  KinSweepDev* Sp = &SW;
  KinOutDev Oc = O;
  void* args[] = {Tp, Sp, &Oc, &counter};
  e = cudaLaunchKernel(fn, dim3(grid), dim3(32), args, smem, stream);
  if (e == cudaSuccess) *used = true;
  return e;
}

// KIN_JIT=0: never; KIN_JIT=1: always; unset: launches of >= 8,192
// simulations (where the one-time NVRTC compilation, ~10 s per variant, cached
// in memory and on disk, is amortised).
bool jit_wanted(uint64_t n_sims, int force) {
  if (force >= 0) return force != 0;
  static const int env = [] {
    const char* v = std::getenv("KIN_JIT");
    return (v && *v) ? (std::atoi(v) != 0 ? 1 : 0) : -1;
  }();
  if (env >= 0) return env != 0;
  return n_sims >= 8192;
}

void jit_prepare(JitModel* model) {
  if (model->policy.empty()) model->policy = generate_policy(*model);
}

cudaError_t launch_stochastic_jit(const JitModel& model, const KinTables& T, const KinSweepDev& S,
                                  const KinOutDev& O, bool count, unsigned long long* counter, int* ovf_flag,
                                  bool int_state, cudaStream_t stream, bool* used) {
  *used = false;
  if (S.n_local == 0) {
    *used = true;
    return cudaSuccess;
  }
  const bool philox = S.rng_mode == KIN_RNG_PHILOX;
  const std::string policy = model.policy.empty() ? generate_policy(model) : model.policy;
  const bool global_state = S.gstate != nullptr;
  // split layout (x[] in shared memory, a[] + av[] global) when x[] takes at
  // most 16 KB per warp (>= 13 resident warps/SM): C5 tau 1075 -> 906 ms
  const size_t smem_x_bytes = static_cast<size_t>(T.n) * KIN_STOCH_BLOCK * (int_state ? sizeof(int32_t) : sizeof(double));
  const bool smem_x = global_state && S.gstate_x_smem != 0 && smem_x_bytes <= 16 * 1024;
  const int firing = S.firing == KIN_FIRING_BINOMIAL ? 1 : 0;
  const std::string key = policy + variant_key(count, philox, int_state, global_state, smem_x, firing);
  std::shared_ptr<JitKernel> jk;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      jk = it->second;
    } else {
      jk = compile(policy, count, philox, int_state, global_state, smem_x, firing);
      g_cache[key] = jk;
    }
  }
  if (!jk->ok) return cudaSuccess;  // caller falls back to the table-driven kernel
  const size_t smem = S.gstate ? (smem_x ? smem_x_bytes : 0)
                              : static_cast<size_t>(T.m + S.n_axes) * KIN_STOCH_BLOCK * sizeof(double) + smem_x_bytes;
  if (smem > 227 * 1024) return cudaSuccess;
  const void* fn = reinterpret_cast<const void*>(jk->kern);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, KIN_STOCH_BLOCK, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaSuccess;
  {  // development knob: cap the resident warps per SM (residency studies)
    const int cap = jit_knob("KIN_JIT_WARPS_PER_SM", 0);
    if (cap > 0 && cap < per_sm) per_sm = cap;
  }
  uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  if (S.gstate && S.gstate_warps < resident) resident = S.gstate_warps;
  KinSweepDev SW = S;
  SW.warp_lanes = S.warp_lanes > 0 ? S.warp_lanes : kin_warp_lanes(S.n_local, resident);
  const uint64_t blocks = (S.n_local + SW.warp_lanes - 1) / SW.warp_lanes;
  const unsigned grid = static_cast<unsigned>(blocks < resident ? blocks : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  KinTables* Tp = const_cast<KinTables*>(&T);
  KinSweepDev* Sp = &SW;
  KinOutDev Oc = O;
  void* args[] = {Tp, Sp, &Oc, &counter, &ovf_flag};
  // Global-memory state: the live part (the resident blocks' regions) is
  // rewritten every leap; ask L2 to keep it (persisting access-policy window
  // over exactly those bytes) instead of writing it back to HBM.
  bool window = false;
  if (global_state && jit_knob("KIN_JIT_L2_PERSIST", 1) != 0) {
    const size_t live = static_cast<size_t>(grid) *
                        (smem_x ? gstate_live_doubles(T, S, true) : gstate_live_doubles(T, S, false)) * sizeof(double);
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (max_persist > 0 && max_window > 0 && live > 0) {
      const size_t bytes = std::min<size_t>(live, static_cast<size_t>(max_window));
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(bytes, static_cast<size_t>(max_persist)));
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = S.gstate;
      v.accessPolicyWindow.num_bytes = bytes;
      v.accessPolicyWindow.hitRatio = static_cast<float>(std::min(1.0, static_cast<double>(max_persist) / bytes));
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      window = cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
      cudaGetLastError();
    }
  }
  e = cudaLaunchKernel(fn, dim3(grid), dim3(KIN_STOCH_BLOCK), args, smem, stream);
  if (window) {  // later work on this stream (statistics, copies) streams normally
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaGetLastError();
  }
  if (e == cudaSuccess) *used = true;
  return e;
}

}  // namespace kin

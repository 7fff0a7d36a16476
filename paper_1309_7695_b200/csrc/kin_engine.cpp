// kin_engine.cpp — host side of the B200 sweep engine: the C ABI of
// include/kin_abi.h.
//
// Replaces the reference's ensemble layer (proj/include/kinetics/ensemble.hpp):
//   parameter_sweep  ensemble.hpp:126-130  -> kin_sweep_run / kin_sweep_submit (KIN_SEED_SWEEP)
//   run_ensemble     ensemble.hpp:91-99    -> kin_ensemble_run (KIN_SEED_ENSEMBLE)
//   run_single       ensemble.hpp:73-76    -> kin_run_single (KIN_SEED_DIRECT)
//   merge_statistics ensemble.hpp:56-57    -> kin_stats_merge
// and the model loader ReactionNetwork::create (model.hpp:47-53).
//
// The reference's worker pool (contiguous run ranges per std::thread,
// ensemble.hpp:91-96) becomes the context's GPUs: the simulation index space
// is cut into whole-point chunks assigned cyclically to the devices (balances
// the cost gradient along the sweep axes), or — for ranges with fewer points
// than devices — into equal run ranges whose cut points' statistics are
// Chan-merged in ascending chunk order.  The calling thread enqueues every
// chunk asynchronously (kernels on one of the device's two compute streams,
// copy-out on its copy stream); kin_sweep_wait collects them.  Per-run results
// depend only on the global simulation index, never on the device count
// (SPEC.md:449).  No collective: each device copies its chunk's outputs straight
// into the caller's host buffers at the chunk's global offset.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/kin_abi.h"
#include "kin_device.cuh"
#include "kin_jit.h"
#include "kin_launch.h"
#include "kin_tables.h"

namespace {

// NVTX ranges (SURVEY §5 tracing): host-side phases of a call — the sweep
// table upload, each device's simulation + statistics launches, the copy-out
// enqueue and the wait — visible in Nsight Systems / ncu --nvtx.  Header-only
// NVTX v3: a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void set_err(kin_error* e, int code, const std::string& msg) {
  if (!e) return;
  e->code = code;
  std::snprintf(e->message, sizeof(e->message), "%s", msg.c_str());
}

// Kernel-variant choices come from kin_sweep_desc (lanes_per_sim, variant);
// these environment variables are TEST/STUDY overrides only, read once per
// process (never per launch): -1 / 0 = not set.
struct EnvOverrides {
  int int_state = -1, gstate = -1, gstate_split = -1, hybrid_gstate = -1, lsoda_gstate = -1;
  int ode_lanes = 0, group_lanes = 0;
};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

const EnvOverrides& env_overrides() {
  static const EnvOverrides ov = [] {
    EnvOverrides o;
    o.int_state = env_int("KIN_INT_STATE", -1);
    o.gstate = env_int("KIN_GSTATE", -1);
    o.gstate_split = env_int("KIN_GSTATE_SPLIT", -1);
    o.hybrid_gstate = env_int("KIN_HYBRID_GSTATE", -1);
    o.lsoda_gstate = env_int("KIN_LSODA_GSTATE", -1);
    o.ode_lanes = env_int("KIN_ODE_LANES", 0);
    o.group_lanes = env_int("KIN_GROUP_LANES", 0);
    return o;
  }();
  return ov;
}

// ---- the partitioner (kin_abi.h kin_sweep_plan) ---------------------------------
// The reference's worker pool (contiguous run ranges per std::thread,
// ensemble.hpp:91-96) becomes the context's devices.
struct PlanPart {
  int dev = 0;
  bool inter = false;
  uint64_t s0 = 0, s1 = 0;                       // contiguous
  uint64_t pt_first = 0, pt_stride = 0, n_pts = 0;  // interleaved
  uint64_t out_first = 0, out_pitch = 0;         // caller-local sims
};

int plan_parts(uint64_t s0, uint64_t s1, uint64_t R, int D, int sh_i, int sh_n, std::vector<PlanPart>* parts,
               std::string* msg) {
  parts->clear();
  if (R == 0 || D < 1 || s1 < s0) { *msg = "bad plan arguments"; return KIN_ERR_USAGE; }
  if (sh_n <= 1) { sh_n = 1; sh_i = 0; }
  if (sh_i < 0 || sh_i >= sh_n) { *msg = "shard_index out of range"; return KIN_ERR_INPUT; }
  const uint64_t S = s1 - s0;
  const bool whole = s0 % R == 0 && s1 % R == 0;
  if (sh_n > 1 && !whole) { *msg = "a sharded call needs a range of whole points"; return KIN_ERR_INPUT; }
  if (S == 0) return KIN_OK;
  const uint64_t P0 = s0 / R, P1 = s1 / R;
  if (sh_n > 1 || (whole && D > 1 && P1 - P0 >= static_cast<uint64_t>(D))) {
    // interleaved: device d takes the caller's points d, d+D, ... (cyclic by point)
    const uint64_t n = static_cast<uint64_t>(sh_n);
    const uint64_t K = P1 - P0 > static_cast<uint64_t>(sh_i) ? (P1 - P0 - sh_i + n - 1) / n : 0;
    for (int d = 0; d < D; ++d) {
      if (K <= static_cast<uint64_t>(d)) break;
      PlanPart p;
      p.dev = d;
      p.inter = true;
      p.pt_first = P0 + sh_i + n * d;
      p.pt_stride = n * D;
      p.n_pts = (K - d + D - 1) / D;
      p.out_first = static_cast<uint64_t>(d) * R;
      p.out_pitch = static_cast<uint64_t>(D) * R;
      if (D == 1 && n == 1) {  // one device, no shard: a plain contiguous range
        p.inter = false;
        p.s0 = s0;
        p.s1 = s1;
        p.out_first = 0;
      }
      parts->push_back(p);
    }
    return KIN_OK;
  }
  std::vector<uint64_t> bounds{s0};
  const uint64_t points = (s1 - 1) / R - s0 / R + 1;  // points the range touches
  if (D > 1 && points < static_cast<uint64_t>(D)) {
    // fewer points than devices (run_ensemble): split the runs evenly; the
    // statistics of a point cut by a part edge are Chan-merged across its parts
    const uint64_t n_chunks = std::min<uint64_t>(S, static_cast<uint64_t>(D));
    for (uint64_t c = 1; c < n_chunks; ++c) bounds.push_back(s0 + S * c / n_chunks);
  } else if (D > 1) {
    // a range that cuts points: D whole-point chunks (edges snapped to points)
    for (int c = 1; c < D; ++c) {
      uint64_t b = s0 + S * c / D;
      b = (b + R - 1) / R * R;
      b = std::min(std::max(b, bounds.back()), s1);
      bounds.push_back(b);
    }
  }
  bounds.push_back(s1);
  for (size_t c = 0; c + 1 < bounds.size(); ++c) {
    if (bounds[c] >= bounds[c + 1]) continue;
    PlanPart p;
    p.dev = static_cast<int>(c % D);
    p.s0 = bounds[c];
    p.s1 = bounds[c + 1];
    p.out_first = bounds[c] - s0;
    parts->push_back(p);
  }
  return KIN_OK;
}

// ---- model (ReactionNetwork::create, model.hpp:47-53) -------------------------
struct HostModel {
  int n = 0, m = 0;
  std::vector<double> x0, rate_base, params;
  std::vector<int> rate_param;
  std::vector<int> rt_ptr, rt_species, rt_stoich;
  std::vector<int> col_ptr, col_species, col_delta;
  std::vector<int> row_ptr, row_reaction, row_delta;
  std::vector<int> g;
  int fprop = 0;
};

int load_model(const kin_model_desc* d, HostModel* H, std::string* msg) {
  if (!d) { *msg = "null model descriptor"; return KIN_ERR_USAGE; }
  const int n = d->n_species, m = d->n_reactions, np = d->n_params;
  if (n < 0 || m < 0 || np < 0) { *msg = "negative model dimension"; return KIN_ERR_INPUT; }
  if (n > 4096 || m > 8192) { *msg = "model too large for the device tables"; return KIN_ERR_INPUT; }
  if ((n > 0 && !d->initial_amounts) || (m > 0 && (!d->rate_constants || !d->reactant_ptr || !d->product_ptr)) ||
      (np > 0 && !d->param_values)) {
    *msg = "missing model array";
    return KIN_ERR_USAGE;
  }
  const int max_order = d->max_order <= 0 ? 2 : d->max_order;
  if (max_order > 3) { *msg = "max_order above 3 is not supported"; return KIN_ERR_INPUT; }
  HostModel& M = *H;
  M = HostModel{};
  M.n = n;
  M.m = m;
  for (int i = 0; i < n; ++i) {
    if (d->initial_amounts[i] < 0) { *msg = "species " + std::to_string(i) + ": negative initial amount"; return KIN_ERR_INPUT; }
    M.x0.push_back(static_cast<double>(d->initial_amounts[i]));
  }
  for (int p = 0; p < np; ++p) {
    if (!(d->param_values[p] > 0.0) || !std::isfinite(d->param_values[p])) {
      *msg = "param " + std::to_string(p) + ": rate must be positive";
      return KIN_ERR_INPUT;
    }
    M.params.push_back(d->param_values[p]);
  }
  std::vector<int> nu(static_cast<size_t>(n) * m, 0);
  M.g.assign(n, 1);
  M.rt_ptr.push_back(0);
  M.col_ptr.push_back(0);
  for (int j = 0; j < m; ++j) {
    const int rp = d->rate_param ? d->rate_param[j] : -1;
    if (rp >= np || rp < -1) { *msg = "reaction " + std::to_string(j) + ": unknown parameter"; return KIN_ERR_INPUT; }
    const double c = rp >= 0 ? d->param_values[rp] : d->rate_constants[j];
    if (!(c > 0.0) || !std::isfinite(c)) { *msg = "reaction " + std::to_string(j) + ": rate must be positive"; return KIN_ERR_INPUT; }
    M.rate_base.push_back(d->rate_constants[j]);
    M.rate_param.push_back(rp);
    int order = 0, prev = -1;
    for (int p = d->reactant_ptr[j]; p < d->reactant_ptr[j + 1]; ++p) {
      const int s = d->reactant_species[p], st = d->reactant_stoich[p];
      if (s < 0 || s >= n) { *msg = "reaction " + std::to_string(j) + ": undeclared species"; return KIN_ERR_INPUT; }
      if (s <= prev) { *msg = "reaction " + std::to_string(j) + ": reactants must be species-ascending and unique"; return KIN_ERR_INPUT; }
      if (st <= 0) { *msg = "reaction " + std::to_string(j) + ": stoichiometry must be positive"; return KIN_ERR_INPUT; }
      prev = s;
      order += st;
      M.rt_species.push_back(s);
      M.rt_stoich.push_back(st);
      M.fprop += 1 + (st <= 1 ? 0 : (st == 2 ? 3 : 5));
      nu[static_cast<size_t>(s) * m + j] -= st;
    }
    if (order > max_order) {
      *msg = "reaction " + std::to_string(j) + ": reactant order " + std::to_string(order) + " exceeds " + std::to_string(max_order);
      return KIN_ERR_INPUT;
    }
    for (int p = d->reactant_ptr[j]; p < d->reactant_ptr[j + 1]; ++p)
      M.g[d->reactant_species[p]] = std::max(M.g[d->reactant_species[p]], order);
    prev = -1;
    for (int p = d->product_ptr[j]; p < d->product_ptr[j + 1]; ++p) {
      const int s = d->product_species[p], st = d->product_stoich[p];
      if (s < 0 || s >= n) { *msg = "reaction " + std::to_string(j) + ": undeclared species"; return KIN_ERR_INPUT; }
      if (s <= prev) { *msg = "reaction " + std::to_string(j) + ": products must be species-ascending and unique"; return KIN_ERR_INPUT; }
      if (st <= 0) { *msg = "reaction " + std::to_string(j) + ": stoichiometry must be positive"; return KIN_ERR_INPUT; }
      prev = s;
      nu[static_cast<size_t>(s) * m + j] += st;
    }
    M.rt_ptr.push_back(static_cast<int>(M.rt_species.size()));
    for (int s = 0; s < n; ++s) {
      const int dl = nu[static_cast<size_t>(s) * m + j];
      if (dl == 0) continue;
      if (dl < -128 || dl > 127) {
        *msg = "reaction " + std::to_string(j) + ": net stoichiometry " + std::to_string(dl) +
               " out of range (the device tables hold net changes in [-128, 127])";
        return KIN_ERR_INPUT;
      }
      M.col_species.push_back(s);
      M.col_delta.push_back(dl);
    }
    M.col_ptr.push_back(static_cast<int>(M.col_species.size()));
  }
  M.row_ptr.push_back(0);
  for (int s = 0; s < n; ++s) {
    for (int j = 0; j < m; ++j) {
      const int dl = nu[static_cast<size_t>(s) * m + j];
      if (dl != 0) { M.row_reaction.push_back(j); M.row_delta.push_back(dl); }
    }
    M.row_ptr.push_back(static_cast<int>(M.row_reaction.size()));
  }
  return KIN_OK;
}

// ---- sweep validation (SweepConfig, ensemble.hpp:101-113) ----
struct Layout {
  uint64_t P = 1, R = 1, S = 1;
};

int sweep_layout(const kin_sweep_desc* d, Layout* L, std::string* msg) {
  if (!d) { *msg = "null sweep descriptor"; return KIN_ERR_USAGE; }
  if (d->n_axes < 0 || d->n_axes > KIN_MAX_AXES || (d->n_axes > 0 && !d->axes)) {
    *msg = "at most " + std::to_string(KIN_MAX_AXES) + " sweep axes";
    return KIN_ERR_INPUT;
  }
  uint64_t P = 1;
  for (int ax = 0; ax < d->n_axes; ++ax) {
    const kin_sweep_axis& A = d->axes[ax];
    if (A.n_values <= 0 || !A.values) { *msg = "axis " + std::to_string(ax) + ": empty value list"; return KIN_ERR_INPUT; }
    if (P > (uint64_t{1} << 40) / static_cast<uint64_t>(A.n_values)) { *msg = "sweep too large"; return KIN_ERR_INPUT; }
    P *= static_cast<uint64_t>(A.n_values);
  }
  if (d->runs_per_point == 0) { *msg = "runs_per_point must be >= 1"; return KIN_ERR_INPUT; }
  L->P = P;
  L->R = d->runs_per_point;
  L->S = P * d->runs_per_point;
  return KIN_OK;
}

int validate_sweep(const HostModel& net, const kin_sweep_desc* d, const Layout& L, std::string* msg) {
  const kin_method& M = d->method;
  if (M.kind == KIN_METHOD_HYBRID &&
      !(M.theta_x >= 0.0 && M.theta_a >= 0.0 && M.repartition_interval >= 0.0)) {
    *msg = "hybrid thresholds and repartition interval must be non-negative";
    return KIN_ERR_INPUT;
  }
  if (M.kind < 0 || M.kind > KIN_METHOD_LSODA) { *msg = "unknown method kind"; return KIN_ERR_INPUT; }
  if ((M.kind == KIN_METHOD_TAU_FIXED || M.kind == KIN_METHOD_CLE) && !(M.tau > 0.0)) { *msg = "tau must be positive"; return KIN_ERR_INPUT; }
  if (M.kind == KIN_METHOD_TAU_ADAPTIVE && !(M.epsilon > 0.0 && M.epsilon < 1.0)) { *msg = "epsilon must be in (0,1)"; return KIN_ERR_INPUT; }
  if (M.integrator.max_steps == 0) { *msg = "max_steps must be positive"; return KIN_ERR_INPUT; }
  if ((M.kind == KIN_METHOD_ODE || M.kind == KIN_METHOD_LSODA || M.kind == KIN_METHOD_HYBRID) &&
      !(M.integrator.rel_tol > 0.0 && M.integrator.abs_tol > 0.0)) {
    *msg = "tolerances must be positive";
    return KIN_ERR_INPUT;
  }
  if (!(d->t_end >= 0.0) || !std::isfinite(d->t_end)) { *msg = "t_end must be finite and non-negative"; return KIN_ERR_INPUT; }
  if (d->n_grid < 0 || (d->n_grid > 0 && !d->grid)) { *msg = "bad grid"; return KIN_ERR_USAGE; }
  for (int g = 0; g < d->n_grid; ++g) {
    if (!(d->grid[g] >= 0.0 && d->grid[g] <= d->t_end)) { *msg = "grid point outside [0, t_end]"; return KIN_ERR_INPUT; }
    if (g > 0 && !(d->grid[g] > d->grid[g - 1])) { *msg = "grid must be strictly increasing"; return KIN_ERR_INPUT; }
  }
  for (int ax = 0; ax < d->n_axes; ++ax) {
    const kin_sweep_axis& A = d->axes[ax];
    if (A.kind == KIN_AXIS_PARAM) {
      if (A.index < 0 || A.index >= static_cast<int>(net.params.size())) {
        *msg = "axis " + std::to_string(ax) + ": unknown parameter";
        return KIN_ERR_INPUT;
      }
      for (int v = 0; v < A.n_values; ++v)
        if (!(A.values[v] > 0.0) || !std::isfinite(A.values[v])) {
          *msg = "axis " + std::to_string(ax) + ": rate values must be positive";
          return KIN_ERR_INPUT;
        }
    } else if (A.kind == KIN_AXIS_INITIAL) {
      if (A.index < 0 || A.index >= net.n) { *msg = "axis " + std::to_string(ax) + ": unknown species"; return KIN_ERR_INPUT; }
      for (int v = 0; v < A.n_values; ++v)
        if (!(A.values[v] >= 0.0) || A.values[v] != std::floor(A.values[v]) || A.values[v] > 9007199254740992.0) {
          *msg = "axis " + std::to_string(ax) + ": initial amounts must be non-negative integers";
          return KIN_ERR_INPUT;
        }
    } else if (A.kind == KIN_AXIS_SCALE) {
      if (A.index < 0 || A.span <= 0 || A.index + A.span > net.m) {
        *msg = "axis " + std::to_string(ax) + ": scale range outside the reactions";
        return KIN_ERR_INPUT;
      }
      for (int v = 0; v < A.n_values; ++v)
        if (!(A.values[v] > 0.0) || !std::isfinite(A.values[v])) {
          *msg = "axis " + std::to_string(ax) + ": scale factors must be positive";
          return KIN_ERR_INPUT;
        }
    } else {
      *msg = "axis " + std::to_string(ax) + ": unknown axis kind";
      return KIN_ERR_INPUT;
    }
  }
  {  // every reaction's rate follows at most one axis
    std::vector<int> bound(net.m, -1);
    for (int ax = 0; ax < d->n_axes; ++ax) {
      const kin_sweep_axis& A = d->axes[ax];
      for (int j = 0; j < net.m; ++j) {
        const bool hit = A.kind == KIN_AXIS_PARAM ? net.rate_param[j] == A.index
                                                  : (A.kind == KIN_AXIS_SCALE && j >= A.index && j < A.index + A.span);
        if (!hit) continue;
        if (bound[j] >= 0) {
          *msg = "reaction " + std::to_string(j) + ": rate bound to two sweep axes";
          return KIN_ERR_INPUT;
        }
        bound[j] = ax;
      }
    }
  }
  if (d->seed_mode == KIN_SEED_DIRECT && L.S != 1) { *msg = "direct seeding needs exactly one simulation"; return KIN_ERR_INPUT; }
  if (d->rng_mode != KIN_RNG_COMPAT && d->rng_mode != KIN_RNG_PHILOX) { *msg = "unknown rng_mode"; return KIN_ERR_INPUT; }
  if (M.firing != KIN_FIRING_POISSON && M.firing != KIN_FIRING_BINOMIAL) { *msg = "unknown firing law"; return KIN_ERR_INPUT; }
  if (d->output_mode != KIN_OUTPUT_FULL && d->output_mode != KIN_OUTPUT_STATS_ONLY) { *msg = "unknown output_mode"; return KIN_ERR_INPUT; }
  if (d->lanes_per_sim < 0 || d->lanes_per_sim > 32) { *msg = "lanes_per_sim must be in [0, 32]"; return KIN_ERR_INPUT; }
  if (d->shard_count < 0 || (d->shard_count > 1 && (d->shard_index < 0 || d->shard_index >= d->shard_count))) {
    *msg = "shard_index out of range";
    return KIN_ERR_INPUT;
  }
  return KIN_OK;
}

// Pack the model + the sweep's axis bindings into the kernel-parameter tables.
int pack_tables(const HostModel& H, const kin_sweep_desc* d, KinTables* T, std::string* msg) {
  std::memset(T, 0, sizeof(KinTables));
  T->n = H.n;
  T->m = H.m;
  T->nnz = static_cast<int32_t>(H.col_species.size());
  T->n_grid = d->n_grid;
  T->fprop = H.fprop;
  // effective parameter values (non-swept) and which axis overrides what
  std::vector<int> param_axis(H.params.size(), -1), x0_axis(H.n, -1);
  for (int ax = 0; ax < d->n_axes; ++ax) {
    if (d->axes[ax].kind == KIN_AXIS_PARAM) param_axis[d->axes[ax].index] = ax;
    else if (d->axes[ax].kind == KIN_AXIS_INITIAL) x0_axis[d->axes[ax].index] = ax;
  }
  size_t off = 0;
  bool overflow = false;
  auto put = [&](const void* src, size_t bytes, size_t align) -> uint32_t {
    off = (off + align - 1) / align * align;
    if (off + bytes > KIN_TABLE_BYTES) { overflow = true; return 0; }
    const uint32_t at = static_cast<uint32_t>(off);
    if (bytes) std::memcpy(T->blob + off, src, bytes);
    off += bytes;
    return at;
  };
  // rate table: c_j with non-swept parameters resolved; a reaction on a sweep
  // axis takes rate[j] * (axis value) — rate[j] = 1 for a parameter axis (exact:
  // the value itself), its own constant for a scale axis
  std::vector<double> rate(H.m);
  std::vector<int8_t> rate_axis(H.m, -1);
  for (int j = 0; j < H.m; ++j) {
    const int rp = H.rate_param[j];
    rate[j] = rp >= 0 ? H.params[rp] : H.rate_base[j];
    if (rp >= 0 && param_axis[rp] >= 0) {
      rate_axis[j] = static_cast<int8_t>(param_axis[rp]);
      rate[j] = 1.0;
    }
  }
  for (int ax = 0; ax < d->n_axes; ++ax)
    if (d->axes[ax].kind == KIN_AXIS_SCALE)
      for (int j = d->axes[ax].index; j < d->axes[ax].index + d->axes[ax].span; ++j) rate_axis[j] = static_cast<int8_t>(ax);
  std::vector<int8_t> x0ax(H.n);
  for (int i = 0; i < H.n; ++i) x0ax[i] = static_cast<int8_t>(x0_axis[i]);
  std::vector<double> gd(H.g.begin(), H.g.end());
  if (H.rt_species.size() > 32767 || H.col_species.size() > 32767) { *msg = "model too large for the device tables"; return KIN_ERR_INPUT; }
  std::vector<int16_t> rt_ptr(H.rt_ptr.begin(), H.rt_ptr.end()), col_ptr(H.col_ptr.begin(), H.col_ptr.end()),
      row_ptr(H.row_ptr.begin(), H.row_ptr.end());
  std::vector<uint32_t> rt(H.rt_species.size()), col(H.col_species.size()), row(H.row_reaction.size());
  for (size_t p = 0; p < rt.size(); ++p)
    rt[p] = static_cast<uint32_t>(H.rt_species[p]) | (static_cast<uint32_t>(H.rt_stoich[p]) << 16);
  for (size_t p = 0; p < col.size(); ++p)
    col[p] = static_cast<uint32_t>(H.col_species[p]) | (static_cast<uint32_t>(H.col_delta[p] + 128) << 16);
  for (size_t p = 0; p < row.size(); ++p)
    row[p] = static_cast<uint32_t>(H.row_reaction[p]) | (static_cast<uint32_t>(H.row_delta[p] + 128) << 16);
  for (size_t p = 0; p < H.rt_stoich.size(); ++p)
    if (H.rt_stoich[p] > 255) { *msg = "reactant stoichiometry above 255 is not supported by the device tables"; return KIN_ERR_INPUT; }
  T->off_rate = put(rate.data(), rate.size() * 8, 8);
  T->off_x0 = put(H.x0.data(), H.x0.size() * 8, 8);
  T->off_g = put(gd.data(), gd.size() * 8, 8);
  T->off_rt = put(rt.data(), rt.size() * 4, 4);
  T->off_col = put(col.data(), col.size() * 4, 4);
  T->off_row = put(row.data(), row.size() * 4, 4);
  T->off_rt_ptr = put(rt_ptr.data(), rt_ptr.size() * 2, 2);
  T->off_col_ptr = put(col_ptr.data(), col_ptr.size() * 2, 2);
  T->off_row_ptr = put(row_ptr.data(), row_ptr.size() * 2, 2);
  // compact reaction descriptors (<= 3 reactant terms, stoich <= 3 each)
  std::vector<uint64_t> rdesc(H.m, 0);
  for (int j = 0; j < H.m; ++j) {
    const int nt = H.rt_ptr[j + 1] - H.rt_ptr[j];
    if (nt > 3) { *msg = "reaction " + std::to_string(j) + ": more than 3 reactant species"; return KIN_ERR_INPUT; }
    uint64_t dsc = static_cast<uint64_t>(nt) << 54;
    for (int t = 0; t < nt; ++t) {
      const int p = H.rt_ptr[j] + t;
      dsc |= static_cast<uint64_t>(H.rt_species[p]) << (16 * t);
      dsc |= static_cast<uint64_t>(H.rt_stoich[p] & 3) << (48 + 2 * t);
    }
    dsc |= static_cast<uint64_t>(rate_axis[j] + 1) << 56;
    rdesc[j] = dsc;
  }
  // propensity dependency graph: firing j changes species col(j); every
  // reaction with one of them as a reactant must be re-evaluated.
  std::vector<int16_t> dep_ptr(1, 0);
  std::vector<uint16_t> dep;
  {
    std::vector<std::vector<int>> by_species(H.n);
    for (int k = 0; k < H.m; ++k)
      for (int p = H.rt_ptr[k]; p < H.rt_ptr[k + 1]; ++p) by_species[H.rt_species[p]].push_back(k);
    std::vector<char> mark(H.m);
    for (int j = 0; j < H.m; ++j) {
      std::fill(mark.begin(), mark.end(), 0);
      for (int p = H.col_ptr[j]; p < H.col_ptr[j + 1]; ++p)
        for (int k : by_species[H.col_species[p]]) mark[k] = 1;
      for (int k = 0; k < H.m; ++k)
        if (mark[k]) dep.push_back(static_cast<uint16_t>(k));
      if (dep.size() > 32767) { *msg = "model too large for the device tables"; return KIN_ERR_INPUT; }
      dep_ptr.push_back(static_cast<int16_t>(dep.size()));
    }
  }
  T->off_rdesc = put(rdesc.data(), rdesc.size() * 8, 8);
  T->off_dep = put(dep.data(), dep.size() * 2, 2);
  T->off_dep_ptr = put(dep_ptr.data(), dep_ptr.size() * 2, 2);
  T->off_rate_axis = put(rate_axis.data(), rate_axis.size(), 1);
  T->off_x0_axis = put(x0ax.data(), x0ax.size(), 1);
  if (overflow) { *msg = "model too large for the device tables"; return KIN_ERR_INPUT; }
  // Work-balancing orders for kernels that spread a simulation's species /
  // reactions over L lanes (Dopri5: lane l takes slots l, l+L, ...): sorted by
  // descending nu-row length / reactant-term count, so the lanes of a warp
  // walk rows of similar length together.  Optional (offset 0 = identity).
  {
    std::vector<int16_t> sp(H.n), rx(H.m);
    for (int i = 0; i < H.n; ++i) sp[i] = static_cast<int16_t>(i);
    for (int j = 0; j < H.m; ++j) rx[j] = static_cast<int16_t>(j);
    std::stable_sort(sp.begin(), sp.end(), [&](int16_t u, int16_t v) {
      return H.row_ptr[u + 1] - H.row_ptr[u] > H.row_ptr[v + 1] - H.row_ptr[v];
    });
    std::stable_sort(rx.begin(), rx.end(), [&](int16_t u, int16_t v) {
      return H.rt_ptr[u + 1] - H.rt_ptr[u] > H.rt_ptr[v + 1] - H.rt_ptr[v];
    });
    const size_t save = off;
    const uint32_t o1 = put(sp.data(), sp.size() * 2, 2);
    const uint32_t o2 = put(rx.data(), rx.size() * 2, 2);
    if (overflow || o1 == 0 || o2 == 0) {
      overflow = false;
      off = save;
      T->off_sp_perm = T->off_rx_perm = 0;
    } else {
      T->off_sp_perm = o1;
      T->off_rx_perm = o2;
    }
  }
  // the grid rides along when it fits (offset 0 = "use the global copy")
  const size_t save = off;
  const uint32_t og = put(d->grid, static_cast<size_t>(d->n_grid) * 8, 8);
  if (overflow || d->n_grid == 0 || og == 0) {
    overflow = false;
    off = save;
    T->off_grid = 0;
  } else {
    T->off_grid = og;
  }
  T->used = static_cast<uint32_t>(off);
  return KIN_OK;
}

// ---- LSODA coefficients (cfode; same recurrences as oracle/kin_lsoda.hpp) ------
void lsoda_coeffs(std::vector<double>* out) {
  double elco[2][13][14] = {};
  double tesco[2][13][3] = {};
  {
    double pc[13];
    elco[0][1][0] = 1.0;
    elco[0][1][1] = 1.0;
    tesco[0][1][0] = 0.0;
    tesco[0][1][1] = 2.0;
    tesco[0][2][0] = 1.0;
    tesco[0][12][2] = 0.0;
    pc[0] = 1.0;
    double rqfac = 1.0;
    for (int nq = 2; nq <= 12; ++nq) {
      const double rq1fac = rqfac;
      rqfac = rqfac / nq;
      const int nqm1 = nq - 1;
      const double fnqm1 = nqm1;
      pc[nq - 1] = 0.0;
      for (int i = nq - 1; i >= 1; --i) pc[i] = pc[i - 1] + fnqm1 * pc[i];
      pc[0] = fnqm1 * pc[0];
      double pint = pc[0], xpin = pc[0] / 2.0, tsign = 1.0;
      for (int i = 1; i < nq; ++i) {
        tsign = -tsign;
        pint += tsign * pc[i] / (i + 1);
        xpin += tsign * pc[i] / (i + 2);
      }
      elco[0][nq][0] = pint * rq1fac;
      elco[0][nq][1] = 1.0;
      for (int i = 1; i < nq; ++i) elco[0][nq][i + 1] = rq1fac * pc[i] / (i + 1);
      const double agamq = rqfac * xpin;
      const double ragq = 1.0 / agamq;
      tesco[0][nq][1] = ragq;
      if (nq < 12) tesco[0][nq + 1][0] = ragq * rqfac / (nq + 1);
      tesco[0][nq - 1][2] = ragq;
    }
  }
  {
    double pc[7];
    pc[0] = 1.0;
    double rq1fac = 1.0;
    for (int nq = 1; nq <= 5; ++nq) {
      const double fnq = nq;
      pc[nq] = 0.0;
      for (int i = nq; i >= 1; --i) pc[i] = pc[i - 1] + fnq * pc[i];
      pc[0] = fnq * pc[0];
      for (int i = 0; i <= nq; ++i) elco[1][nq][i] = pc[i] / pc[1];
      elco[1][nq][1] = 1.0;
      tesco[1][nq][0] = rq1fac;
      tesco[1][nq][1] = (nq + 1) / elco[1][nq][0];
      tesco[1][nq][2] = (nq + 2) / elco[1][nq][0];
      rq1fac = rq1fac / fnq;
    }
  }
  out->assign(&elco[0][0][0], &elco[0][0][0] + 2 * 13 * 14);
  out->insert(out->end(), &tesco[0][0][0], &tesco[0][0][0] + 2 * 13 * 3);
}

// ---- device slots -------------------------------------------------------------
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Per-launch device state: outputs, scratch, the launch record used by the
// int32-overflow retry, and the events ordering compute -> copy-out.  A slot
// owns one Buffers for the device-resident API (kin_sweep_launch/fetch) and a
// pool reused by asynchronous jobs (kin_sweep_submit/wait).
struct Buffers {
  DevBuf<double> traj, mean, m2, axis, grid;
  DevBuf<double> gstate;  // per-warp simulation state in global memory (large models)
  DevBuf<uint64_t> meta, work;
  DevBuf<int32_t> status;
  DevBuf<unsigned long long> counter;
  DevBuf<int> ovf;
  int* ovf_host = nullptr;  // pinned copy of the overflow flag
  cudaStream_t st = nullptr;  // compute stream of this launch (one of the slot's)
  cudaStream_t cs = nullptr;  // copy stream of its async copy-out (paired with st)
  cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};  // sim start, sim end, stats end
  cudaEvent_t ev_done = nullptr, ev_copied = nullptr;
  bool timed_stats = false;
  uint64_t s0 = 0, s1 = 0, P0 = 0, nP = 0, R = 1;
  PlanPart part;  // the caller-layout mapping of this launch (copy_out)
  int G = 0, N = 0;
  bool have_stats = false, have_work = false, valid = false;
  bool stats_only = false;     // KIN_OUTPUT_STATS_ONLY launch: no trajectory copy-out
  uint64_t base_point = 0, point_end = 0;  // device-resident form: the call's point range
  uint64_t stats_row0 = 0;     // first whole point's row in mean/m2
  std::unique_ptr<KinTables> last_T;
  KinSweepDev last_SD{};
  KinOutDev last_O{};
  bool last_int_state = false, last_count = false, pending_check = false, last_jit = false;
  const char* kernel_name = "";
  uint64_t last_base = 0, last_S = 0;
  int last_gn = 0;
  // statistics of the (at most two) points this chunk holds only some runs of
  // (chunk edges inside a point): Welford over the chunk's runs, merged across
  // chunks by kin_sweep_wait (Chan, ascending chunk order)
  DevBuf<double> pmean, pm2;                     // [n_partial][gn]
  double* h_pmean = nullptr;                     // pinned copies
  double* h_pm2 = nullptr;
  size_t h_pcap = 0;
  int n_partial = 0;
  uint64_t partial_point[2] = {0, 0}, partial_n[2] = {0, 0}, partial_base[2] = {0, 0};
  void release() {
    traj.release(); mean.release(); m2.release(); axis.release(); grid.release(); gstate.release();
    pmean.release(); pm2.release();
    if (h_pmean) cudaFreeHost(h_pmean);
    if (h_pm2) cudaFreeHost(h_pm2);
    h_pmean = h_pm2 = nullptr;
    h_pcap = 0;
    meta.release(); work.release(); status.release(); counter.release(); ovf.release();
    if (ovf_host) cudaFreeHost(ovf_host);
    ovf_host = nullptr;
    for (auto& e : tev) if (e) cudaEventDestroy(e);
    if (ev_done) cudaEventDestroy(ev_done);
    if (ev_copied) cudaEventDestroy(ev_copied);
    ev_done = ev_copied = nullptr;
    for (auto& e : tev) e = nullptr;
  }
};

struct Slot {
  int device = 0;
  cudaStream_t stream = nullptr;       // kernels (device-resident API; every other async job)
  cudaStream_t aux_stream = nullptr;   // kernels of the alternate async jobs: two independent
                                       // sweeps in flight overlap (one fills the SMs the
                                       // other's tail leaves idle)
  cudaStream_t copy_stream = nullptr;  // copy-out of the async jobs on `stream`
  cudaStream_t aux_copy_stream = nullptr;  // ... and of those on `aux_stream`: a job's D2H
                                           // starts when its own kernel ends, not behind
                                           // the other stream's (longer) job
  unsigned job_rr = 0;
  DevBuf<double> lgamma_tab;  // glibc lgamma(k+1), k < KIN_LGAMMA_N
  DevBuf<double> lsoda_co;    // cfode elco/tesco
  void* stage = nullptr;
  size_t stage_cap = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  Buffers main;
  std::vector<std::unique_ptr<Buffers>> pool;
  std::mutex mu;
};

struct Job {
  struct Part {
    int slot;
    Buffers* buf;
  };
  std::vector<Part> parts;
  kin_sweep_out out{};
  uint64_t s0 = 0, s1 = 0, base_point = 0;
  uint64_t n_local = 0, np_local = 0;  // caller-local simulations / statistics points
  int sh_i = 0, sh_n = 1;
  Layout L;
  // global simulation index of caller-local simulation s
  uint64_t global_of(uint64_t s) const {
    if (sh_n <= 1) return s0 + s;
    const uint64_t k = s / L.R;
    return (s0 / L.R + sh_i + static_cast<uint64_t>(sh_n) * k) * L.R + (s - k * L.R);
  }
  int32_t* status_pinned = nullptr;  // when the caller did not ask for status
  int rc = KIN_OK;
  kin_error err{};
};

}  // namespace

struct kin_ctx {
  std::vector<std::unique_ptr<Slot>> slots;
  std::mutex jobs_mu;
  uint64_t next_ticket = 1;
  std::map<uint64_t, std::unique_ptr<Job>> jobs;
};

struct kin_model {
  kin_ctx* ctx;
  HostModel host;
  // per-model JIT policies, one per sweep-axis binding of the rates (generated
  // once, not per launch)
  std::mutex jit_mu;
  std::map<std::vector<int>, std::unique_ptr<kin::JitModel>> jit_cache;
};

namespace {

int cuda_fail(kin_error* err, cudaError_t e, const char* what) {
  set_err(err, KIN_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
  return KIN_ERR_DEVICE;
}

#define KIN_CUDA(call, what)                        \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_fail(err, e_, what); \
  } while (0)

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// D2H into a caller buffer on `st`: asynchronous when the destination is pinned
// (sync=false leaves it in flight), else staged through a pinned double buffer
// (always synchronous).
int copy_d2h(Slot& sl, cudaStream_t st, void* dst, const void* src, size_t bytes, bool sync, kin_error* err) {
  if (bytes == 0) return KIN_OK;
  if (is_pinned(dst)) {
    KIN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    if (sync) KIN_CUDA(cudaStreamSynchronize(st), "D2H sync");
    return KIN_OK;
  }
  const size_t piece = size_t{32} << 20;
  if (!sl.stage) {
    KIN_CUDA(cudaMallocHost(&sl.stage, 2 * piece), "pinned staging");
    sl.stage_cap = 2 * piece;
    KIN_CUDA(cudaEventCreateWithFlags(&sl.ev[0], cudaEventDisableTiming), "event");
    KIN_CUDA(cudaEventCreateWithFlags(&sl.ev[1], cudaEventDisableTiming), "event");
  }
  char* out = static_cast<char*>(dst);
  const char* in = static_cast<const char*>(src);
  char* buf[2] = {static_cast<char*>(sl.stage), static_cast<char*>(sl.stage) + piece};
  size_t pending_off = 0, pending_len = 0;
  int pending_b = -1, b = 0;
  for (size_t off = 0; off < bytes; off += piece) {
    const size_t len = std::min(piece, bytes - off);
    KIN_CUDA(cudaMemcpyAsync(buf[b], in + off, len, cudaMemcpyDeviceToHost, st), "D2H");
    KIN_CUDA(cudaEventRecord(sl.ev[b], st), "event");
    if (pending_b >= 0) {
      KIN_CUDA(cudaEventSynchronize(sl.ev[pending_b]), "D2H sync");
      std::memcpy(out + pending_off, buf[pending_b], pending_len);
    }
    pending_b = b;
    pending_off = off;
    pending_len = len;
    b ^= 1;
  }
  KIN_CUDA(cudaEventSynchronize(sl.ev[pending_b]), "D2H sync");
  std::memcpy(out + pending_off, buf[pending_b], pending_len);
  return KIN_OK;
}

// `rows` contiguous device rows of row_bytes each into host rows dpitch bytes
// apart (an interleaved part's points into the caller's layout): one 2D copy
// into pinned memory, else row by row through the staging path.
int copy_d2h_rows(Slot& sl, cudaStream_t st, void* dst, size_t dpitch, const void* src, size_t row_bytes,
                  uint64_t rows, bool sync, kin_error* err) {
  if (rows == 0 || row_bytes == 0) return KIN_OK;
  if (rows == 1 || dpitch == row_bytes) return copy_d2h(sl, st, dst, src, row_bytes * rows, sync, err);
  if (is_pinned(dst)) {
    KIN_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, row_bytes, row_bytes, rows, cudaMemcpyDeviceToHost, st), "D2H 2D");
    if (sync) KIN_CUDA(cudaStreamSynchronize(st), "D2H sync");
    return KIN_OK;
  }
  // pageable: gather whole rows through a pinned bounce buffer
  const size_t piece = size_t{32} << 20;
  const uint64_t per = std::max<uint64_t>(1, piece / row_bytes);
  std::vector<char> tmp;
  for (uint64_t r0 = 0; r0 < rows; r0 += per) {
    const uint64_t nr = std::min<uint64_t>(per, rows - r0);
    tmp.resize(nr * row_bytes);
    if (int rc = copy_d2h(sl, st, tmp.data(), static_cast<const char*>(src) + r0 * row_bytes, nr * row_bytes, true, err))
      return rc;
    for (uint64_t r = 0; r < nr; ++r)
      std::memcpy(static_cast<char*>(dst) + (r0 + r) * dpitch, tmp.data() + r * row_bytes, row_bytes);
  }
  return KIN_OK;
}

// Model structure + sweep binding for the per-model JIT kernel.
kin::JitModel jit_model(const HostModel& H, const kin_sweep_desc* d) {
  kin::JitModel j;
  j.n = H.n;
  j.m = H.m;
  j.rt_ptr = H.rt_ptr;
  j.rt_species = H.rt_species;
  j.rt_stoich = H.rt_stoich;
  j.col_ptr = H.col_ptr;
  j.col_species = H.col_species;
  j.col_delta = H.col_delta;
  j.row_ptr = H.row_ptr;
  j.row_reaction = H.row_reaction;
  j.row_delta = H.row_delta;
  j.g.assign(H.g.begin(), H.g.end());
  std::vector<int> param_axis(H.params.size(), -1);
  for (int ax = 0; ax < d->n_axes; ++ax)
    if (d->axes[ax].kind == KIN_AXIS_PARAM) param_axis[d->axes[ax].index] = ax;
  j.rate_axis.assign(H.m, -1);
  j.rate_scaled.assign(H.m, 0);
  for (int r = 0; r < H.m; ++r)
    if (H.rate_param[r] >= 0) j.rate_axis[r] = param_axis[H.rate_param[r]];
  for (int ax = 0; ax < d->n_axes; ++ax)
    if (d->axes[ax].kind == KIN_AXIS_SCALE)
      for (int r = d->axes[ax].index; r < d->axes[ax].index + d->axes[ax].span; ++r) {
        j.rate_axis[r] = ax;
        j.rate_scaled[r] = 1;
      }
  // dependency graph (same construction as pack_tables)
  std::vector<std::vector<int>> by_species(H.n);
  for (int k = 0; k < H.m; ++k)
    for (int p = H.rt_ptr[k]; p < H.rt_ptr[k + 1]; ++p) by_species[H.rt_species[p]].push_back(k);
  std::vector<char> mark(H.m);
  j.dep_ptr.push_back(0);
  for (int r = 0; r < H.m; ++r) {
    std::fill(mark.begin(), mark.end(), 0);
    for (int p = H.col_ptr[r]; p < H.col_ptr[r + 1]; ++p)
      for (int k : by_species[H.col_species[p]]) mark[k] = 1;
    for (int k = 0; k < H.m; ++k)
      if (mark[k]) j.dep.push_back(k);
    j.dep_ptr.push_back(static_cast<int>(j.dep.size()));
  }
  return j;
}

// The model's JIT policy for this sweep's rate bindings, built once per binding.
const kin::JitModel& jit_model_cached(const kin_model* model, const kin_sweep_desc* d) {
  kin_model* m = const_cast<kin_model*>(model);
  std::vector<int> key(m->host.m, -1);
  std::vector<int> param_axis(m->host.params.size(), -1);
  for (int ax = 0; ax < d->n_axes; ++ax)
    if (d->axes[ax].kind == KIN_AXIS_PARAM) param_axis[d->axes[ax].index] = ax;
  for (int r = 0; r < m->host.m; ++r)
    if (m->host.rate_param[r] >= 0) key[r] = param_axis[m->host.rate_param[r]];
  for (int ax = 0; ax < d->n_axes; ++ax)  // scale axes: 1000 + axis (distinct from parameter bindings)
    if (d->axes[ax].kind == KIN_AXIS_SCALE)
      for (int r = d->axes[ax].index; r < d->axes[ax].index + d->axes[ax].span; ++r) key[r] = 1000 + ax;
  std::lock_guard<std::mutex> lk(m->jit_mu);
  auto it = m->jit_cache.find(key);
  if (it != m->jit_cache.end()) return *it->second;
  auto jm = std::make_unique<kin::JitModel>(jit_model(m->host, d));
  kin::jit_prepare(jm.get());
  const kin::JitModel& ref = *jm;
  m->jit_cache.emplace(std::move(key), std::move(jm));
  return ref;
}

// Statistics kernels of a FULL-mode launch (whole points, then the partial points).
int launch_stats(Slot& sl, Buffers& bf, kin_error* err) {
  (void)sl;
  const size_t gn = static_cast<size_t>(bf.last_gn);
  if (bf.have_stats) {
    cudaError_t e = kin::launch_point_stats(bf.traj.p, bf.last_gn, bf.R, bf.last_base, bf.nP, 0, bf.mean.p, bf.m2.p,
                                            bf.st);
    if (e != cudaSuccess) return cuda_fail(err, e, "statistics kernel launch");
  }
  for (int k = 0; k < bf.n_partial; ++k) {
    cudaError_t e = kin::launch_point_stats(bf.traj.p, bf.last_gn, bf.partial_n[k], bf.partial_base[k], 1, 0,
                                            bf.pmean.p + k * gn, bf.pm2.p + k * gn, bf.st);
    if (e != cudaSuccess) return cuda_fail(err, e, "statistics kernel launch");
  }
  return KIN_OK;
}

// The simulation kernel of one launch (SD.local_begin / SD.n_local select the
// simulations; O is indexed from 0).  Picks the kernel variant from the method,
// the descriptor (lanes_per_sim, variant flags), the model's size and — for
// studies and tests only — the process's environment overrides.
int launch_sim(Slot& sl, Buffers& bf, const kin_model* model, const kin_sweep_desc* d, KinTables& T,
               KinSweepDev& SD, const KinOutDev& O, bool want_work, bool allow_int_state, kin_error* err) {
  NvtxRange nv("kin: simulation kernel launch");
  const HostModel& H = model->host;
  const EnvOverrides& ov = env_overrides();
  const uint32_t var = d->variant;
  const uint64_t S = SD.n_local;
  auto pick_gstate = [&](bool automatic, int env) {
    if (var & KIN_VARIANT_GLOBAL_STATE) return true;
    if (var & KIN_VARIANT_SMEM_STATE) return false;
    if (env >= 0) return env != 0;
    return automatic;
  };
  auto global_state_for = [&](size_t per_warp_doubles) -> int {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, sl.device);
    const uint64_t cap = std::min<uint64_t>((S + 31) / 32, static_cast<uint64_t>(sms) * 24);
    KIN_CUDA(bf.gstate.ensure(cap * per_warp_doubles), "cudaMalloc simulation state");
    SD.gstate = bf.gstate.p;
    SD.gstate_warps = cap;
    return KIN_OK;
  };
  cudaError_t e = cudaSuccess;
  const int kind = d->method.kind;
  bf.last_int_state = false;  // set below only by the int32-state stochastic launch
  if (kind == KIN_METHOD_ODE) {
    // lanes per simulation: the descriptor's, else by species count (ode_pick_lanes)
    const int ode_lanes = d->lanes_per_sim > 0 ? d->lanes_per_sim : ov.ode_lanes;
    e = kin::launch_dopri5(T, SD, O, want_work, ode_lanes, bf.st);
    bf.kernel_name = "dopri5_kernel";
  } else if (kind == KIN_METHOD_HYBRID) {
    KIN_CUDA(bf.counter.ensure(1), "cudaMalloc counter");
    // the Dopri5 vectors per simulation: in global memory when a warp's state
    // would take more than 48 KB of shared memory (<= 4 warps/SM, or no launch
    // at all above 227 KB).  (Measured on C1, 20.6 KB/warp: shared 97.5 ms,
    // global 100.4 ms.)
    if (pick_gstate(kin::hybrid_smem_bytes(T, SD) > 48 * 1024, ov.hybrid_gstate))
      if (int rc = global_state_for(kin::hybrid_state_doubles_per_warp(T, SD))) return rc;
    // the per-model JIT variant (straight-line propensities and row sums) for
    // the launches the JIT rule takes (>= 8,192 simulations, or forced)
    bool used = false;
    const int force_jit = (var & KIN_VARIANT_TABLE) ? 0 : ((var & KIN_VARIANT_JIT) ? 1 : -1);
    if (kin::jit_wanted(S, force_jit)) {
      const kin::JitModel& jm = jit_model_cached(model, d);
      e = kin::launch_hybrid_jit(jm, T, SD, O, want_work, bf.counter.p, SD.gstate ? 0 : kin::hybrid_smem_bytes(T, SD),
                                 bf.st, &used);
    }
    if (e == cudaSuccess && !used) e = kin::launch_hybrid(T, SD, O, want_work, bf.counter.p, bf.st);
    bf.kernel_name = used ? "kin_jit_hybrid" : "hybrid_kernel";
  } else if (kind == KIN_METHOD_CLE) {
    KIN_CUDA(bf.counter.ensure(1), "cudaMalloc counter");
    e = kin::launch_cle(T, SD, O, want_work, bf.counter.p, bf.st);
    bf.kernel_name = "cle_kernel";
  } else if (kind == KIN_METHOD_LSODA) {
    KIN_CUDA(bf.counter.ensure(1), "cudaMalloc counter");
    // Nordsieck array, Jacobian and LU per simulation: in global memory when a
    // warp's state would take more than 48 KB of shared memory
    if (pick_gstate(kin::lsoda_smem_bytes(T, SD) > 48 * 1024, ov.lsoda_gstate))
      if (int rc = global_state_for(kin::lsoda_state_doubles_per_warp(T, SD))) return rc;
    // the per-model JIT variant (straight-line RHS) for the launches the JIT
    // rule takes (>= 8,192 simulations, or forced)
    bool used = false;
    const int force_jit = (var & KIN_VARIANT_TABLE) ? 0 : ((var & KIN_VARIANT_JIT) ? 1 : -1);
    if (kin::jit_wanted(S, force_jit)) {
      const kin::JitModel& jm = jit_model_cached(model, d);
      e = kin::launch_lsoda_jit(jm, T, SD, O, sl.lsoda_co.p, want_work, bf.counter.p,
                                SD.gstate ? 0 : kin::lsoda_smem_bytes(T, SD), bf.st, &used);
    }
    if (e == cudaSuccess && !used) e = kin::launch_lsoda(T, SD, O, want_work, sl.lsoda_co.p, bf.counter.p, bf.st);
    bf.kernel_name = used ? "kin_jit_lsoda" : "lsoda_kernel";
  } else {
    KIN_CUDA(bf.counter.ensure(1), "cudaMalloc counter");
    KIN_CUDA(bf.ovf.ensure(1), "cudaMalloc overflow flag");
    // Philox mode: L lanes per simulation (the descriptor's lanes_per_sim; 1 =
    // one thread per simulation).  Compat mode is one thread per simulation:
    // the reference stream is sequential within a run.
    int lanes = d->lanes_per_sim > 0 ? d->lanes_per_sim : ov.group_lanes;
    if (d->rng_mode != KIN_RNG_PHILOX) {
      if (d->lanes_per_sim > 1) {
        set_err(err, KIN_ERR_INPUT, "lanes_per_sim > 1 needs rng_mode PHILOX for stochastic methods");
        return KIN_ERR_INPUT;
      }
      lanes = 1;
    } else if (lanes <= 0) {
      lanes = kin::stochastic_group_pick_lanes(H.n, H.m);
    }
    if (SD.firing == KIN_FIRING_BINOMIAL) lanes = 1;  // the binomial leap is sequential over reactions
    if (lanes != 1) {
      e = kin::launch_stochastic_group(T, SD, O, want_work, lanes, bf.counter.p, bf.st);
      bf.kernel_name = "stochastic_group_kernel";
    } else {
      // int32 amounts when every initial amount is far inside int32 range
      double xmax = 0.0;
      for (double v : H.x0) xmax = std::max(xmax, v);
      for (int ax = 0; ax < d->n_axes; ++ax)
        if (d->axes[ax].kind == KIN_AXIS_INITIAL)
          for (int v = 0; v < d->axes[ax].n_values; ++v) xmax = std::max(xmax, d->axes[ax].values[v]);
      bool int_state = allow_int_state && xmax < 1073741824.0 && !(var & KIN_VARIANT_DOUBLE_STATE) &&
                       ov.int_state != 0;
      // Large models: when a warp's state would take more than 24 KB of shared
      // memory (fewer than ~9 resident warps per SM), keep it in global memory
      // instead — same [slot][lane] layout, L1/L2-cached — and let registers
      // set the residency.
      const size_t smem_warp = static_cast<size_t>(T.m + SD.n_axes) * 32 * sizeof(double) +
                               static_cast<size_t>(T.n) * 32 * (int_state ? sizeof(int32_t) : sizeof(double));
      if (pick_gstate(smem_warp > 24 * 1024, ov.gstate)) {
        // sized for double amounts: the int32-overflow re-run reuses it
        if (int rc = global_state_for(static_cast<size_t>(T.m + SD.n_axes + T.n) * 32)) return rc;
        // amounts in shared memory, propensities in global (JIT kernel only;
        // it applies the size rule)
        SD.gstate_x_smem = !(var & KIN_VARIANT_NO_SPLIT) && ov.gstate_split != 0;
      }
      KIN_CUDA(cudaMemsetAsync(bf.ovf.p, 0, sizeof(int), bf.st), "memset");
      bool used = false;
      const int force_jit = (var & KIN_VARIANT_TABLE) ? 0 : ((var & KIN_VARIANT_JIT) ? 1 : -1);
      if (kin::jit_wanted(S, force_jit)) {
        const kin::JitModel& jm = jit_model_cached(model, d);
        e = kin::launch_stochastic_jit(jm, T, SD, O, want_work, bf.counter.p, bf.ovf.p, int_state, bf.st, &used);
      }
      if (e == cudaSuccess && !used)
        e = kin::launch_stochastic(T, SD, O, want_work, bf.counter.p, bf.ovf.p, int_state, bf.st);
      bf.last_jit = used;
      bf.kernel_name = used ? "kin_jit_stoch" : "stochastic_kernel";
      bf.last_int_state = int_state;
    }
    if (bf.last_int_state) {
      if (!bf.last_T) bf.last_T.reset(new KinTables);
      *bf.last_T = T;
      bf.last_SD = SD;
      bf.last_O = O;
      bf.last_count = want_work;
    }
  }
  if (e == cudaErrorInvalidConfiguration) {
    // the launchers' own pre-check: the per-simulation state of this model does
    // not fit the kernel's shared-memory budget (a property of the input)
    cudaGetLastError();
    set_err(err, KIN_ERR_INPUT,
            std::string("model too large for the ") + bf.kernel_name +
                " (per-simulation state exceeds the shared-memory budget)");
    return KIN_ERR_INPUT;
  }
  if (e != cudaSuccess) return cuda_fail(err, e, "simulation kernel launch");
  return KIN_OK;
}

// Device trajectory budget of a KIN_OUTPUT_STATS_ONLY launch (doubles): the
// runs stream through a buffer of at most this many samples.
constexpr size_t kStatsOnlyBudget = size_t{1} << 28;  // 2 GiB

// Launch one part of a call on a slot (device-resident results in bf).
int launch_range(Slot& sl, Buffers& bf, const kin_model* model, const kin_sweep_desc* d, const Layout& L,
                 const PlanPart& part, bool want_stats, bool want_work, kin_error* err, bool want_partials = false) {
  NvtxRange nv("kin: launch part (tables + H2D + kernels)");
  const HostModel& H = model->host;
  if (!bf.st) bf.st = sl.stream;
  KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
  KinTables* T = new KinTables;
  std::unique_ptr<KinTables> Tguard(T);
  std::string msg;
  if (int rc = pack_tables(H, d, T, &msg)) { set_err(err, rc, msg); return rc; }
  const uint64_t R = L.R;
  const uint64_t S = part.inter ? part.n_pts * R : part.s1 - part.s0;
  const int G = d->n_grid, N = H.n;
  const size_t gn = static_cast<size_t>(G) * N;
  const bool stats_only = d->output_mode == KIN_OUTPUT_STATS_ONLY;
  // trajectory buffer: every simulation (FULL) or a bounded run window (STATS_ONLY)
  uint64_t window = S;
  if (stats_only) {
    const uint64_t forced = d->variant >> 16;  // KIN_VARIANT_STATS_WINDOW (tests)
    window = forced ? forced : kStatsOnlyBudget / std::max<size_t>(gn, 1);
    window = std::max<uint64_t>(1, std::min<uint64_t>(S, window));
  }
  KIN_CUDA(bf.traj.ensure(std::max<size_t>(gn * window, 1)), "cudaMalloc traj");
  KIN_CUDA(bf.meta.ensure(std::max<uint64_t>(S * 6, 1)), "cudaMalloc meta");
  KIN_CUDA(bf.status.ensure(std::max<uint64_t>(S, 1)), "cudaMalloc status");
  if (want_work) KIN_CUDA(bf.work.ensure(std::max<uint64_t>(S, 1)), "cudaMalloc work");
  // axis values and grid
  size_t nax = 0;
  for (int ax = 0; ax < d->n_axes; ++ax) nax += d->axes[ax].n_values;
  KIN_CUDA(bf.axis.ensure(std::max<size_t>(nax, 1)), "cudaMalloc axes");
  KIN_CUDA(bf.grid.ensure(std::max<int>(G, 1)), "cudaMalloc grid");
  KinSweepDev SD;
  std::memset(&SD, 0, sizeof(SD));
  // simulations per warp of the thread-per-simulation stochastic kernels:
  // the descriptor's request (variant bits 8..13), else the launchers' fill rule
  SD.warp_lanes = static_cast<int32_t>((d->variant >> 8) & 0x3F);
  if (SD.warp_lanes > 32) SD.warp_lanes = 32;
  SD.kind = d->method.kind;
  SD.rng_mode = d->rng_mode;
  SD.tau = d->method.tau;
  SD.epsilon = d->method.epsilon;
  SD.firing = (SD.kind == KIN_METHOD_TAU_ADAPTIVE || SD.kind == KIN_METHOD_TAU_FIXED) ? d->method.firing : 0;
  SD.rel_tol = d->method.integrator.rel_tol;
  SD.abs_tol = d->method.integrator.abs_tol;
  SD.h_init = d->method.integrator.h_init;
  SD.h_max = d->method.integrator.h_max;
  SD.max_steps = d->method.integrator.max_steps;
  SD.hyb_theta_x = d->method.theta_x;
  SD.hyb_theta_a = d->method.theta_a;
  SD.hyb_rep = d->method.repartition_interval;
  SD.n_axes = d->n_axes;
  SD.seed_mode = d->seed_mode;
  size_t at = 0;
  for (int ax = 0; ax < d->n_axes; ++ax) {
    SD.axis_kind[ax] = d->axes[ax].kind;
    SD.axis_n[ax] = d->axes[ax].n_values;
    SD.axis_values[ax] = bf.axis.p + at;
    KIN_CUDA(cudaMemcpyAsync(bf.axis.p + at, d->axes[ax].values, sizeof(double) * d->axes[ax].n_values,
                             cudaMemcpyHostToDevice, bf.st), "H2D axes");
    at += d->axes[ax].n_values;
  }
  if (G) KIN_CUDA(cudaMemcpyAsync(bf.grid.p, d->grid, sizeof(double) * G, cudaMemcpyHostToDevice, bf.st), "H2D grid");
  SD.runs = R;
  SD.master_seed = d->master_seed;
  SD.sim_begin = part.inter ? 0 : part.s0;
  SD.pt_first = part.inter ? part.pt_first : 0;
  SD.pt_stride = part.inter ? part.pt_stride : 0;
  SD.local_begin = 0;
  SD.n_local = S;
  SD.t_end = d->t_end;
  SD.grid = bf.grid.p;
  SD.lgamma_tab = sl.lgamma_tab.p;
  if (!bf.tev[0])
    for (auto& ev : bf.tev) KIN_CUDA(cudaEventCreate(&ev), "event");
  KIN_CUDA(cudaEventRecord(bf.tev[0], bf.st), "event");
  // Points of this part, in part-local order: local point t holds part-local
  // simulations [t*R - off, (t+1)*R - off) clipped to [0, S) (off: the first
  // simulation's run index inside its point; interleaved parts are whole points).
  const uint64_t off = part.inter ? 0 : part.s0 % R;
  const uint64_t n_touch = S ? (S - 1 + off) / R + 1 : 0;
  const bool head_partial = off != 0;
  const bool tail_partial = S && (S + off) % R != 0;
  const uint64_t t_whole0 = head_partial ? 1 : 0;
  const uint64_t t_whole1 = tail_partial ? n_touch - 1 : n_touch;
  const uint64_t nP = t_whole1 > t_whole0 ? t_whole1 - t_whole0 : 0;
  bf.n_partial = 0;
  if (!stats_only) {
    KinOutDev O{bf.traj.p, bf.meta.p, bf.status.p, want_work ? bf.work.p : nullptr};
    if (int rc = launch_sim(sl, bf, model, d, *T, SD, O, want_work, true, err)) return rc;
    KIN_CUDA(cudaEventRecord(bf.tev[1], bf.st), "event");
    // per-point statistics for points entirely inside the part, and (when the
    // caller merges parts) partial statistics of the points cut by a part edge
    if (want_stats && want_partials && S) {
      auto add = [&](uint64_t l0, uint64_t l1) {
        const int k = bf.n_partial++;
        bf.partial_point[k] = (part.s0 + l0) / R;
        bf.partial_n[k] = l1 - l0;
        bf.partial_base[k] = l0;
      };
      if (head_partial) add(0, std::min(S, R - off));
      if (tail_partial && (n_touch > 1 || !head_partial)) add((n_touch - 1) * R - off, S);
    }
    bf.last_base = t_whole0 * R - off;
  } else {
    // STATS_ONLY: run-ascending windows of at most `window` simulations; after
    // each window the statistics kernel continues the Welford accumulators of
    // the points it touched (acc[t] = mean/m2 of local point t), so the result
    // is the same operation sequence as one Welford pass over all runs.
    SD.gstate_x_smem = 0;
    if (want_stats && n_touch) {
      KIN_CUDA(bf.mean.ensure(gn * n_touch), "cudaMalloc mean");
      KIN_CUDA(bf.m2.ensure(gn * n_touch), "cudaMalloc m2");
    }
    for (uint64_t l0 = 0; l0 < S; l0 += window) {
      const uint64_t l1 = std::min(S, l0 + window);
      KinSweepDev SW = SD;
      SW.local_begin = l0;
      SW.n_local = l1 - l0;
      KinOutDev O{bf.traj.p, bf.meta.p + l0 * 6, bf.status.p + l0, want_work ? bf.work.p + l0 : nullptr};
      if (int rc = launch_sim(sl, bf, model, d, *T, SW, O, want_work, false, err)) return rc;
      if (!want_stats) continue;
      // points touched by [l0, l1): a run of (t, first run in window, runs)
      uint64_t l = l0;
      while (l < l1) {
        const uint64_t t = (l + off) / R;
        const uint64_t t_begin = t * R > off ? t * R - off : 0;  // part-local first sim of point t
        const uint64_t t_end = std::min(S, (t + 1) * R - off);
        const uint64_t done = l - t_begin;                    // runs of t before this window
        if (done == 0 && t_end - t_begin == R && l + R <= l1) {
          // a run of whole fresh points
          const uint64_t k = std::min<uint64_t>((l1 - l) / R, t_whole1 > t ? t_whole1 - t : 1);
          cudaError_t e = kin::launch_point_stats(bf.traj.p, static_cast<int>(gn), R, l - l0, k, 0,
                                                  bf.mean.p + t * gn, bf.m2.p + t * gn, bf.st);
          if (e != cudaSuccess) return cuda_fail(err, e, "statistics kernel launch");
          l += k * R;
        } else {
          const uint64_t runs = std::min(t_end, l1) - l;
          cudaError_t e = kin::launch_point_stats(bf.traj.p, static_cast<int>(gn), runs, l - l0, 1, done,
                                                  bf.mean.p + t * gn, bf.m2.p + t * gn, bf.st);
          if (e != cudaSuccess) return cuda_fail(err, e, "statistics kernel launch");
          l += runs;
        }
      }
    }
    KIN_CUDA(cudaEventRecord(bf.tev[1], bf.st), "event");
    if (want_stats && want_partials && S) {
      auto add = [&](uint64_t t, uint64_t l0, uint64_t l1) {
        const int k = bf.n_partial++;
        bf.partial_point[k] = (part.s0 + l0) / R;
        bf.partial_n[k] = l1 - l0;
        bf.partial_base[k] = t;  // STATS_ONLY: the accumulator row
      };
      if (head_partial) add(0, 0, std::min(S, R - off));
      if (tail_partial && (n_touch > 1 || !head_partial)) add(n_touch - 1, (n_touch - 1) * R - off, S);
      if (bf.n_partial) {
        KIN_CUDA(bf.pmean.ensure(gn * 2), "cudaMalloc partial mean");
        KIN_CUDA(bf.pm2.ensure(gn * 2), "cudaMalloc partial m2");
        for (int k = 0; k < bf.n_partial; ++k) {
          KIN_CUDA(cudaMemcpyAsync(bf.pmean.p + k * gn, bf.mean.p + bf.partial_base[k] * gn, gn * sizeof(double),
                                   cudaMemcpyDeviceToDevice, bf.st), "D2D partial");
          KIN_CUDA(cudaMemcpyAsync(bf.pm2.p + k * gn, bf.m2.p + bf.partial_base[k] * gn, gn * sizeof(double),
                                   cudaMemcpyDeviceToDevice, bf.st), "D2D partial");
        }
      }
    }
  }
  bf.timed_stats = false;
  if (!stats_only && want_stats) {
    if (bf.n_partial) {
      KIN_CUDA(bf.pmean.ensure(gn * 2), "cudaMalloc partial mean");
      KIN_CUDA(bf.pm2.ensure(gn * 2), "cudaMalloc partial m2");
    }
    if (nP) {
      KIN_CUDA(bf.mean.ensure(gn * nP), "cudaMalloc mean");
      KIN_CUDA(bf.m2.ensure(gn * nP), "cudaMalloc m2");
    }
  }
  bf.last_gn = static_cast<int>(gn);
  bf.R = R;
  bf.nP = nP;
  bf.have_stats = want_stats && nP;
  bf.stats_only = stats_only;
  bf.stats_row0 = stats_only ? t_whole0 : 0;
  if (!stats_only) {
    if (int rc = launch_stats(sl, bf, err)) return rc;
    if (bf.have_stats || bf.n_partial) {
      KIN_CUDA(cudaEventRecord(bf.tev[2], bf.st), "event");
      bf.timed_stats = true;
    }
  }
  bf.pending_check = bf.last_int_state;
  bf.last_S = S;
  bf.s0 = part.inter ? 0 : part.s0;
  bf.s1 = bf.s0 + S;
  bf.P0 = part.inter ? 0 : (part.s0 + R - 1) / R;
  bf.part = part;
  bf.G = G;
  bf.N = N;
  bf.have_work = want_work;
  bf.valid = true;
  return KIN_OK;
}

// Complete a launch: wait for it and, if an int32 amount overflowed, re-run the
// stochastic kernel with double amounts (and the statistics) — same results.
int finish_launch(Slot& sl, Buffers& bf, kin_error* err) {
  KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
  KIN_CUDA(cudaStreamSynchronize(bf.st), "stream sync");
  if (!bf.pending_check) return KIN_OK;
  bf.pending_check = false;
  int flag = 0;
  KIN_CUDA(cudaMemcpy(&flag, bf.ovf.p, sizeof(int), cudaMemcpyDeviceToHost), "D2H overflow flag");
  if (!flag) return KIN_OK;
  KIN_CUDA(cudaMemsetAsync(bf.ovf.p, 0, sizeof(int), bf.st), "memset");
  cudaError_t e = kin::launch_stochastic(*bf.last_T, bf.last_SD, bf.last_O, bf.last_count, bf.counter.p, bf.ovf.p,
                                         false, bf.st);
  if (e != cudaSuccess) return cuda_fail(err, e, "simulation kernel relaunch");
  if (int rc = launch_stats(sl, bf, err)) return rc;
  KIN_CUDA(cudaStreamSynchronize(bf.st), "stream sync");
  return KIN_OK;
}

// Copy a launch's results into caller buffers (offsets relative to base_sim /
// base_point of the caller's arrays).  async: on the slot's copy stream, left
// in flight (the caller orders it after the launch); otherwise synchronous on
// the compute stream.
int copy_out(Slot& sl, Buffers& bf, const kin_sweep_out* out, uint64_t base_point, bool sync, kin_error* err) {
  NvtxRange nv("kin: copy-out (D2H into the caller layout)");
  cudaStream_t st = sync ? bf.st : (bf.cs ? bf.cs : sl.copy_stream);
  const uint64_t S = bf.s1 - bf.s0;
  const size_t gn = static_cast<size_t>(bf.G) * bf.N;
  const PlanPart& pt = bf.part;
  // per-simulation arrays: one row (contiguous part) or one row of R runs per
  // point, rows out_pitch simulations apart in the caller's layout (interleaved)
  const uint64_t rows = pt.inter ? pt.n_pts : 1;
  const uint64_t row = pt.inter ? bf.R : S;
  const uint64_t pitch = pt.inter ? pt.out_pitch : S;
  const uint64_t so = pt.out_first;
  auto put = [&](void* dst_base, size_t elem, const void* src) -> int {
    return copy_d2h_rows(sl, st, static_cast<char*>(dst_base) + so * elem, pitch * elem, src, row * elem, rows, sync,
                         err);
  };
  // traj: device layout == host layout [S][G][N] (STATS_ONLY never materialises it)
  if (out->traj && S && gn && !bf.stats_only)
    if (int rc = put(out->traj, gn * sizeof(double), bf.traj.p)) return rc;
  if (out->meta && S)
    if (int rc = put(out->meta, 6 * sizeof(uint64_t), bf.meta.p)) return rc;
  if (out->status && S)
    if (int rc = put(out->status, sizeof(int32_t), bf.status.p)) return rc;
  if (out->work && S && bf.have_work)
    if (int rc = put(out->work, sizeof(uint64_t), bf.work.p)) return rc;
  if (bf.have_stats) {
    const uint64_t prow = pt.inter ? 1 : bf.nP, prows = pt.inter ? pt.n_pts : 1;
    const uint64_t ppitch = pt.inter ? pt.out_pitch / bf.R : bf.nP;
    const uint64_t po = pt.inter ? pt.out_first / bf.R : bf.P0 - base_point;
    const size_t eb = gn * sizeof(double);
    const double* src_mean = bf.mean.p + bf.stats_row0 * gn;
    const double* src_m2 = bf.m2.p + bf.stats_row0 * gn;
    if (out->mean)
      if (int rc = copy_d2h_rows(sl, st, out->mean + po * gn, ppitch * eb, src_mean, prow * eb, prows, sync, err)) return rc;
    if (out->m2)
      if (int rc = copy_d2h_rows(sl, st, out->m2 + po * gn, ppitch * eb, src_m2, prow * eb, prows, sync, err)) return rc;
  }
  if (bf.n_partial) {
    const size_t need = static_cast<size_t>(bf.n_partial) * gn;
    if (bf.h_pcap < need) {
      if (bf.h_pmean) cudaFreeHost(bf.h_pmean);
      if (bf.h_pm2) cudaFreeHost(bf.h_pm2);
      bf.h_pmean = bf.h_pm2 = nullptr;
      KIN_CUDA(cudaMallocHost(&bf.h_pmean, need * sizeof(double)), "pinned partial mean");
      KIN_CUDA(cudaMallocHost(&bf.h_pm2, need * sizeof(double)), "pinned partial m2");
      bf.h_pcap = need;
    }
    KIN_CUDA(cudaMemcpyAsync(bf.h_pmean, bf.pmean.p, need * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H partial");
    KIN_CUDA(cudaMemcpyAsync(bf.h_pm2, bf.pm2.p, need * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H partial");
  }
  if (bf.pending_check && bf.ovf_host)
    KIN_CUDA(cudaMemcpyAsync(bf.ovf_host, bf.ovf.p, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H flag");
  if (sync) KIN_CUDA(cudaStreamSynchronize(st), "stream sync");
  return KIN_OK;
}

int fetch_range(Slot& sl, Buffers& bf, kin_sweep_out* out, uint64_t base_point, kin_error* err) {
  if (int rc = finish_launch(sl, bf, err)) return rc;
  return copy_out(sl, bf, out, base_point, true, err);
}

// Chunk plan of kin_sweep_run (see kin_abi.h kin_sweep_plan).
// merge_statistics (ensemble.hpp:56-57): Chan's parallel
// update of (n, mean, m2) — the oracle's kin_oracle_stats_merge formula.
void stats_merge(uint64_t* na, double* mean_a, double* m2_a, uint64_t nb, const double* mean_b, const double* m2_b,
                 uint64_t len) {
  if (nb == 0) return;
  if (*na == 0) {
    *na = nb;
    for (uint64_t q = 0; q < len; ++q) {
      mean_a[q] = mean_b[q];
      m2_a[q] = m2_b[q];
    }
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

int prepare(const kin_model* model, const kin_sweep_desc* desc, Layout* L, uint64_t* s0, uint64_t* s1,
            kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!model || !desc) { set_err(err, KIN_ERR_USAGE, "null argument"); return KIN_ERR_USAGE; }
  std::string msg;
  if (int rc = sweep_layout(desc, L, &msg)) { set_err(err, rc, msg); return rc; }
  if (int rc = validate_sweep(model->host, desc, *L, &msg)) { set_err(err, rc, msg); return rc; }
  *s0 = desc->sim_begin;
  *s1 = desc->sim_end == 0 ? L->S : std::min<uint64_t>(desc->sim_end, L->S);
  if (*s0 > *s1) { set_err(err, KIN_ERR_USAGE, "inverted simulation range"); return KIN_ERR_USAGE; }
  if (desc->shard_count > 1 && (*s0 % L->R != 0 || *s1 % L->R != 0)) {
    set_err(err, KIN_ERR_INPUT, "a sharded call needs a range of whole points");
    return KIN_ERR_INPUT;
  }
  return KIN_OK;
}

// Caller-local sizes of a call: simulations and statistics points.
void local_sizes(const kin_sweep_desc* d, const Layout& L, uint64_t s0, uint64_t s1, uint64_t* n_sims,
                 uint64_t* n_points) {
  if (d->shard_count > 1) {
    const uint64_t P = (s1 - s0) / L.R, n = static_cast<uint64_t>(d->shard_count);
    const uint64_t K = P > static_cast<uint64_t>(d->shard_index) ? (P - d->shard_index + n - 1) / n : 0;
    *n_sims = K * L.R;
    *n_points = K;
  } else {
    *n_sims = s1 - s0;
    const uint64_t p0 = (s0 + L.R - 1) / L.R, p1 = s1 / L.R;
    *n_points = p1 > p0 ? p1 - p0 : 0;
  }
}

// Points cut by part edges: Chan-merge their per-part statistics in ascending
// part order (ensemble.hpp:91-99: per-worker accumulators merged in ascending
// worker-range order) into the caller's mean/m2.
void merge_partials(const std::vector<Buffers*>& bufs, const kin_sweep_out& out, uint64_t base_point,
                    uint64_t point_end) {
  if (!out.mean && !out.m2) return;
  std::map<uint64_t, std::pair<uint64_t, std::vector<double>>> acc;  // point -> (n, [mean | m2])
  size_t gn = 0;
  for (const Buffers* bp : bufs) {
    const Buffers& bf = *bp;
    gn = static_cast<size_t>(bf.last_gn);
    for (int k = 0; k < bf.n_partial; ++k) {
      auto& a = acc[bf.partial_point[k]];
      if (a.second.empty()) a.second.assign(2 * gn, 0.0);
      stats_merge(&a.first, a.second.data(), a.second.data() + gn, bf.partial_n[k], bf.h_pmean + k * gn,
                  bf.h_pm2 + k * gn, gn);
    }
  }
  for (const auto& kv : acc) {
    const uint64_t pt = kv.first;
    if (pt < base_point || pt >= point_end) continue;  // not whole inside the call's range: no statistics
    if (out.mean) std::memcpy(out.mean + (pt - base_point) * gn, kv.second.second.data(), gn * sizeof(double));
    if (out.m2) std::memcpy(out.m2 + (pt - base_point) * gn, kv.second.second.data() + gn, gn * sizeof(double));
  }
}

}  // namespace

extern "C" {

int32_t kin_abi_version(void) { return KIN_ABI_VERSION; }

const char* kin_status_string(int32_t code) {
  switch (code) {
    case KIN_OK: return "ok";
    case KIN_ERR_INPUT: return "input/validation error";
    case KIN_ERR_SIMULATION: return "simulation failure";
    case KIN_ERR_DEVICE: return "device (CUDA) error";
    case KIN_ERR_USAGE: return "usage error";
    default: return "unknown status";
  }
}

uint64_t kin_splitmix64_mix(uint64_t v) { return kin::splitmix64_mix(v); }
uint64_t kin_derive_run_seed(uint64_t m, uint64_t i) { return kin::derive_run_seed(m, i); }

void kin_stats_merge(uint64_t* n_a, double* mean_a, double* m2_a, uint64_t n_b, const double* mean_b,
                     const double* m2_b, uint64_t len) {
  stats_merge(n_a, mean_a, m2_a, n_b, mean_b, m2_b, len);
}

int32_t kin_visible_devices(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return count;
}

int kin_ctx_create(const int32_t* ids, int32_t n, kin_ctx** out, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!out) { set_err(err, KIN_ERR_USAGE, "null output"); return KIN_ERR_USAGE; }
  *out = nullptr;
  int count = 0;
  KIN_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (count == 0) { set_err(err, KIN_ERR_DEVICE, "no CUDA device"); return KIN_ERR_DEVICE; }
  std::vector<int> devs;
  if (!ids || n <= 0) devs.push_back(0);
  else devs.assign(ids, ids + n);
  auto ctx = std::make_unique<kin_ctx>();
  for (int dv : devs) {
    if (dv < 0 || dv >= count) { set_err(err, KIN_ERR_USAGE, "device id out of range"); return KIN_ERR_USAGE; }
    auto sl = std::make_unique<Slot>();
    sl->device = dv;
    KIN_CUDA(cudaSetDevice(dv), "cudaSetDevice");
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dv);
    if (major < 10) { set_err(err, KIN_ERR_DEVICE, "engine is built for sm_100a (B200) only"); return KIN_ERR_DEVICE; }
    KIN_CUDA(cudaStreamCreateWithFlags(&sl->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    KIN_CUDA(cudaStreamCreateWithFlags(&sl->aux_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    KIN_CUDA(cudaStreamCreateWithFlags(&sl->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    KIN_CUDA(cudaStreamCreateWithFlags(&sl->aux_copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    // lgamma(k+1) from the host libm (the oracle's, glibc) for the PTRS test
    std::vector<double> lg(KIN_LGAMMA_N);
    // (lgamma_r: glibc's lgamma writes the global signgam — a data race when
    // contexts are created from several threads)
    for (int k = 0; k < KIN_LGAMMA_N; ++k) {
      int sign = 0;
      lg[k] = lgamma_r(static_cast<double>(k) + 1.0, &sign);
    }
    KIN_CUDA(sl->lgamma_tab.ensure(KIN_LGAMMA_N), "cudaMalloc lgamma table");
    KIN_CUDA(cudaMemcpy(sl->lgamma_tab.p, lg.data(), sizeof(double) * KIN_LGAMMA_N, cudaMemcpyHostToDevice), "H2D lgamma");
    std::vector<double> co;
    lsoda_coeffs(&co);
    KIN_CUDA(sl->lsoda_co.ensure(co.size()), "cudaMalloc lsoda coefficients");
    KIN_CUDA(cudaMemcpy(sl->lsoda_co.p, co.data(), sizeof(double) * co.size(), cudaMemcpyHostToDevice), "H2D lsoda");
    ctx->slots.push_back(std::move(sl));
  }
  *out = ctx.release();
  return KIN_OK;
}

void kin_ctx_destroy(kin_ctx* ctx) {
  if (!ctx) return;
  for (auto& kv : ctx->jobs) {
    kin_error e;
    (void)e;
    if (kv.second->status_pinned) cudaFreeHost(kv.second->status_pinned);
  }
  for (auto& sl : ctx->slots) {
    cudaSetDevice(sl->device);
    cudaStreamSynchronize(sl->stream);
    cudaStreamSynchronize(sl->aux_stream);
    cudaStreamSynchronize(sl->copy_stream);
    cudaStreamSynchronize(sl->aux_copy_stream);
    sl->main.release();
    for (auto& b : sl->pool) b->release();
    sl->lgamma_tab.release();
    sl->lsoda_co.release();
    if (sl->stage) cudaFreeHost(sl->stage);
    for (auto& e : sl->ev) if (e) cudaEventDestroy(e);
    cudaStreamDestroy(sl->stream);
    cudaStreamDestroy(sl->aux_stream);
    cudaStreamDestroy(sl->copy_stream);
    cudaStreamDestroy(sl->aux_copy_stream);
  }
  delete ctx;
}

int32_t kin_ctx_device_count(const kin_ctx* ctx) { return ctx ? static_cast<int32_t>(ctx->slots.size()) : 0; }

void* kin_ctx_stream(kin_ctx* ctx, int32_t slot) {
  if (!ctx || slot < 0 || slot >= static_cast<int32_t>(ctx->slots.size())) return nullptr;
  return ctx->slots[slot]->stream;
}

int kin_model_upload(kin_ctx* ctx, const kin_model_desc* desc, kin_model** out, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || !out) { set_err(err, KIN_ERR_USAGE, "null argument"); return KIN_ERR_USAGE; }
  auto m = std::make_unique<kin_model>();
  m->ctx = ctx;
  std::string msg;
  if (int rc = load_model(desc, &m->host, &msg)) { set_err(err, rc, msg); return rc; }
  *out = m.release();
  return KIN_OK;
}

void kin_model_free(kin_model* model) { delete model; }

int kin_sweep_size(const kin_sweep_desc* desc, uint64_t* np, uint64_t* ns, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  Layout L;
  std::string msg;
  if (int rc = sweep_layout(desc, &L, &msg)) { set_err(err, rc, msg); return rc; }
  if (np) *np = L.P;
  if (ns) *ns = L.S;
  return KIN_OK;
}

int kin_sweep_run(kin_ctx* ctx, const kin_model* model, const kin_sweep_desc* desc, kin_sweep_out* out,
                  kin_error* err) {
  uint64_t ticket = 0;
  if (int rc = kin_sweep_submit(ctx, model, desc, out, &ticket, err)) return rc;
  return kin_sweep_wait(ctx, ticket, err);
}

int kin_sweep_submit(kin_ctx* ctx, const kin_model* model, const kin_sweep_desc* desc, kin_sweep_out* out,
                     uint64_t* ticket, kin_error* err) {
  if (!ctx || !ticket) { set_err(err, KIN_ERR_USAGE, "null argument"); return KIN_ERR_USAGE; }
  NvtxRange nv("kin_sweep_submit");
  auto job = std::make_unique<Job>();
  uint64_t s0, s1;
  if (int rc = prepare(model, desc, &job->L, &s0, &s1, err)) return rc;
  const Layout& L = job->L;
  if (out) job->out = *out;
  if (desc->output_mode == KIN_OUTPUT_STATS_ONLY) job->out.traj = nullptr;
  job->s0 = s0;
  job->s1 = s1;
  job->sh_n = desc->shard_count > 1 ? desc->shard_count : 1;
  job->sh_i = job->sh_n > 1 ? desc->shard_index : 0;
  job->base_point = (s0 + L.R - 1) / L.R;
  local_sizes(desc, L, s0, s1, &job->n_local, &job->np_local);
  const uint64_t S = job->n_local;
  if (!job->out.status && S) {
    KIN_CUDA(cudaMallocHost(&job->status_pinned, sizeof(int32_t) * S), "pinned status");
    job->out.status = job->status_pinned;
  }
  const int D = static_cast<int>(ctx->slots.size());
  std::vector<PlanPart> plan;
  {
    std::string msg;
    if (int rc = plan_parts(s0, s1, L.R, D, job->sh_i, job->sh_n, &plan, &msg)) {
      set_err(err, rc, msg);
      if (job->status_pinned) cudaFreeHost(job->status_pinned);
      return rc;
    }
  }
  const bool stats = job->out.mean || job->out.m2;
  const bool partials = stats && plan.size() > 1 && !plan[0].inter;
  auto enqueue = [&]() -> int {
    for (const PlanPart& part : plan) {
      Slot& sl = *ctx->slots[part.dev];
      std::lock_guard<std::mutex> lk(sl.mu);
      KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
      Buffers* bf;
      if (!sl.pool.empty()) {
        bf = sl.pool.back().release();
        sl.pool.pop_back();
      } else {
        bf = new Buffers;
      }
      job->parts.push_back({part.dev, bf});
      const bool aux = sl.job_rr++ & 1u;
      bf->st = aux ? sl.aux_stream : sl.stream;
      bf->cs = aux ? sl.aux_copy_stream : sl.copy_stream;
      if (int rc = launch_range(sl, *bf, model, desc, L, part, stats, job->out.work != nullptr, err, partials))
        return rc;
      if (!bf->ev_done) KIN_CUDA(cudaEventCreateWithFlags(&bf->ev_done, cudaEventDisableTiming), "event");
      if (!bf->ev_copied) KIN_CUDA(cudaEventCreateWithFlags(&bf->ev_copied, cudaEventDisableTiming), "event");
      if (!bf->ovf_host) KIN_CUDA(cudaMallocHost(&bf->ovf_host, sizeof(int)), "pinned flag");
      KIN_CUDA(cudaEventRecord(bf->ev_done, bf->st), "event");
      // copy-out on the copy stream, overlapping the next launches on `stream`
      KIN_CUDA(cudaStreamWaitEvent(bf->cs, bf->ev_done, 0), "stream wait");
      if (int rc = copy_out(sl, *bf, &job->out, job->base_point, false, err)) return rc;
      KIN_CUDA(cudaEventRecord(bf->ev_copied, bf->cs), "event");
    }
    return KIN_OK;
  };
  if (int rc = enqueue()) {
    // a part failed to enqueue: drain the parts already in flight and give
    // their buffers back, so nothing writes into `out` after we return
    for (auto& part : job->parts) {
      Slot& sl = *ctx->slots[part.slot];
      cudaSetDevice(sl.device);
      if (part.buf->st) cudaStreamSynchronize(part.buf->st);
      cudaStreamSynchronize(sl.copy_stream);
      cudaStreamSynchronize(sl.aux_copy_stream);
      std::lock_guard<std::mutex> lk(sl.mu);
      part.buf->pending_check = false;
      sl.pool.emplace_back(part.buf);
    }
    job->parts.clear();
    if (job->status_pinned) cudaFreeHost(job->status_pinned);
    return rc;
  }
  std::lock_guard<std::mutex> lk(ctx->jobs_mu);
  *ticket = ctx->next_ticket++;
  ctx->jobs[*ticket] = std::move(job);
  return KIN_OK;
}

int kin_ensemble_run(kin_ctx* ctx, const kin_model* model, const kin_method* method, uint64_t n_runs,
                     uint64_t master_seed, double t_end, const double* grid, int32_t n_grid, int32_t rng_mode,
                     kin_sweep_out* out, kin_error* err) {
  if (!method) { set_err(err, KIN_ERR_USAGE, "null method"); return KIN_ERR_USAGE; }
  kin_sweep_desc d;
  std::memset(&d, 0, sizeof d);
  d.method = *method;
  d.runs_per_point = n_runs;
  d.master_seed = master_seed;
  d.seed_mode = KIN_SEED_ENSEMBLE;
  d.rng_mode = rng_mode;
  d.t_end = t_end;
  d.n_grid = n_grid;
  d.grid = grid;
  // no trajectories requested (no RunSink): statistics only, runs streamed
  // through a bounded device window
  if (out && !out->traj) d.output_mode = KIN_OUTPUT_STATS_ONLY;
  return kin_sweep_run(ctx, model, &d, out, err);
}

int kin_run_single(kin_ctx* ctx, const kin_model* model, const kin_method* method, double t_end,
                   const double* grid, int32_t n_grid, uint64_t seed, int32_t rng_mode, double* samples,
                   uint64_t* meta, kin_error* err) {
  if (!method) { set_err(err, KIN_ERR_USAGE, "null method"); return KIN_ERR_USAGE; }
  kin_sweep_desc d;
  std::memset(&d, 0, sizeof d);
  d.method = *method;
  d.runs_per_point = 1;
  d.master_seed = seed;
  d.seed_mode = KIN_SEED_DIRECT;
  d.rng_mode = rng_mode;
  d.t_end = t_end;
  d.n_grid = n_grid;
  d.grid = grid;
  kin_sweep_out o;
  std::memset(&o, 0, sizeof o);
  o.traj = samples;
  o.meta = meta;
  return kin_sweep_run(ctx, model, &d, &o, err);
}

int kin_sweep_wait(kin_ctx* ctx, uint64_t ticket, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  NvtxRange nv("kin_sweep_wait");
  std::unique_ptr<Job> job;
  if (!ctx) { set_err(err, KIN_ERR_USAGE, "null context"); return KIN_ERR_USAGE; }
  {
    std::lock_guard<std::mutex> lk(ctx->jobs_mu);
    if (!ctx->jobs.count(ticket)) { set_err(err, KIN_ERR_USAGE, "unknown ticket"); return KIN_ERR_USAGE; }
    job = std::move(ctx->jobs[ticket]);
    ctx->jobs.erase(ticket);
  }
  int rc = KIN_OK;
  for (auto& part : job->parts) {
    Slot& sl = *ctx->slots[part.slot];
    Buffers& bf = *part.buf;
    // every part's copy-out is waited for, even after an error: its buffers go
    // back to the pool and its D2H must not write into `out` after we return
    cudaError_t ce = cudaSetDevice(sl.device);
    if (ce == cudaSuccess) ce = cudaEventSynchronize(bf.ev_copied);
    if (ce != cudaSuccess) {
      if (rc == KIN_OK) rc = cuda_fail(err, ce, "copy-out");
      cudaStreamSynchronize(bf.st);
      cudaStreamSynchronize(sl.copy_stream);
      cudaStreamSynchronize(sl.aux_copy_stream);
      bf.pending_check = false;
      continue;
    }
    if (rc == KIN_OK && bf.pending_check && *bf.ovf_host) {
      // an int32 amount overflowed: redo this part with double amounts
      std::lock_guard<std::mutex> lk(sl.mu);
      bf.pending_check = true;
      if ((rc = finish_launch(sl, bf, err)) == KIN_OK) rc = copy_out(sl, bf, &job->out, job->base_point, true, err);
    }
    bf.pending_check = false;
  }
  if (rc == KIN_OK) {
    std::vector<Buffers*> bufs;
    for (auto& part : job->parts) bufs.push_back(part.buf);
    merge_partials(bufs, job->out, job->base_point, job->s1 / job->L.R);
  }
  for (auto& part : job->parts) {
    Slot& sl = *ctx->slots[part.slot];
    std::lock_guard<std::mutex> lk(sl.mu);
    sl.pool.emplace_back(part.buf);
  }
  job->parts.clear();
  if (rc == KIN_OK) {
    const uint64_t S = job->n_local;
    for (uint64_t s = 0; s < S; ++s) {  // caller-local order is ascending in the global index
      const int32_t st = job->out.status[s];
      if (st != KIN_SIM_OK) {
        const uint64_t g = job->global_of(s);
        if (err) {
          err->code = KIN_ERR_SIMULATION;
          err->sim_status = st;
          err->sim_index = g;
          err->point_index = g / job->L.R;
          err->run_index = g % job->L.R;
          std::snprintf(err->message, sizeof(err->message), "simulation %llu (point %llu, run %llu) failed: status %d",
                        (unsigned long long)g, (unsigned long long)(g / job->L.R),
                        (unsigned long long)(g % job->L.R), st);
        }
        rc = KIN_ERR_SIMULATION;
        break;
      }
    }
  }
  if (job->status_pinned) cudaFreeHost(job->status_pinned);
  return rc;
}

int kin_sweep_plan(uint64_t s0, uint64_t s1, uint64_t R, int32_t D, int32_t sh_i, int32_t sh_n, int32_t max_parts,
                   kin_sweep_part* parts, int32_t* n_parts, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!n_parts || (max_parts > 0 && !parts)) { set_err(err, KIN_ERR_USAGE, "bad argument"); return KIN_ERR_USAGE; }
  std::vector<PlanPart> plan;
  std::string msg;
  if (int rc = plan_parts(s0, s1, R, D, sh_i, sh_n, &plan, &msg)) { set_err(err, rc, msg); return rc; }
  if (static_cast<int64_t>(plan.size()) > max_parts) { set_err(err, KIN_ERR_USAGE, "max_parts too small"); return KIN_ERR_USAGE; }
  for (size_t i = 0; i < plan.size(); ++i) {
    const PlanPart& p = plan[i];
    kin_sweep_part& q = parts[i];
    std::memset(&q, 0, sizeof q);
    q.device = p.dev;
    q.interleaved = p.inter ? 1 : 0;
    q.sim_begin = p.s0;
    q.sim_end = p.s1;
    q.pt_first = p.pt_first;
    q.pt_stride = p.pt_stride;
    q.n_points = p.n_pts;
    q.out_first = p.out_first;
    q.out_pitch = p.out_pitch;
  }
  *n_parts = static_cast<int32_t>(plan.size());
  return KIN_OK;
}

int kin_sweep_local_size(const kin_sweep_desc* desc, uint64_t* np, uint64_t* ns, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  Layout L;
  std::string msg;
  if (int rc = sweep_layout(desc, &L, &msg)) { set_err(err, rc, msg); return rc; }
  const uint64_t s0 = desc->sim_begin;
  const uint64_t s1 = desc->sim_end == 0 ? L.S : std::min<uint64_t>(desc->sim_end, L.S);
  if (s0 > s1) { set_err(err, KIN_ERR_USAGE, "inverted simulation range"); return KIN_ERR_USAGE; }
  uint64_t a = 0, b = 0;
  local_sizes(desc, L, s0, s1, &a, &b);
  if (ns) *ns = a;
  if (np) *np = b;
  return KIN_OK;
}

int kin_sweep_launch(kin_ctx* ctx, const kin_model* model, const kin_sweep_desc* desc, int32_t slot,
                     int32_t want_stats, int32_t want_work, kin_error* err) {
  if (!ctx || slot < -1 || slot >= static_cast<int32_t>(ctx->slots.size())) {
    set_err(err, KIN_ERR_USAGE, "bad context/slot");
    return KIN_ERR_USAGE;
  }
  Layout L;
  uint64_t s0, s1;
  if (int rc = prepare(model, desc, &L, &s0, &s1, err)) return rc;
  const int sh_n = desc->shard_count > 1 ? desc->shard_count : 1, sh_i = sh_n > 1 ? desc->shard_index : 0;
  std::vector<PlanPart> plan;
  std::string msg;
  const int D = slot < 0 ? static_cast<int>(ctx->slots.size()) : 1;
  if (int rc = plan_parts(s0, s1, L.R, D, sh_i, sh_n, &plan, &msg)) { set_err(err, rc, msg); return rc; }
  for (int dv = 0; dv < static_cast<int>(ctx->slots.size()); ++dv) ctx->slots[dv]->main.valid = slot >= 0 && dv != slot && ctx->slots[dv]->main.valid;
  const bool partials = want_stats && plan.size() > 1 && !plan[0].inter;
  for (const PlanPart& p : plan) {
    Slot& sl = *ctx->slots[slot < 0 ? p.dev : slot];
    std::lock_guard<std::mutex> lk(sl.mu);
    if (int rc = launch_range(sl, sl.main, model, desc, L, p, want_stats != 0, want_work != 0, err, partials)) return rc;
    sl.main.base_point = (s0 + L.R - 1) / L.R;
    sl.main.point_end = s1 / L.R;
  }
  return KIN_OK;
}

int kin_sweep_sync(kin_ctx* ctx, int32_t slot, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || slot < -1 || slot >= static_cast<int32_t>(ctx->slots.size())) {
    set_err(err, KIN_ERR_USAGE, "bad context/slot");
    return KIN_ERR_USAGE;
  }
  for (int dv = 0; dv < static_cast<int>(ctx->slots.size()); ++dv) {
    if (slot >= 0 && dv != slot) continue;
    Slot& sl = *ctx->slots[dv];
    std::lock_guard<std::mutex> lk(sl.mu);
    if (!sl.main.valid) continue;
    if (int rc = finish_launch(sl, sl.main, err)) return rc;
  }
  return KIN_OK;
}

int kin_sweep_fetch(kin_ctx* ctx, int32_t slot, kin_sweep_out* out, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || !out || slot < -1 || slot >= static_cast<int32_t>(ctx->slots.size())) {
    set_err(err, KIN_ERR_USAGE, "bad argument");
    return KIN_ERR_USAGE;
  }
  std::vector<Buffers*> bufs;
  uint64_t base_point = 0, point_end = 0;
  for (int dv = 0; dv < static_cast<int>(ctx->slots.size()); ++dv) {
    if (slot >= 0 && dv != slot) continue;
    Slot& sl = *ctx->slots[dv];
    std::lock_guard<std::mutex> lk(sl.mu);
    if (!sl.main.valid) continue;
    if (int rc = fetch_range(sl, sl.main, out, sl.main.base_point, err)) return rc;
    bufs.push_back(&sl.main);
    base_point = sl.main.base_point;
    point_end = sl.main.point_end;
  }
  if (bufs.empty()) { set_err(err, KIN_ERR_USAGE, "nothing launched on this slot"); return KIN_ERR_USAGE; }
  merge_partials(bufs, *out, base_point, point_end);
  return KIN_OK;
}

int kin_jit_check(const kin_model_desc* desc, const kin_sweep_desc* sweep, char* log, int32_t log_cap,
                  kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  HostModel H;
  std::string msg;
  if (int rc = load_model(desc, &H, &msg)) { set_err(err, rc, msg); return rc; }
  if (!sweep) { set_err(err, KIN_ERR_USAGE, "null sweep"); return KIN_ERR_USAGE; }
  const kin::JitModel jm = jit_model(H, sweep);
  std::string lg;
  // the method's JIT kernel: the hybrid PDMP kernel for KIN_METHOD_HYBRID,
  // else the stochastic (SSA / tau-leaping) kernel
  const bool philox = sweep->rng_mode == KIN_RNG_PHILOX;
  const bool ok = sweep->method.kind == KIN_METHOD_HYBRID ? kin::jit_compile_check_hybrid(jm, false, philox, &lg)
                  : sweep->method.kind == KIN_METHOD_LSODA ? kin::jit_compile_check_lsoda(jm, false, &lg)
                                                           : kin::jit_compile_check(jm, false, philox, true, &lg);
  if (log && log_cap > 0) std::snprintf(log, static_cast<size_t>(log_cap), "%s", lg.c_str());
  if (!ok) { set_err(err, KIN_ERR_INPUT, "NVRTC compilation of the model kernel failed"); return KIN_ERR_INPUT; }
  return KIN_OK;
}

int kin_sweep_kernel_ms(kin_ctx* ctx, int32_t slot, double* sim_ms, double* stats_ms, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || slot < 0 || slot >= static_cast<int32_t>(ctx->slots.size())) {
    set_err(err, KIN_ERR_USAGE, "bad context/slot");
    return KIN_ERR_USAGE;
  }
  Slot& sl = *ctx->slots[slot];
  const Buffers& bm = sl.main;
  if (!bm.valid || !bm.tev[0]) { set_err(err, KIN_ERR_USAGE, "nothing launched on this slot"); return KIN_ERR_USAGE; }
  KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
  float a = 0.0f, b = 0.0f;
  KIN_CUDA(cudaEventElapsedTime(&a, bm.tev[0], bm.tev[1]), "event time");
  if (bm.timed_stats) KIN_CUDA(cudaEventElapsedTime(&b, bm.tev[1], bm.tev[2]), "event time");
  if (sim_ms) *sim_ms = a;
  if (stats_ms) *stats_ms = bm.timed_stats ? b : 0.0;
  return KIN_OK;
}

const char* kin_sweep_kernel_name(kin_ctx* ctx, int32_t slot) {
  if (!ctx || slot < 0 || slot >= static_cast<int32_t>(ctx->slots.size())) return "";
  return ctx->slots[slot]->main.kernel_name;
}

int kin_device_rng_draws(kin_ctx* ctx, uint64_t seed, int32_t kind, double mean, int32_t n, uint64_t* out_bits,
                         kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || ctx->slots.empty() || n < 0 || (n > 0 && !out_bits)) {
    set_err(err, KIN_ERR_USAGE, "bad argument");
    return KIN_ERR_USAGE;
  }
  Slot& sl = *ctx->slots[0];
  KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
  uint64_t* d = nullptr;
  KIN_CUDA(cudaMalloc(&d, sizeof(uint64_t) * std::max(n, 1)), "cudaMalloc");
  cudaError_t e = kin::launch_rng_draws(seed, kind, mean, n, d, sl.lgamma_tab.p, sl.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_bits, d, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, sl.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sl.stream);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(err, e, "rng draws");
  return KIN_OK;
}

int kin_device_binomial_draws(kin_ctx* ctx, uint64_t seed, uint64_t n_trials, double p, int32_t n, uint64_t* out,
                              kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || ctx->slots.empty() || n < 0 || (n > 0 && !out)) {
    set_err(err, KIN_ERR_USAGE, "bad argument");
    return KIN_ERR_USAGE;
  }
  Slot& sl = *ctx->slots[0];
  KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
  uint64_t* d = nullptr;
  KIN_CUDA(cudaMalloc(&d, sizeof(uint64_t) * std::max(n, 1)), "cudaMalloc");
  cudaError_t e = kin::launch_binomial_draws(seed, n_trials, p, n, d, sl.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, sl.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sl.stream);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(err, e, "binomial draws");
  return KIN_OK;
}

int kin_device_unit(kin_ctx* ctx, const kin_model* model, int32_t kind, const double* x, const double* params,
                    int32_t n_params, double* out, int32_t out_cap, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || ctx->slots.empty() || !model || !x || !out || kind < 0 || kind > 6) {
    set_err(err, KIN_ERR_USAGE, "bad argument");
    return KIN_ERR_USAGE;
  }
  const HostModel& H = model->host;
  const int need_params[7] = {0, 1, 2, H.m, 1 + H.m, 0, 3};
  const int need_out[7] = {H.m, 1, 2, H.n + 1, H.n + 1, H.n, 2 * H.n + 1};
  if (n_params < need_params[kind] || (need_params[kind] && !params) || out_cap < need_out[kind]) {
    set_err(err, KIN_ERR_USAGE, "params/out too small for this unit");
    return KIN_ERR_USAGE;
  }
  // tables for a sweep with no axes (the unit reads rates, reactant terms and nu)
  const double g0 = 0.0;
  kin_sweep_desc d;
  std::memset(&d, 0, sizeof d);
  d.runs_per_point = 1;
  d.n_grid = 1;
  d.grid = &g0;
  auto T = std::make_unique<KinTables>();
  std::string msg;
  if (int rc = pack_tables(H, &d, T.get(), &msg)) { set_err(err, rc, msg); return rc; }
  Slot& sl = *ctx->slots[0];
  std::lock_guard<std::mutex> lk(sl.mu);
  KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
  const size_t nx = static_cast<size_t>(std::max(H.n, 1)), np = static_cast<size_t>(std::max(n_params, 1));
  const size_t no = static_cast<size_t>(need_out[kind]);
  double* dev = nullptr;
  KIN_CUDA(cudaMalloc(&dev, sizeof(double) * (nx + np + no)), "cudaMalloc");
  cudaError_t e = cudaMemcpyAsync(dev, x, sizeof(double) * H.n, cudaMemcpyHostToDevice, sl.stream);
  if (e == cudaSuccess && n_params > 0)
    e = cudaMemcpyAsync(dev + nx, params, sizeof(double) * n_params, cudaMemcpyHostToDevice, sl.stream);
  if (e == cudaSuccess) e = kin::launch_unit(*T, kind, dev, dev + nx, dev + nx + np, sl.stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, dev + nx + np, sizeof(double) * no, cudaMemcpyDeviceToHost, sl.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sl.stream);
  cudaFree(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "unit kernel");
  return KIN_OK;
}

int kin_measure_fp64_peak(kin_ctx* ctx, double* tflops, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!ctx || ctx->slots.empty() || !tflops) { set_err(err, KIN_ERR_USAGE, "bad argument"); return KIN_ERR_USAGE; }
  Slot& sl = *ctx->slots[0];
  KIN_CUDA(cudaSetDevice(sl.device), "cudaSetDevice");
  KIN_CUDA(kin::measure_fp64_peak(sl.stream, tflops), "fp64 peak");
  return KIN_OK;
}

}  // extern "C"

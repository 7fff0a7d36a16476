// kin_cli.cpp — `simulate` / `sweep` / `replay` over the C-ABI (include/kin_cli.h):
// the reference's CLI surface for the sweep path (cli.hpp, SPEC.md:477-494,
// :513-524).  Flow: parse flags -> parse the model (kin_model_text.h) and the
// sweep file -> kin_sweep_run on the GPU(s) -> CSV (kin_io.h) -> manifest.
// Nothing is written before the simulation has succeeded, so a failing run
// leaves no output file.  Host code only.
#include "../../include/kin_cli.h"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/kin_abi.h"
#include "../../include/kin_io.h"
#include "../../include/kin_model_text.h"

namespace {

constexpr const char* kToolVersion = "0.1.0";  // cli.hpp:5

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void usage(const std::string& m) { throw Fail{KIN_EXIT_USAGE, m}; }
[[noreturn]] void input(const std::string& m) { throw Fail{KIN_EXIT_INPUT, m}; }

const char* kUsage =
    "usage: kinetics-b200 simulate --model PATH --method {ssa|tau|cle|ode|lsoda|hybrid} --t-end T --samples N\n"
    "                              --seed S [--runs R] [--epsilon E] [--tau T] [--rtol R] [--atol A]\n"
    "                              [--tol R[,A]] [--max-steps N] [--rng compat|philox] [--max-order 2|3]\n"
    "                              [--theta-x X] [--theta-a A] [--repartition R] [--workers N] --out PATH\n"
    "       kinetics-b200 sweep --model PATH --sweep PATH --t-end T --samples N [--rng compat|philox]\n"
    "                           [--max-order 2|3] [--workers N] --out PATH\n"
    "       kinetics-b200 replay MANIFEST\n";

bool read_file(const std::string& path, std::string* out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  *out = ss.str();
  return true;
}

std::string hex64(uint64_t v) {
  char b[20];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
  return b;
}

std::string fmt(double v) {
  char b[32];
  kin_format_double(v, b, sizeof b);
  return b;
}

std::string trim(const std::string& s) {
  size_t b = s.find_first_not_of(" \t\r\n"), e = s.find_last_not_of(" \t\r\n");
  return b == std::string::npos ? "" : s.substr(b, e - b + 1);
}

double num(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const double d = std::strtod(v.c_str(), &end);
  if (v.empty() || *end) usage("bad value for " + flag + ": '" + v + "'");
  return d;
}

uint64_t unum(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  if (v.empty() || v[0] == '-') usage("bad value for " + flag + ": '" + v + "'");
  const unsigned long long u = std::strtoull(v.c_str(), &end, 0);
  if (*end) usage("bad value for " + flag + ": '" + v + "'");
  return u;
}

// ---- method ---------------------------------------------------------------
struct MethodSpec {
  std::string name = "";
  double epsilon = 0.03, tau = 0.0, rtol = 1e-6, atol = 1e-9;  // ensemble.hpp:59-71, deterministic.hpp:14-20
  double theta_x = 100.0, theta_a = 10.0, repartition = 0.0;    // HybridConfig, hybrid.hpp:21-26
  uint64_t max_steps = 10000000;
  kin_method to_c() const {
    kin_method m;
    std::memset(&m, 0, sizeof m);
    if (name == "ssa") m.kind = KIN_METHOD_SSA;
    else if (name == "tau") m.kind = tau > 0.0 ? KIN_METHOD_TAU_FIXED : KIN_METHOD_TAU_ADAPTIVE;
    else if (name == "ode") m.kind = KIN_METHOD_ODE;
    else if (name == "lsoda") m.kind = KIN_METHOD_LSODA;
    else if (name == "cle") m.kind = KIN_METHOD_CLE;
    else if (name == "hybrid") m.kind = KIN_METHOD_HYBRID;
    m.tau = tau;
    m.theta_x = theta_x;
    m.theta_a = theta_a;
    m.repartition_interval = repartition;
    m.epsilon = epsilon;
    m.integrator.rel_tol = rtol;
    m.integrator.abs_tol = atol;
    m.integrator.h_init = 0.0;
    m.integrator.h_max = HUGE_VAL;
    m.integrator.max_steps = max_steps;
    return m;
  }
  std::string label() const {
    if (name == "tau") return tau > 0.0 ? "tau-fixed" : "tau-adaptive";
    return name;
  }
};

void check_method(const MethodSpec& m) {
  if (m.name != "ssa" && m.name != "tau" && m.name != "ode" && m.name != "lsoda" && m.name != "cle" &&
      m.name != "hybrid")
    usage("unknown method '" + m.name + "'");
  if (m.name == "hybrid" && !(m.theta_x >= 0.0 && m.theta_a >= 0.0 && m.repartition >= 0.0))
    input("hybrid thresholds and repartition interval must be non-negative");
  if (m.name == "cle" && !(m.tau > 0.0)) input("method 'cle' needs a positive step (--tau, or tau= in a sweep file)");
}

// ---- sweep file ---------------------------------------------
struct Axis {
  std::string name;  // parameter name, or "init:<species>"
  std::vector<double> values;
};
struct SweepFile {
  std::vector<Axis> axes;
  uint64_t runs = 1;
  uint64_t seed = 0;
  MethodSpec method;
  bool have_method = false;
};

// "lo:hi:n [log]" -> n values, endpoints exact: lo + (hi-lo)*k/(n-1), or
// lo*(hi/lo)^(k/(n-1)) computed as exp(log lo + k*(log hi - log lo)/(n-1))
std::vector<double> parse_values(const std::string& text, long ln) {
  auto bad = [&](const std::string& m) -> Fail { return Fail{KIN_EXIT_INPUT, "sweep file line " + std::to_string(ln) + ": " + m}; };
  std::string t = trim(text);
  bool logsp = false;
  if (t.size() > 4 && t.compare(t.size() - 4, 4, " log") == 0) {
    logsp = true;
    t = trim(t.substr(0, t.size() - 4));
  }
  std::vector<double> v;
  auto to_d = [&](const std::string& s) {
    char* end = nullptr;
    const std::string u = trim(s);
    const double d = std::strtod(u.c_str(), &end);
    if (u.empty() || *end || !std::isfinite(d)) throw bad("bad number '" + u + "'");
    return d;
  };
  if (t.find(':') != std::string::npos) {
    const size_t a = t.find(':'), b = t.find(':', a + 1);
    if (b == std::string::npos || t.find(':', b + 1) != std::string::npos) throw bad("range must be lo:hi:n");
    const double lo = to_d(t.substr(0, a)), hi = to_d(t.substr(a + 1, b - a - 1));
    const std::string ns = trim(t.substr(b + 1));
    char* end = nullptr;
    const long n = std::strtol(ns.c_str(), &end, 10);
    if (ns.empty() || *end || n < 1) throw bad("range count must be a positive integer");
    if (logsp && !(lo > 0.0 && hi > 0.0)) throw bad("log range needs positive bounds");
    for (long k = 0; k < n; ++k) {
      double x;
      if (n == 1 || k == 0) x = lo;
      else if (k == n - 1) x = hi;
      else if (logsp) x = std::exp(std::log(lo) + (std::log(hi) - std::log(lo)) * static_cast<double>(k) / static_cast<double>(n - 1));
      else x = lo + (hi - lo) * static_cast<double>(k) / static_cast<double>(n - 1);
      v.push_back(x);
    }
  } else {
    if (logsp) throw bad("'log' applies to lo:hi:n ranges only");
    size_t s = 0;
    for (;;) {
      const size_t c = t.find(',', s);
      v.push_back(to_d(t.substr(s, c == std::string::npos ? std::string::npos : c - s)));
      if (c == std::string::npos) break;
      s = c + 1;
    }
  }
  return v;
}

SweepFile parse_sweep_file(const std::string& text) {
  SweepFile sf;
  std::istringstream in(text);
  std::string raw;
  long ln = 0;
  while (std::getline(in, raw)) {
    ++ln;
    const size_t h = raw.find('#');
    const std::string line = trim(h == std::string::npos ? raw : raw.substr(0, h));
    if (line.empty()) continue;
    const size_t sp = line.find_first_of(" \t");
    const std::string kw = line.substr(0, sp);
    const std::string rest = sp == std::string::npos ? "" : trim(line.substr(sp));
    auto bad = [&](const std::string& m) -> Fail { return Fail{KIN_EXIT_INPUT, "sweep file line " + std::to_string(ln) + ": " + m}; };
    if (kw == "axis") {
      const size_t eq = rest.find('=');
      if (eq == std::string::npos) throw bad("expected 'axis <param> = <values>'");
      Axis a;
      a.name = trim(rest.substr(0, eq));
      if (a.name.empty()) throw bad("missing axis name");
      a.values = parse_values(rest.substr(eq + 1), ln);
      sf.axes.push_back(a);
    } else if (kw == "runs") {
      char* end = nullptr;
      const long long r = std::strtoll(rest.c_str(), &end, 10);
      if (rest.empty() || *end || r < 1) throw bad("runs must be a positive integer");
      sf.runs = static_cast<uint64_t>(r);
    } else if (kw == "seed") {
      char* end = nullptr;
      if (rest.empty() || rest[0] == '-') throw bad("seed must be a non-negative integer");
      sf.seed = std::strtoull(rest.c_str(), &end, 0);
      if (*end) throw bad("seed must be a non-negative integer");
    } else if (kw == "method") {
      std::istringstream ms(rest);
      std::string tok;
      ms >> sf.method.name;
      while (ms >> tok) {
        const size_t eq = tok.find('=');
        if (eq == std::string::npos) throw bad("method options are key=value");
        const std::string k = tok.substr(0, eq), v = tok.substr(eq + 1);
        char* end = nullptr;
        const double d = std::strtod(v.c_str(), &end);
        if (v.empty() || *end) throw bad("bad value for method option '" + k + "'");
        if (k == "epsilon") sf.method.epsilon = d;
        else if (k == "tau") sf.method.tau = d;
        else if (k == "rtol") sf.method.rtol = d;
        else if (k == "atol") sf.method.atol = d;
        else if (k == "max_steps") sf.method.max_steps = static_cast<uint64_t>(d);
        else if (k == "theta_x") sf.method.theta_x = d;
        else if (k == "theta_a") sf.method.theta_a = d;
        else if (k == "repartition") sf.method.repartition = d;
        else throw bad("unknown method option '" + k + "'");
      }
      sf.have_method = true;
    } else {
      throw bad("unknown keyword '" + kw + "'");
    }
  }
  if (!sf.have_method) input("sweep file: missing 'method' line");
  return sf;
}

// ---- flags ------------------------------------------------------------------
struct Flags {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k) const {
    auto it = kv.find(k);
    if (it == kv.end()) usage("missing required flag " + k);
    return it->second;
  }
};

Flags parse_flags(const std::vector<std::string>& args, size_t from, const std::vector<std::string>& allowed) {
  Flags f;
  for (size_t i = from; i < args.size(); ++i) {
    const std::string& a = args[i];
    bool ok = false;
    for (const auto& al : allowed) ok |= a == al;
    if (!ok) usage("unknown flag '" + a + "'");
    if (i + 1 >= args.size()) usage("flag " + a + " needs a value");
    if (f.kv.count(a)) usage("flag " + a + " given twice");
    f.kv[a] = args[++i];
  }
  return f;
}

// ---- execution ----------------------------------------------------------------
struct Model {
  kin_model_text* m = nullptr;
  ~Model() { kin_model_text_free(m); }
};

struct Ctx {
  kin_ctx* ctx = nullptr;
  kin_model* model = nullptr;
  ~Ctx() {
    if (model) kin_model_free(model);
    if (ctx) kin_ctx_destroy(ctx);
  }
};

int workers_wanted(const Flags& f) {
  long w = 0;
  if (const char* e = std::getenv("KINETICS_WORKERS")) {  // env overrides --workers
    char* end = nullptr;
    w = std::strtol(e, &end, 10);
    if (!*e || *end || w < 1) usage(std::string("bad KINETICS_WORKERS '") + e + "'");
  } else if (f.has("--workers")) {
    w = static_cast<long>(unum("--workers", f.get("--workers")));
    if (w < 1) usage("--workers must be >= 1");
  }
  const int vis = kin_visible_devices();
  if (vis <= 0) throw Fail{KIN_EXIT_SIMULATION, "no CUDA device visible (this engine runs on B200 GPUs)"};
  return w == 0 ? vis : static_cast<int>(std::min<long>(w, vis));
}

int sim_error(int rc, const kin_error& e, const std::string& what) {
  const int code = rc == KIN_ERR_INPUT ? KIN_EXIT_INPUT : rc == KIN_ERR_USAGE ? KIN_EXIT_USAGE : KIN_EXIT_SIMULATION;
  std::string m = what + ": " + e.message;
  if (rc == KIN_ERR_SIMULATION)
    m += " (simulation " + std::to_string(e.sim_index) + ", point " + std::to_string(e.point_index) + ", run " +
         std::to_string(e.run_index) + ")";
  throw Fail{code, m};
}

struct Common {
  std::string model_path, model_text, out;
  Model model;
  int max_order = 2;
  int rng = KIN_RNG_COMPAT;
  double t_end = 0.0;
  uint64_t samples = 0;
  int workers = 1;
  std::vector<double> grid;
};

void load_common(const Flags& f, Common* c) {
  c->model_path = f.get("--model");
  c->out = f.get("--out");
  c->t_end = num("--t-end", f.get("--t-end"));
  c->samples = unum("--samples", f.get("--samples"));
  if (!(c->t_end >= 0.0) || !std::isfinite(c->t_end)) usage("--t-end must be a finite non-negative number");
  if (c->samples < 2) usage("--samples must be >= 2 (grid points including t=0 and t_end)");
  if (f.has("--max-order")) {
    const uint64_t mo = unum("--max-order", f.get("--max-order"));
    if (mo != 2 && mo != 3) usage("--max-order must be 2 or 3");
    c->max_order = static_cast<int>(mo);
  }
  if (f.has("--rng")) {
    const std::string r = f.get("--rng");
    if (r == "compat") c->rng = KIN_RNG_COMPAT;
    else if (r == "philox") c->rng = KIN_RNG_PHILOX;
    else usage("--rng must be compat or philox");
  }
  for (uint64_t g = 0; g < c->samples; ++g)  // uniform grid t_end*g/(G-1), both ends exact
    c->grid.push_back(c->t_end * static_cast<double>(g) / static_cast<double>(c->samples - 1));
  if (!read_file(c->model_path, &c->model_text)) input("cannot read model file '" + c->model_path + "'");
  kin_error e;
  if (kin_model_parse(c->model_text.data(), static_cast<int64_t>(c->model_text.size()), c->max_order, &c->model.m,
                      &e) != KIN_OK)
    input(c->model_path + ": " + e.message);
}

void open_engine(Common& c, const Flags& f, Ctx* x) {
  c.workers = workers_wanted(f);
  std::vector<int32_t> ids;
  for (int i = 0; i < c.workers; ++i) ids.push_back(i);
  kin_error e;
  int rc = kin_ctx_create(ids.data(), static_cast<int32_t>(ids.size()), &x->ctx, &e);
  if (rc) sim_error(rc, e, "device setup");
  rc = kin_model_upload(x->ctx, kin_model_text_desc(c.model.m), &x->model, &e);
  if (rc) sim_error(rc, e, "model");
}

std::vector<const char*> species_names(const Common& c) {
  std::vector<const char*> v;
  const kin_model_desc* d = kin_model_text_desc(c.model.m);
  for (int i = 0; i < d->n_species; ++i) v.push_back(kin_model_text_species_name(c.model.m, i));
  return v;
}

struct Written {
  uint64_t bytes = 0, hash = 0;
};

Written write_csv(const kin_csv_table& t, const std::string& path) {
  Written w;
  kin_error e;
  if (kin_csv_write(&t, path.c_str(), 0, &w.bytes, &w.hash, &e) != KIN_OK) input(e.message);
  return w;
}

void write_manifest(const std::string& out, const std::vector<std::string>& args,
                    const std::vector<std::pair<std::string, std::string>>& fields, const Written& w, double secs) {
  std::ofstream m(out + ".manifest", std::ios::binary);
  if (!m) input("cannot write manifest '" + out + ".manifest'");
  m << "# kinetics-b200 run manifest (SPEC.md:471-474); replay: kinetics-b200 replay " << out << ".manifest\n";
  m << "tool = kinetics-b200\ntool_version = " << kToolVersion << "\nabi_version = " << kin_abi_version() << "\n";
  for (size_t i = 1; i < args.size(); ++i) m << "arg = " << args[i] << "\n";
  for (const auto& kv : fields) m << kv.first << " = " << kv.second << "\n";
  m << "output = " << out << "\noutput_bytes = " << w.bytes << "\noutput_fnv1a64 = " << hex64(w.hash) << "\n";
  m << "wall_seconds = " << fmt(secs) << "\n";
}

std::vector<std::pair<std::string, std::string>> common_fields(const Common& c, const std::string& method_label,
                                                               const MethodSpec& ms) {
  return {{"model", c.model_path},
          {"model_fnv1a64", hex64(kin_fnv1a64(c.model_text.data(), c.model_text.size()))},
          {"method", method_label},
          {"epsilon", fmt(ms.epsilon)},
          {"tau", fmt(ms.tau)},
          {"rel_tol", fmt(ms.rtol)},
          {"abs_tol", fmt(ms.atol)},
          {"max_steps", std::to_string(ms.max_steps)},
          {"theta_x", fmt(ms.theta_x)},
          {"theta_a", fmt(ms.theta_a)},
          {"repartition_interval", fmt(ms.repartition)},
          {"rng", c.rng == KIN_RNG_PHILOX ? "philox" : "compat"},
          {"max_order", std::to_string(c.max_order)},
          {"t_end", fmt(c.t_end)},
          {"samples", std::to_string(c.samples)},
          {"workers", std::to_string(c.workers)}};
}

int cmd_simulate(const std::vector<std::string>& args, Written* result) {
  const auto t0 = std::chrono::steady_clock::now();
  const Flags f = parse_flags(args, 2, {"--model", "--method", "--t-end", "--samples", "--seed", "--runs",
                                        "--epsilon", "--tau", "--rtol", "--atol", "--tol", "--max-steps", "--rng",
                                        "--max-order", "--workers", "--out", "--theta-x", "--theta-a", "--repartition"});
  MethodSpec ms;
  ms.name = f.get("--method");
  const uint64_t seed = unum("--seed", f.get("--seed"));
  const uint64_t runs = f.has("--runs") ? unum("--runs", f.get("--runs")) : 1;
  if (runs < 1) usage("--runs must be >= 1");
  if (f.has("--epsilon")) ms.epsilon = num("--epsilon", f.get("--epsilon"));
  if (f.has("--tau")) ms.tau = num("--tau", f.get("--tau"));
  if (f.has("--rtol")) ms.rtol = num("--rtol", f.get("--rtol"));
  if (f.has("--atol")) ms.atol = num("--atol", f.get("--atol"));
  if (f.has("--tol")) {
    const std::string t = f.get("--tol");
    const size_t c = t.find(',');
    ms.rtol = num("--tol", t.substr(0, c));
    if (c != std::string::npos) ms.atol = num("--tol", t.substr(c + 1));
  }
  if (f.has("--max-steps")) ms.max_steps = unum("--max-steps", f.get("--max-steps"));
  if (f.has("--theta-x")) ms.theta_x = num("--theta-x", f.get("--theta-x"));  // "inf" accepted
  if (f.has("--theta-a")) ms.theta_a = num("--theta-a", f.get("--theta-a"));
  if (f.has("--repartition")) ms.repartition = num("--repartition", f.get("--repartition"));
  if (ms.name != "tau" && ms.name != "cle" && f.has("--tau")) usage("--tau applies to --method tau or cle");
  Common c;
  load_common(f, &c);
  check_method(ms);
  if ((f.has("--theta-x") || f.has("--theta-a") || f.has("--repartition")) && ms.name != "hybrid")
    usage("--theta-x/--theta-a/--repartition apply to --method hybrid");
  Ctx x;
  open_engine(c, f, &x);
  const kin_model_desc* md = kin_model_text_desc(c.model.m);
  const int N = md->n_species, G = static_cast<int>(c.samples);
  kin_sweep_desc d;
  std::memset(&d, 0, sizeof d);
  d.method = ms.to_c();
  d.n_axes = 0;
  d.runs_per_point = runs;
  d.master_seed = seed;
  d.t_end = c.t_end;
  d.n_grid = G;
  d.grid = c.grid.data();
  d.rng_mode = c.rng;
  d.seed_mode = runs == 1 ? KIN_SEED_DIRECT : KIN_SEED_ENSEMBLE;  // run_single(seed) / run_ensemble(master)
  std::vector<double> traj, mean, m2;
  kin_sweep_out o;
  std::memset(&o, 0, sizeof o);
  std::vector<uint64_t> meta(runs * 6);
  std::vector<int32_t> status(runs);
  o.meta = meta.data();
  o.status = status.data();
  if (runs == 1) {
    traj.resize(static_cast<size_t>(G) * N);
    o.traj = traj.data();
  } else {
    mean.resize(static_cast<size_t>(G) * N);
    m2.resize(static_cast<size_t>(G) * N);
    o.mean = mean.data();
    o.m2 = m2.data();
  }
  kin_error e;
  const int rc = kin_sweep_run(x.ctx, x.model, &d, &o, &e);
  if (rc) sim_error(rc, e, "simulate");
  const auto names = species_names(c);
  kin_csv_table t;
  std::memset(&t, 0, sizeof t);
  t.kind = runs == 1 ? KIN_CSV_TRAJECTORY : KIN_CSV_STATISTICS;
  t.n_species = N;
  t.species = names.data();
  t.n_grid = G;
  t.grid = c.grid.data();
  t.samples = traj.data();
  t.mean = mean.data();
  t.m2 = m2.data();
  t.n_runs = runs;
  const Written w = write_csv(t, c.out);
  auto fields = common_fields(c, ms.label(), ms);
  fields.insert(fields.begin(), {"command", "simulate"});
  fields.push_back({"seed", std::to_string(seed)});
  fields.push_back({"runs", std::to_string(runs)});
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  write_manifest(c.out, args, fields, w, secs);
  if (result) *result = w;
  return KIN_EXIT_OK;
}

int cmd_sweep(const std::vector<std::string>& args, Written* result) {
  const auto t0 = std::chrono::steady_clock::now();
  const Flags f = parse_flags(args, 2, {"--model", "--sweep", "--t-end", "--samples", "--rng", "--max-order",
                                        "--workers", "--out"});
  Common c;
  const std::string sweep_path = f.get("--sweep");
  load_common(f, &c);
  std::string stext;
  if (!read_file(sweep_path, &stext)) input("cannot read sweep file '" + sweep_path + "'");
  const SweepFile sf = parse_sweep_file(stext);
  check_method(sf.method);
  const kin_model_desc* md = kin_model_text_desc(c.model.m);
  std::vector<kin_sweep_axis> axes;
  std::vector<std::string> axis_names;
  for (const Axis& a : sf.axes) {
    kin_sweep_axis ax;
    std::memset(&ax, 0, sizeof ax);
    if (a.name.rfind("init:", 0) == 0) {
      const int32_t s = kin_model_text_species_index(c.model.m, a.name.substr(5).c_str());
      if (s < 0) input("sweep axis names undeclared species '" + a.name.substr(5) + "'");
      ax.kind = KIN_AXIS_INITIAL;
      ax.index = s;
    } else {
      const int32_t p = kin_model_text_param_index(c.model.m, a.name.c_str());
      if (p < 0) input("sweep axis names undeclared parameter '" + a.name + "'");
      ax.kind = KIN_AXIS_PARAM;
      ax.index = p;
    }
    ax.n_values = static_cast<int32_t>(a.values.size());
    ax.values = a.values.data();
    axes.push_back(ax);
    axis_names.push_back(a.name);
  }
  Ctx x;
  open_engine(c, f, &x);
  kin_sweep_desc d;
  std::memset(&d, 0, sizeof d);
  d.method = sf.method.to_c();
  d.n_axes = static_cast<int32_t>(axes.size());
  d.axes = axes.data();
  d.runs_per_point = sf.runs;
  d.master_seed = sf.seed;
  d.t_end = c.t_end;
  d.n_grid = static_cast<int32_t>(c.samples);
  d.grid = c.grid.data();
  d.rng_mode = c.rng;
  d.seed_mode = KIN_SEED_SWEEP;
  uint64_t P = 0, S = 0;
  kin_error e;
  int rc = kin_sweep_size(&d, &P, &S, &e);
  if (rc) sim_error(rc, e, "sweep");
  const size_t GN = static_cast<size_t>(c.samples) * md->n_species;
  std::vector<double> mean(P * GN), m2(P * GN);
  std::vector<uint64_t> meta(S * 6);
  std::vector<int32_t> status(S);
  kin_sweep_out o;
  std::memset(&o, 0, sizeof o);
  o.meta = meta.data();
  o.status = status.data();
  o.mean = mean.data();
  o.m2 = m2.data();
  rc = kin_sweep_run(x.ctx, x.model, &d, &o, &e);
  if (rc) sim_error(rc, e, "sweep");
  // point coordinates, Cartesian with the last axis fastest
  std::vector<double> coords(P * axes.size());
  for (uint64_t p = 0; p < P; ++p) {
    uint64_t rem = p;
    for (int a = static_cast<int>(axes.size()) - 1; a >= 0; --a) {
      const uint64_t nv = static_cast<uint64_t>(axes[a].n_values);
      coords[p * axes.size() + a] = axes[a].values[rem % nv];
      rem /= nv;
    }
  }
  const auto names = species_names(c);
  std::vector<const char*> anames;
  for (const auto& s : axis_names) anames.push_back(s.c_str());
  kin_csv_table t;
  std::memset(&t, 0, sizeof t);
  t.kind = KIN_CSV_SWEEP;
  t.n_species = md->n_species;
  t.species = names.data();
  t.n_grid = static_cast<int32_t>(c.samples);
  t.grid = c.grid.data();
  t.n_axes = static_cast<int32_t>(anames.size());
  t.axis_names = anames.data();
  t.n_points = P;
  t.point_values = coords.data();
  t.mean = mean.data();
  t.m2 = m2.data();
  t.n_runs = sf.runs;
  const Written w = write_csv(t, c.out);
  auto fields = common_fields(c, sf.method.label(), sf.method);
  fields.insert(fields.begin(), {"command", "sweep"});
  fields.push_back({"sweep", sweep_path});
  fields.push_back({"sweep_fnv1a64", hex64(kin_fnv1a64(stext.data(), stext.size()))});
  fields.push_back({"seed", std::to_string(sf.seed)});
  fields.push_back({"runs", std::to_string(sf.runs)});
  fields.push_back({"points", std::to_string(P)});
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  write_manifest(c.out, args, fields, w, secs);
  if (result) *result = w;
  return KIN_EXIT_OK;
}

int run(const std::vector<std::string>& args, Written* result);

// replay: re-run the manifest's argument list and check the output hash
int cmd_replay(const std::vector<std::string>& args) {
  if (args.size() != 3) usage("replay takes exactly one MANIFEST path");
  std::string text;
  if (!read_file(args[2], &text)) input("cannot read manifest '" + args[2] + "'");
  std::vector<std::string> argv{args[0]};
  std::map<std::string, std::string> kv;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    const size_t eq = line.find(" = ");
    if (eq == std::string::npos) input("malformed manifest line '" + line + "'");
    const std::string k = line.substr(0, eq), v = line.substr(eq + 3);
    if (k == "arg") argv.push_back(v);
    else kv[k] = v;
  }
  if (argv.size() < 2 || (argv[1] != "simulate" && argv[1] != "sweep")) input("manifest holds no replayable command");
  for (const char* key : {"model", "sweep"}) {
    if (!kv.count(key)) continue;
    std::string content;
    if (!read_file(kv[key], &content)) input(std::string("cannot read ") + key + " file '" + kv[key] + "'");
    if (hex64(kin_fnv1a64(content.data(), content.size())) != kv[std::string(key) + "_fnv1a64"])
      input(std::string(key) + " file '" + kv[key] + "' changed since the manifest was written");
  }
  Written w;
  const int rc = run(argv, &w);
  if (rc) return rc;
  if (hex64(w.hash) != kv["output_fnv1a64"] || std::to_string(w.bytes) != kv["output_bytes"])
    throw Fail{KIN_EXIT_SIMULATION, "replay produced different output (fnv1a64 " + hex64(w.hash) + ", manifest " +
                                        kv["output_fnv1a64"] + ")"};
  std::fprintf(stdout, "replay ok: %s (%s bytes, fnv1a64 %s)\n", kv["output"].c_str(), kv["output_bytes"].c_str(),
               kv["output_fnv1a64"].c_str());
  return KIN_EXIT_OK;
}

int run(const std::vector<std::string>& args, Written* result) {
  if (args.size() < 2) usage("missing command");
  const std::string& cmd = args[1];
  if (cmd == "--help" || cmd == "-h" || cmd == "help") {
    std::fputs(kUsage, stdout);
    return KIN_EXIT_OK;
  }
  if (cmd == "--version") {
    std::printf("kinetics-b200 %s (kin_abi %d)\n", kToolVersion, kin_abi_version());
    return KIN_EXIT_OK;
  }
  if (cmd == "simulate") return cmd_simulate(args, result);
  if (cmd == "sweep") return cmd_sweep(args, result);
  if (cmd == "replay") return cmd_replay(args);
  if (cmd == "cme") input("the 'cme' command is not part of this engine (the sweep hot path only)");
  usage("unknown command '" + cmd + "'");
}

}  // namespace

extern "C" int kin_cli_main(int32_t argc, const char* const* argv) {
  std::vector<std::string> args;
  for (int32_t i = 0; i < argc; ++i) args.emplace_back(argv[i] ? argv[i] : "");
  if (args.empty()) args.emplace_back("kinetics-b200");
  try {
    return run(args, nullptr);
  } catch (const Fail& f) {
    std::fprintf(stderr, "kinetics-b200: %s\n", f.msg.c_str());
    if (f.code == KIN_EXIT_USAGE) std::fputs(kUsage, stderr);
    return f.code;
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "kinetics-b200: internal error: %s\n", ex.what());
    return KIN_EXIT_SIMULATION;
  }
}

/*
 * kin_abi.h — C ABI of the B200 batched reaction-kinetics sweep engine.
 *
 * This is the drop-in boundary for the reference's ensemble layer
 * (/root/reference/proj/include/kinetics/ensemble.hpp).  The reference has no
 * FFI of its own: its seam is the C++ API
 *
 *   SweepResults  parameter_sweep(const ReactionNetwork&, const SweepConfig&,
 *                                 unsigned workers);          ensemble.hpp:129-130
 *   EnsembleStatistics run_ensemble(const ReactionNetwork&,
 *                                 const EnsembleOptions&, const RunSink&);
 *                                                             ensemble.hpp:97-99
 *   Trajectory    run_single(const ReactionNetwork&, const Method&, double t_end,
 *                            const std::vector<double>& grid, uint64_t seed);
 *                                                             ensemble.hpp:74-76
 *
 * Each of those is replaced by one call below (kin_sweep_run covers all three:
 * run_ensemble is a sweep with zero axes, run_single a sweep with zero axes and
 * one run whose seed is given directly).  Plain C types only: borrowed const
 * pointers for inputs, caller-allocated host buffers for outputs, an opaque
 * context owning device memory.  No exceptions cross the ABI; errors map 1:1 to
 * the reference's exception classes (errors.hpp:8-44) and CLI exit codes
 * (cli.hpp:7-13).
 */
#ifndef KIN_ABI_H_
#define KIN_ABI_H_

#ifndef __CUDACC_RTC__
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define KIN_ABI_VERSION 3

/* ---- status codes (cli.hpp:8-13 ExitCode; errors.hpp classes) ------------ */
enum kin_status {
  KIN_OK = 0,
  KIN_ERR_INPUT = 1,      /* ParseError / ValidationError (errors.hpp:14-37)   */
  KIN_ERR_SIMULATION = 2, /* SimulationError (errors.hpp:39-44)                */
  KIN_ERR_DEVICE = 3,     /* CUDA failure (new: no reference counterpart)      */
  KIN_ERR_USAGE = 64      /* bad arguments (cli.hpp:12 kExitUsage)             */
};

/* per-simulation status word written by the kernels (SimulationError causes) */
enum kin_sim_status {
  KIN_SIM_OK = 0,
  KIN_SIM_BUDGET = 1,      /* step budget (IntegratorConfig::max_steps) exhausted */
  KIN_SIM_NONFINITE = 2,   /* integrator produced a non-finite value              */
  KIN_SIM_NEGATIVE = 3,    /* apply_reaction would go negative (model.hpp:159-163)*/
  KIN_SIM_STEP_UNDERFLOW = 4 /* step size underflow                               */
};

/* ---- model: ReactionNetwork (model.hpp:13-95) ---------------------------- */
/* Reactant / product multisets are given CSR-by-reaction, species ascending
 * inside each reaction (std::map order, model.hpp:33-34).  nu, its sparse
 * columns/rows and g_i (highest reactant order) are derived by the loader. */
typedef struct kin_model_desc {
  int32_t n_species;
  int32_t n_reactions;
  int32_t n_params;
  const int64_t* initial_amounts;   /* [n_species]  Species::initial_amount  */
  const double* rate_constants;     /* [n_reactions] Reaction::rate_constant */
  const int32_t* rate_param;        /* [n_reactions] param index or -1; NULL = none bound */
  const double* param_values;       /* [n_params]   Parameter::value         */
  const int32_t* reactant_ptr;      /* [n_reactions+1]                        */
  const int32_t* reactant_species;  /* [reactant_ptr[M]]                      */
  const int32_t* reactant_stoich;   /* [reactant_ptr[M]]  > 0                 */
  const int32_t* product_ptr;       /* [n_reactions+1]                        */
  const int32_t* product_species;
  const int32_t* product_stoich;
  int32_t max_order;                /* 2 = reference (model.hpp:38); 3 enables the
                                       order-3 extension (Schlogl, Brusselator) */
} kin_model_desc;

/* ---- method: Method (ensemble.hpp:59-71) + IntegratorConfig --------------- */
enum kin_method_kind {          /* Method::Kind order, ensemble.hpp:62 */
  KIN_METHOD_SSA = 0,
  KIN_METHOD_TAU_ADAPTIVE = 1,
  KIN_METHOD_TAU_FIXED = 2,
  KIN_METHOD_CLE = 3,           /* Chemical Langevin, Euler-Maruyama with step tau (stochastic.hpp:64-75) */
  KIN_METHOD_ODE = 4,           /* Dopri5 RRE, deterministic.hpp:38-95 */
  KIN_METHOD_HYBRID = 5,        /* PDMP: fast reactions by RRE, slow ones by hazard-inversion jumps (hybrid.hpp) */
  KIN_METHOD_LSODA = 6          /* extension: Adams/BDF with stiffness switching */
};

typedef struct kin_integrator_config { /* deterministic.hpp:14-20 */
  double rel_tol;     /* default 1e-6 */
  double abs_tol;     /* default 1e-9 */
  double h_init;      /* 0 = automatic */
  double h_max;       /* +inf = unbounded */
  uint64_t max_steps; /* default 1e7; also bounds stochastic decisions+events */
} kin_integrator_config;

typedef struct kin_method {
  int32_t kind;       /* enum kin_method_kind */
  double tau;         /* TauFixed / Cle step */
  double epsilon;     /* TauAdaptive control, default 0.03 */
  kin_integrator_config integrator;
  /* HybridConfig (hybrid.hpp:21-26), read for KIN_METHOD_HYBRID only */
  double theta_x;              /* amount_threshold, reference default 100 (may be +inf) */
  double theta_a;              /* propensity_threshold, reference default 10 */
  double repartition_interval; /* 0 selects t_end / 100 */
  /* tau-leap firing law (TauAdaptive / TauFixed): enum kin_firing */
  int32_t firing;
} kin_method;

enum kin_firing {
  KIN_FIRING_POISSON = 0,   /* k_j ~ Poisson(a_j tau), reject + halve on a negative
                               amount (stochastic.hpp:53-57) — the reference */
  KIN_FIRING_BINOMIAL = 1   /* extension (north star): k_j ~ Binomial(n_j, p_j) with n_j the
                               reactant-limited firing bound after the reactions before j
                               consumed theirs, p_j = min(1, a_j tau / n_j): amounts never
                               go negative, so a leap is never rejected (Tian & Burrage 2004,
                               Chatterjee et al. 2005, sequential form) */
};

/* ---- sweep: SweepConfig (ensemble.hpp:101-113) ---------------------------- */
enum kin_axis_kind {
  KIN_AXIS_PARAM = 0,    /* rebinds Parameter `index` (with_param, model.hpp:78-80) */
  KIN_AXIS_INITIAL = 1,  /* extension: initial amount of species `index` (integral values) */
  KIN_AXIS_SCALE = 2     /* extension: global scale factor — multiplies the rate constant of
                            reactions [index, index + span) */
};

typedef struct kin_sweep_axis {
  int32_t kind;          /* enum kin_axis_kind */
  int32_t index;
  int32_t n_values;
  const double* values;
  int32_t span;          /* KIN_AXIS_SCALE: number of reactions scaled; else unused */
} kin_sweep_axis;

enum kin_rng_mode {
  KIN_RNG_COMPAT = 0,    /* xoshiro256++ stream per run, bit-compatible with rng.cpp */
  KIN_RNG_PHILOX = 1     /* counter-based Philox4x32-10 keyed per (run, step) */
};

enum kin_seed_mode {
  KIN_SEED_SWEEP = 0,    /* point master = derive(master, k); run seed = derive(point master, r) */
  KIN_SEED_ENSEMBLE = 1, /* run_ensemble: run seed = derive(master, r) (ensemble.hpp:91-99) */
  KIN_SEED_DIRECT = 2    /* run_single: the run seed is master_seed itself */
};

typedef struct kin_sweep_desc {
  kin_method method;
  int32_t n_axes;
  const kin_sweep_axis* axes;   /* Cartesian product, LAST axis fastest */
  uint64_t runs_per_point;
  uint64_t master_seed;
  int32_t seed_mode;            /* enum kin_seed_mode */
  int32_t rng_mode;             /* enum kin_rng_mode */
  double t_end;
  int32_t n_grid;
  const double* grid;           /* strictly increasing, within [0, t_end] */
  /* shard: global simulation indices [sim_begin, sim_end); sim = point*R + run.
     sim_end == 0 means "all".  Per-point statistics are produced only for points
     whose runs all lie inside the shard. */
  uint64_t sim_begin;
  uint64_t sim_end;
  /* interleaved point shard (multi-GPU across processes): this call
     simulates only the points p of [sim_begin, sim_end) (whole points: both
     bounds multiples of runs_per_point) with (p - p_first) % shard_count ==
     shard_index, and its outputs are COMPACT in shard order (local point k =
     global point p_first + shard_index + k*shard_count).  shard_count <= 1:
     every simulation of the range, outputs in global order. */
  int32_t shard_index;
  int32_t shard_count;
  int32_t output_mode;    /* enum kin_output_mode */
  int32_t lanes_per_sim;  /* 0 = automatic; Dopri5: 1/2/4/8/16/32 lanes per simulation;
                             Philox stochastic: 1 (thread per simulation) or 2..32 */
  uint32_t variant;       /* 0 = automatic; OR of enum kin_variant flags (forced kernel
                             choices — studies and tests; results never depend on them) */
  int32_t reserved_;
} kin_sweep_desc;

enum kin_output_mode {
  KIN_OUTPUT_FULL = 0,        /* every array the kin_sweep_out pointers request */
  KIN_OUTPUT_STATS_ONLY = 1   /* parameter_sweep / run_ensemble without a RunSink: per-point
                                 mean/m2 (+ meta/status/work) only; trajectories are never
                                 materialised whole — the runs go through a bounded device
                                 buffer in run-ascending sub-launches whose Welford
                                 accumulators continue across sub-launches (same result
                                 as KIN_OUTPUT_FULL, bit for bit); out->traj is ignored */
};

enum kin_variant {
  KIN_VARIANT_TABLE = 1u << 0,        /* stochastic: table-driven kernel, never the per-model JIT */
  KIN_VARIANT_JIT = 1u << 1,          /* stochastic: per-model JIT at any size */
  KIN_VARIANT_DOUBLE_STATE = 1u << 2, /* stochastic: double amounts (no int32 state) */
  KIN_VARIANT_GLOBAL_STATE = 1u << 3, /* per-simulation state in global memory */
  KIN_VARIANT_SMEM_STATE = 1u << 4,   /* per-simulation state in shared memory */
  KIN_VARIANT_NO_SPLIT = 1u << 5      /* JIT global state: keep x[] global too */
};
/* variant bits 8..13: simulations per warp (1..32) of the thread-per-simulation
   SSA/tau kernels; 0 = the occupancy fill rule */
#define KIN_VARIANT_WARP_LANES(w) ((uint32_t)(w) << 8)
/* variant bits 16..31: KIN_OUTPUT_STATS_ONLY window in simulations (tests;
   0 = the automatic 2 GiB trajectory budget) */
#define KIN_VARIANT_STATS_WINDOW(s) ((uint32_t)(s) << 16)

/* ---- outputs (caller-allocated HOST buffers; any may be NULL) ------------- */
typedef struct kin_sweep_out {
  double* traj;      /* [S][G][N]   Trajectory::samples per simulation of the shard */
  uint64_t* meta;    /* [S][6]      TrajectoryMeta {steps, rejected_leaps,
                                    clamp_events, fallback_ssa_steps, jumps, floored} */
  int32_t* status;   /* [S]         enum kin_sim_status */
  double* mean;      /* [P][G][N]   EnsembleStatistics mean (grid-major per point) */
  double* m2;        /* [P][G][N]   EnsembleStatistics m2 */
  uint64_t* work;    /* [S]         algorithmic FP64 op count per simulation (optional;
                                    selects the instrumented kernel variant) */
} kin_sweep_out;

typedef struct kin_error {
  int32_t code;            /* enum kin_status */
  int32_t sim_status;      /* enum kin_sim_status of the failing run */
  uint64_t sim_index;      /* lowest failing global simulation index */
  uint64_t point_index;
  uint64_t run_index;
  char message[256];
} kin_error;

/* ---- context / device ownership ------------------------------------------ */
typedef struct kin_ctx kin_ctx;
typedef struct kin_model kin_model;

/* merge_statistics (ensemble.hpp:56-57): fold (n_b, mean_b, m2_b) into
   (*n_a, mean_a, m2_a) by Chan's parallel update, element-wise over len values:
   delta = mean_b - mean_a; mean_a += delta*n_b/n; m2_a += m2_b + delta^2*n_a*n_b/n.
   Host function. */
void kin_stats_merge(uint64_t* n_a, double* mean_a, double* m2_a, uint64_t n_b, const double* mean_b,
                     const double* m2_b, uint64_t len);

/* Number of CUDA devices visible to this process (0 without a GPU). */
int32_t kin_visible_devices(void);

/* A context over the listed devices (device_ids NULL/n=0 → device 0; the same
   id may repeat: several slots on one GPU).  Every launch is asynchronous, so
   the calling thread enqueues all devices' work (kernels on per-device
   streams, copy-out on a copy stream) and returns; kin_sweep_wait collects.
   Calls on one context are serialised per device slot (internal locks);
   separate contexts are independent. */
int kin_ctx_create(const int32_t* device_ids, int32_t n_devices, kin_ctx** out,
                   kin_error* err);
void kin_ctx_destroy(kin_ctx* ctx);
int32_t kin_ctx_device_count(const kin_ctx* ctx);

/* ReactionNetwork::create validation (model.hpp:47-53) + upload of the packed
   device tables to every device of the context. */
int kin_model_upload(kin_ctx* ctx, const kin_model_desc* desc, kin_model** out,
                     kin_error* err);
void kin_model_free(kin_model* model);

/* Number of sweep points P and simulations S = P*R of a descriptor. */
int kin_sweep_size(const kin_sweep_desc* desc, uint64_t* n_points,
                   uint64_t* n_sims, kin_error* err);

/* parameter_sweep / run_ensemble / run_single (ensemble.hpp:74-130) end to end:
   H2D of the sweep tables, kernels on every device of the context (shard by
   whole-point chunks, cyclic), D2H into `out`.  Blocking. */
int kin_sweep_run(kin_ctx* ctx, const kin_model* model, const kin_sweep_desc* desc,
                  kin_sweep_out* out, kin_error* err);

/* run_ensemble (ensemble.hpp:91-99): n_runs runs of one model, run i seeded
   with derive_run_seed(master_seed, i); outputs as kin_sweep_run with one
   point (traj [n_runs][G][N], meta/status [n_runs], mean/m2 [G][N]).  Runs are
   split across the context's devices; their statistics are Chan-merged in
   ascending device-range order. */
int kin_ensemble_run(kin_ctx* ctx, const kin_model* model, const kin_method* method, uint64_t n_runs,
                     uint64_t master_seed, double t_end, const double* grid, int32_t n_grid, int32_t rng_mode,
                     kin_sweep_out* out, kin_error* err);

/* run_single (ensemble.hpp:73-76): one run seeded with `seed` itself;
   samples [G][N] and meta[6] (either may be NULL). */
int kin_run_single(kin_ctx* ctx, const kin_model* model, const kin_method* method, double t_end,
                   const double* grid, int32_t n_grid, uint64_t seed, int32_t rng_mode, double* samples,
                   uint64_t* meta, kin_error* err);

/* One device's share of a call (the partitioner's plan; ensemble.hpp:91-99
   worker ranges become devices).  Either INTERLEAVED — n_points whole points,
   global point pt_first + k*pt_stride for local point k, each with its R runs
   (the kernels map local -> global simulation index on the device) — or
   CONTIGUOUS — global simulations [sim_begin, sim_end).  Outputs land in the
   caller's layout at local simulation out_first + k*out_pitch (+ run), rows of
   R simulations (interleaved) or one row of sim_end - sim_begin (contiguous). */
typedef struct kin_sweep_part {
  int32_t device;       /* context device slot */
  int32_t interleaved;
  uint64_t sim_begin, sim_end;          /* contiguous parts */
  uint64_t pt_first, pt_stride, n_points; /* interleaved parts */
  uint64_t out_first, out_pitch;        /* caller-local simulation index of the first
                                           row and the distance between rows */
} kin_sweep_part;

/* The plan kin_sweep_run uses for n_devices GPUs over simulations [s0, s1)
   with R runs per point and the caller's shard (shard_index, shard_count):
   * one device: one part (everything);
   * whole points and at least as many points as devices: ONE interleaved part
     per device — device d takes the caller's points d, d+D, d+2D, ... (cyclic
     by point: balances the cost gradient along the sweep axes, and every
     device gets a single full-occupancy launch);
   * fewer points than devices (run_ensemble): min(S, D) equal contiguous run
     ranges whose cut points get their statistics Chan-merged in ascending
     part order (the reference's per-worker accumulators, ensemble.hpp:91-99);
   * a range that cuts points: D contiguous whole-point chunks.
   Pure host function (no device needed). */
int kin_sweep_plan(uint64_t s0, uint64_t s1, uint64_t runs_per_point, int32_t n_devices, int32_t shard_index,
                   int32_t shard_count, int32_t max_parts, kin_sweep_part* parts, int32_t* n_parts,
                   kin_error* err);

/* Caller-local sizes of a descriptor (its sim range and shard): n_points
   points with statistics (whole points inside the call) and n_sims
   simulations (the length of traj/meta/status/work). */
int kin_sweep_local_size(const kin_sweep_desc* desc, uint64_t* n_points, uint64_t* n_sims, kin_error* err);

/* Asynchronous form of kin_sweep_run: enqueue the sweep (kernels on the
   device's compute stream, copy-out into `out` on its copy stream)
   and return a ticket at once; kin_sweep_wait blocks until the results are in
   `out` and reports errors exactly as kin_sweep_run.  Copy-out of one sweep
   overlaps the kernels of the next.  Outputs must stay valid until the wait;
   with pageable (non-pinned) outputs the copy-out is synchronous. */
int kin_sweep_submit(kin_ctx* ctx, const kin_model* model, const kin_sweep_desc* desc,
                     kin_sweep_out* out, uint64_t* ticket, kin_error* err);
int kin_sweep_wait(kin_ctx* ctx, uint64_t ticket, kin_error* err);

/* ---- device-resident form (benchmarks, chained consumers) -----------------
   Runs the sweep on device `device_slot` of the context into context-owned
   device buffers, on the context's stream, WITHOUT any host copies.  The
   results stay resident until the next call; kin_sweep_fetch copies them out.
   kin_sweep_launch does not synchronize.  device_slot = -1: every slot of the
   context, each with its part of kin_sweep_plan (one launch per device);
   kin_sweep_sync / kin_sweep_fetch with -1 then cover all slots (fetch
   assembles the caller's layout). */
int kin_sweep_launch(kin_ctx* ctx, const kin_model* model,
                     const kin_sweep_desc* desc, int32_t device_slot,
                     int32_t want_stats, int32_t want_work, kin_error* err);
int kin_sweep_sync(kin_ctx* ctx, int32_t device_slot, kin_error* err);
int kin_sweep_fetch(kin_ctx* ctx, int32_t device_slot, kin_sweep_out* out,
                    kin_error* err);
/* cudaStream_t of the device slot, as void* (for event timing by the caller). */
void* kin_ctx_stream(kin_ctx* ctx, int32_t device_slot);
/* Device time (CUDA events on the slot's stream) of the last launch's
   simulation kernel and of its statistics kernel (0 when none ran).  Call
   after kin_sweep_sync. */
int kin_sweep_kernel_ms(kin_ctx* ctx, int32_t device_slot, double* sim_ms,
                        double* stats_ms, kin_error* err);
/* Name of the simulation kernel the last launch on this slot ran (as ncu
   lists it: "kin_jit_stoch", "stochastic_kernel", "stochastic_group_kernel",
   "dopri5_kernel", "lsoda_kernel"); "" before the first launch. */
const char* kin_sweep_kernel_name(kin_ctx* ctx, int32_t device_slot);

/* ---- seams (device unit kernels; SPEC "from_uniforms"/"from_counts") ----- */
uint64_t kin_splitmix64_mix(uint64_t v);                       /* rng.hpp:8-11 */
uint64_t kin_derive_run_seed(uint64_t master, uint64_t index);  /* ensemble.hpp:15-18 */
/* Device RNG draws from RngStream(seed): kind 0 next_u64, 1 draw_uniform,
   2 draw_normal, 3 draw_poisson(mean).  Results as raw 64-bit words. */
int kin_device_rng_draws(kin_ctx* ctx, uint64_t seed, int32_t kind, double mean,
                         int32_t n, uint64_t* out_bits, kin_error* err);

/* Device binomial draws (the KIN_FIRING_BINOMIAL sampler) from RngStream(seed):
   n_draws values of Binomial(n_trials, p), raw counts. */
int kin_device_binomial_draws(kin_ctx* ctx, uint64_t seed, uint64_t n_trials, double p, int32_t n_draws,
                              uint64_t* out, kin_error* err);

/* Device unit seams (SPEC's from_uniforms / from_counts / from_normals forms):
   one function of the path on one state x[N] of `model`, through the same
   device code the sweep kernels run (propensities from the packed tables).
     kind 0 propensities (model.hpp:151-157)          out[M] = a(x)
     kind 1 select_tau (stochastic.hpp:40-46)         params {eps} -> out[0] = tau (+inf if a0 = 0)
     kind 2 ssa_step_from_uniforms (:28-32)           params {u1, u2} -> out {dt, j} ({+inf, -1} if a0 = 0)
     kind 3 tau_leap_step_from_counts (:59-62)        params counts[M] -> out[0..N-1] = x', out[N] = rejected
     kind 4 cle_step_from_normals (:71-75)            params {h, z[M]} -> out[0..N-1] = x', out[N] = clamped
     kind 5 rre_rhs (deterministic.hpp:85-88)         out[N] = dx/dt = nu a(x)
     kind 6 rk_step (deterministic.hpp:26-36)         params {h, rel_tol, abs_tol} -> out[0..N-1] =
                                                      y(t+h) (5th order), out[N] = error norm,
                                                      out[N+1..2N] = f(y(t+h)) (FSAL) */
int kin_device_unit(kin_ctx* ctx, const kin_model* model, int32_t kind, const double* x, const double* params,
                    int32_t n_params, double* out, int32_t out_cap, kin_error* err);

/* Diagnostic: generate and NVRTC-compile (sm_100a) the per-model specialised
   stochastic kernel for this model + sweep binding, without a GPU.  log gets
   the compiler output. */
int kin_jit_check(const kin_model_desc* model, const kin_sweep_desc* sweep, char* log,
                  int32_t log_cap, kin_error* err);

/* Peak FP64 FMA throughput of device slot 0 (TFLOP/s, FMA = 2 flops), from a
   DFMA microbenchmark; used as the roofline denominator. */
int kin_measure_fp64_peak(kin_ctx* ctx, double* tflops, kin_error* err);

const char* kin_status_string(int32_t code);
int32_t kin_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KIN_ABI_H_ */

// kin_tables.h — host/device shared layout of the packed model tables and the
// per-launch sweep descriptor.
//
// The model (ReactionNetwork, model.hpp:44-95) is packed into ONE flat struct
// passed to every kernel as a __grid_constant__ parameter: it lives in the
// kernel-parameter constant bank, so the warp-uniform table walks of the
// thread-per-simulation kernels (loop over reactions j / species i, identical in
// every lane) are served by the constant cache as broadcasts, with no global
// state and no per-model __constant__ symbol (several models/sweeps can be in
// flight on different streams).
#pragma once

#ifdef __CUDACC_RTC__
// NVRTC (per-model JIT kernels, kin_jit.cpp): no libc headers
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned short uint16_t;
typedef short int16_t;
typedef unsigned char uint8_t;
typedef signed char int8_t;
#else
#include <stdint.h>
#endif

#define KIN_MAX_AXES 8
// internal per-simulation status: an int32 amount would overflow; the engine
// re-runs the launch with double amounts (never returned to callers)
#define KIN_SIM_INTERNAL_RETRY 100
#define KIN_TABLE_BYTES 30720
// threads per block of the thread-per-simulation stochastic kernels (a multiple
// of 32; per-thread state is strided by it in shared memory)
#ifndef KIN_STOCH_BLOCK
#define KIN_STOCH_BLOCK 32
#endif  // < 32764-byte kernel parameter limit (sm_70+, CUDA >= 12.1)

// packed entries
//   reactant term : species (bits 0-15) | stoich (bits 16-23)
//   nu entry      : index   (bits 0-15) | (delta + 128) (bits 16-23)
#define KIN_TERM_SPECIES(e) ((int)((e) & 0xFFFF))
#define KIN_TERM_STOICH(e) ((int)(((e) >> 16) & 0xFF))
#define KIN_NU_INDEX(e) ((int)((e) & 0xFFFF))
#define KIN_NU_DELTA(e) ((int)(((e) >> 16) & 0xFF) - 128)
//   reaction descriptor (uint64): reactant species t0,t1,t2 (16 bits each, bits
//   0-47), their stoichiometries (2 bits each, bits 48-53), number of reactant
//   terms (bits 54-55) and the sweep axis carrying c_j plus one (bits 56-63, 0 =
//   none).  Terms are species-ascending (std::map order, model.hpp:33).
#define KIN_RD_SPECIES(d, t) ((int)(((d) >> (16 * (t))) & 0xFFFF))
#define KIN_RD_STOICH(d, t) ((int)(((d) >> (48 + 2 * (t))) & 0x3))
#define KIN_RD_NTERMS(d) ((int)(((d) >> 54) & 0x3))
#define KIN_RD_AXIS(d) ((int)(((d) >> 56) & 0xFF) - 1)

struct KinTables {
  int32_t n;          // species
  int32_t m;          // reactions
  int32_t nnz;        // nonzeros of nu
  int32_t n_grid;
  int32_t fprop;      // algorithmic flops of one full propensity pass (FMA=2)
  int32_t pad0_;
  // byte offsets into blob
  uint32_t off_rate;      // double [m]   rate constant with NON-swept params resolved
  uint32_t off_rate_axis; // int8   [m]   -1, or sweep axis whose value is c_j
  uint32_t off_x0;        // double [n]   initial amounts (exact integers)
  uint32_t off_x0_axis;   // int8   [n]   -1, or sweep axis overriding x0_i
  uint32_t off_g;         // double [n]   g_i (highest reactant order, 1 if none), as double
  uint32_t off_rt_ptr;    // int16  [m+1] reactant CSR (species-ascending)
  uint32_t off_rt;        // uint32 [..]  packed reactant terms
  uint32_t off_col_ptr;   // int16  [m+1] nu columns (species-ascending)
  uint32_t off_col;       // uint32 [nnz] packed (species, delta)
  uint32_t off_row_ptr;   // int16  [n+1] nu rows (reaction-ascending)
  uint32_t off_row;       // uint32 [nnz] packed (reaction, delta)
  uint32_t off_grid;      // double [n_grid] sampling grid (0 when it did not fit: use SweepDev::grid)
  uint32_t off_rdesc;     // uint64 [m]   packed reaction descriptor (KIN_RD_* below)
  uint32_t off_dep_ptr;   // int16  [m+1] reactions whose propensity changes when j fires
  uint32_t off_dep;       // uint16 [..]
  uint32_t off_sp_perm;   // int16  [n]   species by descending nu-row length (0: identity; Dopri5 lane slots)
  uint32_t used;
  uint32_t off_rx_perm;   // int16  [m]   reactions by descending reactant-term count (0: identity)
  alignas(16) unsigned char blob[KIN_TABLE_BYTES];
};

struct KinSweepDev {
  // method (Method, ensemble.hpp:59-71; IntegratorConfig, deterministic.hpp:14-20)
  int32_t kind;
  int32_t rng_mode;
  double tau;
  double epsilon;
  double rel_tol, abs_tol, h_init, h_max;
  uint64_t max_steps;
  double hyb_theta_x, hyb_theta_a, hyb_rep;  // HybridConfig (hybrid.hpp:21-26)
  // sweep (SweepConfig, ensemble.hpp:106-113)
  int32_t n_axes;
  int32_t seed_mode;
  int32_t axis_kind[KIN_MAX_AXES];
  int32_t axis_n[KIN_MAX_AXES];
  const double* axis_values[KIN_MAX_AXES];  // device pointers
  uint64_t runs;        // runs per point R
  uint64_t master_seed;
  uint64_t sim_begin;   // contiguous parts: global index of part-local simulation 0
  uint64_t n_local;     // simulations in this launch
  // Interleaved parts (pt_stride > 0): part-local simulation l = k*runs + r is
  // run r of global point pt_first + k*pt_stride (kin_sweep_part).  A launch
  // covers part-local simulations [local_begin, local_begin + n_local); its
  // outputs are indexed from 0 (global_sim() below).
  uint64_t pt_first;
  uint64_t pt_stride;
  uint64_t local_begin;
  int32_t firing;       // enum kin_firing (tau methods)
  int32_t pad_firing_;
  double t_end;
  const double* grid;   // device pointer [n_grid]
  const double* lgamma_tab;  // device pointer [KIN_LGAMMA_N]: glibc lgamma(k+1)
  // Stochastic kernels, large models: per-simulation state in global memory
  // (null: shared memory).  Block b owns gstate + b * (its per-warp size); the
  // grid never exceeds gstate_warps blocks.
  double* gstate;
  uint64_t gstate_warps;
  // Simulations per warp of the thread-per-simulation kernels (1..32; 0 from
  // the engine = the launcher's fill rule kin_warp_lanes): fewer
  // than 32 when a launch cannot fill the resident warps, so that more warps
  // (each with fewer, less divergent lanes) share the latency.  Set by the
  // launchers (kin_warp_lanes); the per-simulation results do not depend on it.
  int32_t warp_lanes;
  // Global-memory state only: nonzero keeps the amounts x[] in shared memory
  // (the JIT kernel's split layout); the propensity cache stays in gstate.
  // Read by the launchers on the host.
  int32_t gstate_x_smem;
};

// Device outputs of one launch (local simulation index s in [0, n_local)).
struct KinOutDev {
  double* traj;      // [n_local][G][N]  the host layout: each emit is one contiguous run
  uint64_t* meta;    // [n_local][6]
  int32_t* status;   // [n_local]
  uint64_t* work;    // [n_local] or null
};

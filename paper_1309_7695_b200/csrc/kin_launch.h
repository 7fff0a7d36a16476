// kin_launch.h — host-side launchers of the engine's kernels (one per .cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/kin_abi.h"
#include "kin_tables.h"

namespace kin {

// Simulations per warp for a persistent thread-per-simulation SSA/tau launch
// over n_local simulations with `resident` warps: 32, or fewer when the launch
// would leave resident warps empty (a sweep of 16,384 simulations fills only
// 512 warps of 32; as 2,048 warps of 8 it fills 14 per SM).  It pays where the
// lanes' control flow is data-dependent (C2: 162 -> 75 ms); the CLE and hybrid
// kernels, with uniform work per simulation, keep full warps.  KIN_WARP_LANES
// overrides (studies).
int kin_warp_lanes(uint64_t n_local, uint64_t resident);

// kin_stochastic.cu: SSA / tau-adaptive / tau-fixed, thread per simulation.
// `counter` is a device word used by the persistent warps to fetch work;
// int_state stores amounts as int32 (more resident simulations) and sets
// *ovf_flag if one leaves int32 range (the caller re-runs with double amounts).
cudaError_t launch_stochastic(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                              unsigned long long* counter, int* ovf_flag, bool int_state, cudaStream_t stream);

// kin_stochastic_group.cu: Philox mode, L lanes per simulation (lanes <= 0 picks).
int stochastic_group_pick_lanes(int n_species, int n_reactions);
cudaError_t launch_stochastic_group(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                                    int lanes, unsigned long long* counter, cudaStream_t stream);

// kin_ode.cu: Dopri5 RRE integration, L lanes per simulation (L = 0 picks).
int ode_pick_lanes(int n_species);
cudaError_t launch_dopri5(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count, int lanes,
                          cudaStream_t stream);

// kin_lsoda.cu: LSODA-style Adams/BDF, thread per simulation, state in smem.
// coeffs: elco [2][13][14] then tesco [2][13][3] (device).
size_t lsoda_smem_bytes(const KinTables& T, const KinSweepDev& S);
size_t lsoda_state_doubles_per_warp(const KinTables& T, const KinSweepDev& S);
cudaError_t launch_lsoda(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count, const double* coeffs,
                         unsigned long long* counter, cudaStream_t stream);

// kin_stochastic.cu: unit seam (one path function on one state, kin_device_unit).
cudaError_t launch_unit(const KinTables& T, int kind, const double* x, const double* params, double* out,
                        cudaStream_t stream);
// kin_stochastic.cu: Chemical Langevin (Euler-Maruyama) sweep, double amounts.
cudaError_t launch_cle(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                       unsigned long long* counter, cudaStream_t stream);

// kin_hybrid.cu: hybrid PDMP sweep (one thread per simulation, smem state).
size_t hybrid_smem_bytes(const KinTables& T, const KinSweepDev& S);
size_t hybrid_state_doubles_per_warp(const KinTables& T, const KinSweepDev& S);
cudaError_t launch_hybrid(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                          unsigned long long* counter, cudaStream_t stream);

// kin_post.cu: statistics and utilities.
// per-point Welford over runs (ascending run order) of traj_dev [n_local][G*N]
// starting at local simulation first_sim -> mean/m2 [P][G*N]; n_done > 0
// continues accumulators holding the point's first n_done runs
cudaError_t launch_point_stats(const double* traj_dev, int gn, uint64_t runs, uint64_t first_sim, uint64_t n_points,
                               uint64_t n_done, double* mean, double* m2, cudaStream_t stream);
cudaError_t launch_binomial_draws(uint64_t seed, uint64_t n_trials, double p, int n, uint64_t* out,
                                  cudaStream_t stream);
cudaError_t launch_rng_draws(uint64_t seed, int kind, double mean, int n, uint64_t* out, const double* lgamma_tab,
                             cudaStream_t stream);
cudaError_t measure_fp64_peak(cudaStream_t stream, double* tflops);

}  // namespace kin

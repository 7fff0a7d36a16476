// kin_jit.h — per-model specialised stochastic kernels (kin_jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "kin_tables.h"

namespace kin {

// Model structure the generated policy is specialised on (no rate values).
struct JitModel {
  int n = 0, m = 0;
  std::vector<int> rt_ptr, rt_species, rt_stoich;    // reactants per reaction (species-ascending)
  std::vector<int> rate_axis;                        // -1, or the sweep axis carrying c_j
  std::vector<char> rate_scaled;                     // 1: c_j = rate_j * axis value (scale axis)
  std::vector<int> col_ptr, col_species, col_delta;  // nu columns
  std::vector<int> row_ptr, row_reaction, row_delta; // nu rows
  std::vector<int> dep_ptr, dep;                     // propensity dependency graph
  std::vector<double> g;                             // highest reactant order per species
  std::string policy;                                // generated source (jit_prepare), "" = not yet
};

// Generate the model's policy source once (cached in the JitModel).
void jit_prepare(JitModel* model);

// force: 1 always, 0 never, -1 by size (KIN_JIT=0/1, read once per process,
// overrides the size policy for tests)
bool jit_wanted(uint64_t n_sims, int force = -1);

// Generate + NVRTC-compile the policy without loading it (no GPU needed).
bool jit_compile_check(const JitModel& model, bool count, bool philox, bool int_state, std::string* log);
// the hybrid PDMP kernel specialised per model (kin_hybrid_impl.cuh with the
// generated GenModel<double> as its propensity / row-sum policy)
bool jit_compile_check_hybrid(const JitModel& model, bool count, bool philox, std::string* log);
cudaError_t launch_hybrid_jit(const JitModel& model, const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                              bool count, unsigned long long* counter, size_t smem, cudaStream_t stream, bool* used);
// the LSODA kernel with the generated policy's straight-line RHS
bool jit_compile_check_lsoda(const JitModel& model, bool count, std::string* log);
cudaError_t launch_lsoda_jit(const JitModel& model, const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                             const double* coeffs, bool count, unsigned long long* counter, size_t smem,
                             cudaStream_t stream, bool* used);

// Launch the specialised kernel; *used = false means "not available" (NVRTC
// failure or unsupported configuration): the caller launches the table kernel.
cudaError_t launch_stochastic_jit(const JitModel& model, const KinTables& T, const KinSweepDev& S,
                                  const KinOutDev& O, bool count, unsigned long long* counter, int* ovf_flag,
                                  bool int_state, cudaStream_t stream, bool* used);

}  // namespace kin

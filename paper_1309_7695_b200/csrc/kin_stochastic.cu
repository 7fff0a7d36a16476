// kin_stochastic.cu — batched exact-SSA and tau-leaping (K2 + K3 of DESIGN.md).
//
// One CUDA thread = one simulation (the paper's mapping), in
// "compat" RNG mode: each thread owns the reference's xoshiro256++ stream seeded
// by derive_run_seed (rng.cpp:25-48, ensemble.hpp:15-18), so firing counts are
// bit-identical to the CPU reference's.
//
// Per-thread state in shared memory, [slot][thread] layout (lanes touch
// consecutive 8-byte words: conflict-free): amounts x[N] and propensities a[M]
// (evaluated once per decision and reused by a0, select_tau, the Poisson means
// and the SSA selection; SSA events re-evaluate only the reactions whose
// reactants changed, via a dependency graph).  A leap updates x IN PLACE; a
// rejected leap is rolled back by replaying the attempt's draws from a saved
// copy of the RNG state (exact: integer-valued doubles).  Model tables are
// walked with warp-uniform indices out of the kernel-parameter constant bank.
// Persistent warps fetch 32 simulations at a time from a global counter, so the
// grid is exactly one wave and the tail is one simulation, not one block.
//
// Mirrors oracle/kin_oracle.cpp simulate_stochastic() operation for operation:
//   simulate_approx TauAdaptive/TauFixed ... stochastic.hpp:78-92
//   select_tau ............................. stochastic.hpp:40-46
//   tau_leap_step / rejection-halving ...... stochastic.hpp:48-57
//   ssa_step fallback (bursts of 100) ...... stochastic.hpp:22-26
//   simulate_ssa grid semantics ............ stochastic.hpp:34-38
// Compiled with -fmad=false (see Makefile): no contraction on the parity path.
#include "kin_launch.h"
#include "kin_stochastic_impl.cuh"

namespace kin {

namespace {

using stoch::kBlock;
using stoch::TableModel;

template <bool kCount, bool kPhilox, class XT>
__global__ void __launch_bounds__(stoch::kBlock) stochastic_kernel(const __grid_constant__ KinTables T,
                                                                   const __grid_constant__ KinSweepDev S, KinOutDev O,
                                                                   unsigned long long* __restrict__ next,
                                                                   int* ovf_flag) {
  stoch::stochastic_body<TableModel<XT>, kCount, kPhilox, XT>(T, S, O, next, ovf_flag);
}

size_t stochastic_smem_bytes(const KinTables& T, const KinSweepDev& S, int block, bool int_state) {
  return static_cast<size_t>(T.m + S.n_axes) * block * sizeof(double) +
         static_cast<size_t>(T.n) * block * (int_state ? sizeof(int32_t) : sizeof(double));
}

template <class XT>
cudaError_t launch_xt(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                      unsigned long long* counter, int* ovf_flag, cudaStream_t stream) {
  const size_t smem = stochastic_smem_bytes(T, S, kBlock, sizeof(XT) == 4);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  const bool ph = S.rng_mode == KIN_RNG_PHILOX;
  auto kern = count ? (ph ? stochastic_kernel<true, true, XT> : stochastic_kernel<true, false, XT>)
                    : (ph ? stochastic_kernel<false, true, XT> : stochastic_kernel<false, false, XT>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t warps = (S.n_local + 31) / 32;
  const uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  const unsigned grid = static_cast<unsigned>(warps < resident ? warps : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  kern<<<grid, kBlock, smem, stream>>>(T, S, O, counter, ovf_flag);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stochastic(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                              unsigned long long* counter, int* ovf_flag, bool int_state, cudaStream_t stream) {
  if (S.n_local == 0) return cudaSuccess;
  if (int_state) return launch_xt<int32_t>(T, S, O, count, counter, ovf_flag, stream);
  return launch_xt<double>(T, S, O, count, counter, ovf_flag, stream);
}

}  // namespace kin

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

#include <cstdlib>

namespace kin {

int kin_warp_lanes(uint64_t n_local, uint64_t resident) {
  static const int forced = [] {  // study/test override, read once per process
    const char* v = std::getenv("KIN_WARP_LANES");
    const int w = v ? std::atoi(v) : 0;
    return (w >= 1 && w <= 32) ? w : 0;
  }();
  if (forced) return forced;
  if (resident == 0) return 32;
  const uint64_t w = (n_local + resident - 1) / resident;
  return w >= 32 ? 32 : (w < 1 ? 1 : static_cast<int>(w));
}


namespace {

using stoch::kBlock;
using stoch::TableModel;

template <bool kCount, bool kPhilox, class XT, bool kGlobal>
__global__ void __launch_bounds__(stoch::kBlock) stochastic_kernel(const __grid_constant__ KinTables T,
                                                                   const __grid_constant__ KinSweepDev S, KinOutDev O,
                                                                   unsigned long long* __restrict__ next,
                                                                   int* ovf_flag) {
  stoch::stochastic_body<TableModel<XT>, kCount, kPhilox, XT, kGlobal>(T, S, O, next, ovf_flag);
}

// ---- Chemical Langevin Equation, Euler-Maruyama (stochastic.hpp:64-75) ------
// Mirrors oracle/kin_oracle.cpp simulate_cle: per step, propensities at the
// step start; per reaction j (index order) one normal z_j (compat:
// RngStream::draw_normal, Box-Muller with a cached spare, rng.cpp:54-66) and
// the increment a_j h + sqrt(a_j h) z_j applied along nu[:, j]; then negative
// components clamp to 0 (counted).  Steps truncate at grid times.
// Double amounts (the state is real-valued).  log/sin/cos are CUDA's (<= 1-2
// ulp from glibc's), so parity with the oracle is within a tolerance, not bit
// for bit.
// cle_step_from_normals pieces (stochastic.hpp:71-75), shared with the
// kin_device_unit seam: the increment a_j h + sqrt(a_j h) z_j, its application
// along nu[:, j], and the final clamp (count of components set to 0).
__device__ __forceinline__ double cle_increment(double aj, double h, double z) {
  const double d = __dmul_rn(aj, h);
  return __dadd_rn(d, __dmul_rn(sqrt(d), z));
}
template <int B>
__device__ __forceinline__ void cle_apply(const KinTables& T, double* x, int j, double inc) {
  const int p1 = tab_col_ptr(T, j + 1);
  for (int p = tab_col_ptr(T, j); p < p1; ++p) {
    const uint32_t e = tab_col(T, p);
    double* xs = x + KIN_NU_INDEX(e) * B;
    *xs = __dadd_rn(*xs, __dmul_rn(static_cast<double>(KIN_NU_DELTA(e)), inc));
  }
}
template <int B>
__device__ __forceinline__ uint64_t cle_clamp(double* x, int N, bool* bad) {
  uint64_t n = 0;
  for (int i = 0; i < N; ++i) {
    const double v = x[i * B];
    *bad |= !isfinite(v);
    if (v < 0.0) {
      x[i * B] = 0.0;
      ++n;
    }
  }
  return n;
}

template <bool kCount, bool kPhilox>
__device__ __forceinline__ void simulate_cle_one(const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                                                 uint64_t s, double* x, double* a, double* av) {
  constexpr int B = kBlock;
  const uint64_t sim = global_sim(S, s);
  const TableModel<double> sm{T, x, a, av};
  const int N = T.n, M = T.m, G = T.n_grid;
  stoch::init_state<double>(T, S, sim, N, x, av);
  const uint64_t seed = sim_seed(S, sim);
  Xoshiro rng;
  if (!kPhilox) rng.seed(seed);
  const double t_end = S.t_end, tau = S.tau;
  double t = 0.0;
  int gi = 0;
  uint64_t flops = 0, used = 0, step = 0, n_normal = 0, n_clamp = 0;
  int status = 0;
  bool spare_ok = false;
  double spare = 0.0;
  const uint64_t F_prop = static_cast<uint64_t>(T.fprop);
  auto emit = [&]() {
    double* o = O.traj + (static_cast<size_t>(s) * G + gi) * N;
    for (int i = 0; i < N; ++i) o[i] = x[i * B];
    ++gi;
  };
  while (gi < G && tab_grid(T, S, gi) <= t) emit();
  while (t < t_end) {
    if (++used > S.max_steps) { status = KIN_SIM_BUDGET; break; }
    const double t_stop = (gi < G && tab_grid(T, S, gi) < t_end) ? tab_grid(T, S, gi) : t_end;
    double h = tau;
    bool hit = false;
    const double gap = __dsub_rn(t_stop, t);
    if (kCount) flops += 1;
    if (!(h < gap)) { h = gap; hit = true; }
    sm.all_props(M);
    if (kCount) flops += F_prop;
    for (int j = 0; j < M; ++j) {
      double z;
      if (kPhilox) {
        PhiloxSite src(seed, step, static_cast<uint32_t>(j));
        const double u1 = src.uniform();
        const double u2 = src.uniform();
        z = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(2.0 * 3.141592653589793, u2)));
        if (kCount) flops += 4 + 3 + 1 + 2;
      } else if (spare_ok) {
        spare_ok = false;
        z = spare;
      } else {
        const double u1 = rng.uniform();
        const double u2 = rng.uniform();
        const double r = sqrt(__dmul_rn(-2.0, log(u1)));
        const double ang = __dmul_rn(2.0 * 3.141592653589793, u2);
        spare = __dmul_rn(r, sin(ang));
        spare_ok = true;
        z = __dmul_rn(r, cos(ang));
        if (kCount) flops += 4 + 3 + 1 + 2 + 2;
      }
      if (!kPhilox) ++n_normal;
      cle_apply<B>(T, x, j, cle_increment(sm.aval(j), h, z));
      if (kCount) flops += 4 + 2 * static_cast<uint64_t>(tab_col_ptr(T, j + 1) - tab_col_ptr(T, j));
    }
    bool bad = false;
    n_clamp += cle_clamp<B>(x, N, &bad);
    if (bad) { status = KIN_SIM_NONFINITE; break; }
    ++step;
    if (hit) {
      t = t_stop;
    } else {
      t = __dadd_rn(t, h);
      if (kCount) flops += 1;
    }
    while (gi < G && tab_grid(T, S, gi) <= t) emit();
  }
  while (gi < G) emit();
  (void)n_normal;
  uint64_t* me = O.meta + s * 6;
  me[0] = step;
  me[1] = 0;
  me[2] = n_clamp;
  me[3] = 0;
  me[4] = 0;
  me[5] = 0;
  O.status[s] = status;
  if (kCount && O.work) O.work[s] = flops;
}

template <bool kCount, bool kPhilox>
__global__ void __launch_bounds__(stoch::kBlock) cle_kernel(const __grid_constant__ KinTables T,
                                                            const __grid_constant__ KinSweepDev S, KinOutDev O,
                                                            unsigned long long* __restrict__ next) {
  extern __shared__ double smem[];
  constexpr int B = kBlock;
  const int tid = threadIdx.x, lane = tid & 31;
  double* a = smem + tid;
  double* av = smem + static_cast<size_t>(T.m) * B + tid;
  double* x = smem + static_cast<size_t>(T.m + S.n_axes) * B + tid;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, static_cast<unsigned long long>(S.warp_lanes));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (base >= S.n_local) break;
    const uint64_t s = lane < S.warp_lanes ? base + lane : S.n_local;  // lanes >= warp_lanes idle
    if (s < S.n_local) simulate_cle_one<kCount, kPhilox>(T, S, O, s, x, a, av);
    __syncwarp();
  }
}

// ---- unit seams (kin_device_unit): one path function on one state, through
// the same device code the sweep kernels run.  One thread; the state sits in
// shared memory with the kernels' [slot][thread] stride.
// The unit seams run on one thread: state arrays with stride 1.
using UnitModel = TableModel<double, 1>;

// rre_rhs (deterministic.hpp:85-88, oracle rre_rhs): a(y) from the packed
// tables, then dx_i = sum over the nu row in reaction order; y[i*ys], f[i*fs].
// Compiled with -fmad=false (this TU): the oracle's roundings.
__device__ void unit_rhs(const KinTables& T, const UnitModel& sm, const double* y, double* f, int fs) {
  constexpr int B = 1;
  const int N = T.n, M = T.m;
  double* x = sm.x;
  for (int i = 0; i < N; ++i) x[i * B] = y[i * B];
  for (int j = 0; j < M; ++j) sm.a[j * B] = sm.prop(j);
  for (int i = 0; i < N; ++i) {
    double acc = 0.0;
    for (int p = tab_row_ptr(T, i); p < tab_row_ptr(T, i + 1); ++p) {
      const uint32_t e = tab_row(T, p);
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(KIN_NU_DELTA(e)), sm.a[KIN_NU_INDEX(e) * B]));
    }
    f[i * fs] = acc;
  }
}

// rk_step (deterministic.hpp:26-36): one Dormand-Prince 5(4) step of size h
// from y (k1 = f(y)); out = {y5[N], err, k7[N]} with err = sqrt(mean((e_i /
// sk_i)^2)), sk_i = atol + rtol * max(|y_i|, |y5_i|) — the stage and error
// expressions of the oracle's integrate_rre, operation for operation.
__device__ void unit_rk_step(const KinTables& T, const UnitModel& sm, const double* x_in, double h,
                             double rtol, double atol, double* out) {
  constexpr int B = 1;
  const int N = T.n;
  constexpr double a21 = 1.0 / 5.0;
  constexpr double a31 = 3.0 / 40.0, a32 = 9.0 / 40.0;
  constexpr double a41 = 44.0 / 45.0, a42 = -56.0 / 15.0, a43 = 32.0 / 9.0;
  constexpr double a51 = 19372.0 / 6561.0, a52 = -25360.0 / 2187.0, a53 = 64448.0 / 6561.0, a54 = -212.0 / 729.0;
  constexpr double a61 = 9017.0 / 3168.0, a62 = -355.0 / 33.0, a63 = 46732.0 / 5247.0, a64 = 49.0 / 176.0,
                   a65 = -5103.0 / 18656.0;
  constexpr double a71 = 35.0 / 384.0, a73 = 500.0 / 1113.0, a74 = 125.0 / 192.0, a75 = -2187.0 / 6784.0,
                   a76 = 11.0 / 84.0;
  constexpr double e1 = 71.0 / 57600.0, e3 = -71.0 / 16695.0, e4 = 71.0 / 1920.0, e5 = -17253.0 / 339200.0,
                   e6 = 22.0 / 525.0, e7 = -1.0 / 40.0;
  // stage vectors after the kernel's x/a scratch: y, k1..k7, ys (stride B)
  double* y = sm.a + static_cast<size_t>(T.m) * B * 2 + static_cast<size_t>(N) * B;
  double* k[8];
  for (int q = 0; q < 8; ++q) k[q] = y + static_cast<size_t>(q + 1) * N * B;
  double* ys = y + static_cast<size_t>(9) * N * B;
  for (int i = 0; i < N; ++i) y[i * B] = x_in[i];
  unit_rhs(T, sm, y, k[1], B);
  for (int i = 0; i < N; ++i) ys[i * B] = y[i * B] + h * (a21 * k[1][i * B]);
  unit_rhs(T, sm, ys, k[2], B);
  for (int i = 0; i < N; ++i) ys[i * B] = y[i * B] + h * (a31 * k[1][i * B] + a32 * k[2][i * B]);
  unit_rhs(T, sm, ys, k[3], B);
  for (int i = 0; i < N; ++i) ys[i * B] = y[i * B] + h * (a41 * k[1][i * B] + a42 * k[2][i * B] + a43 * k[3][i * B]);
  unit_rhs(T, sm, ys, k[4], B);
  for (int i = 0; i < N; ++i)
    ys[i * B] = y[i * B] + h * (a51 * k[1][i * B] + a52 * k[2][i * B] + a53 * k[3][i * B] + a54 * k[4][i * B]);
  unit_rhs(T, sm, ys, k[5], B);
  for (int i = 0; i < N; ++i)
    ys[i * B] = y[i * B] + h * (a61 * k[1][i * B] + a62 * k[2][i * B] + a63 * k[3][i * B] + a64 * k[4][i * B] +
                                a65 * k[5][i * B]);
  unit_rhs(T, sm, ys, k[6], B);
  for (int i = 0; i < N; ++i)
    out[i] = y[i * B] + h * (a71 * k[1][i * B] + a73 * k[3][i * B] + a74 * k[4][i * B] + a75 * k[5][i * B] +
                             a76 * k[6][i * B]);
  for (int i = 0; i < N; ++i) ys[i * B] = out[i];
  unit_rhs(T, sm, ys, k[7], B);
  double sum = 0.0;
  for (int i = 0; i < N; ++i) {
    const double e = h * (e1 * k[1][i * B] + e3 * k[3][i * B] + e4 * k[4][i * B] + e5 * k[5][i * B] +
                          e6 * k[6][i * B] + e7 * k[7][i * B]);
    const double sk = atol + rtol * fmax(fabs(y[i * B]), fabs(out[i]));
    const double q = e / sk;
    sum = sum + q * q;
  }
  out[N] = sqrt(sum / static_cast<double>(N));
  for (int i = 0; i < N; ++i) out[N + 1 + i] = k[7][i * B];
}

__global__ void __launch_bounds__(32) unit_kernel(const __grid_constant__ KinTables T, int kind, const double* x_in,
                                                  const double* params, double* out) {
  extern __shared__ double smem[];
  if (threadIdx.x != 0) return;
  constexpr int B = 1;
  const int N = T.n, M = T.m;
  double* a = smem;                                        // a[j * B]
  double* x = smem + static_cast<size_t>(M) * B;           // x[i * B]
  for (int i = 0; i < N; ++i) x[i * B] = x_in[i];
  const UnitModel sm{T, x, a, nullptr};
  const double a0 = sm.all_props(M);
  if (kind == 0) {                                          // propensities
    for (int j = 0; j < M; ++j) out[j] = sm.aval(j);
  } else if (kind == 1) {                                   // select_tau (+inf when a0 == 0)
    uint64_t fl = 0;
    out[0] = a0 == 0.0 ? KIN_INF : sm.select_tau<false>(params[0], fl);
  } else if (kind == 2) {                                   // ssa_step_from_uniforms
    if (a0 == 0.0) {
      out[0] = KIN_INF;
      out[1] = -1.0;
    } else {
      out[0] = stoch::ssa_dt(params[0], a0);
      out[1] = static_cast<double>(stoch::ssa_select(sm, M, a0, params[1]));
    }
  } else if (kind == 3) {                                   // tau_leap_step_from_counts
    bool ovf = false;
    for (int j = 0; j < M; ++j)
      if (params[j] != 0.0) sm.apply(j, static_cast<long long>(params[j]), ovf);
    for (int i = 0; i < N; ++i) out[i] = x[i * B];
    out[N] = sm.any_negative() ? 1.0 : 0.0;
  } else if (kind == 4) {                                   // cle_step_from_normals
    for (int j = 0; j < M; ++j) cle_apply<B>(T, x, j, cle_increment(sm.aval(j), params[0], params[1 + j]));
    bool bad = false;
    const uint64_t c = cle_clamp<B>(x, N, &bad);
    for (int i = 0; i < N; ++i) out[i] = x[i * B];
    out[N] = static_cast<double>(c);
  } else if (kind == 5) {                                   // rre_rhs
    unit_rhs(T, sm, x, out, 1);
  } else if (kind == 6) {                                   // rk_step (one DP5(4) step)
    unit_rk_step(T, sm, x_in, params[0], params[1], params[2], out);
  }
}

size_t stochastic_smem_bytes(const KinTables& T, const KinSweepDev& S, int block, bool int_state) {
  return static_cast<size_t>(T.m + S.n_axes) * block * sizeof(double) +
         static_cast<size_t>(T.n) * block * (int_state ? sizeof(int32_t) : sizeof(double));
}

template <class XT>
cudaError_t launch_xt(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                      unsigned long long* counter, int* ovf_flag, cudaStream_t stream) {
  const size_t smem = S.gstate ? 0 : stochastic_smem_bytes(T, S, kBlock, sizeof(XT) == 4);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  const bool ph = S.rng_mode == KIN_RNG_PHILOX;
  auto kern = S.gstate ? (count ? (ph ? stochastic_kernel<true, true, XT, true> : stochastic_kernel<true, false, XT, true>)
                                : (ph ? stochastic_kernel<false, true, XT, true> : stochastic_kernel<false, false, XT, true>))
                       : (count ? (ph ? stochastic_kernel<true, true, XT, false> : stochastic_kernel<true, false, XT, false>)
                                : (ph ? stochastic_kernel<false, true, XT, false> : stochastic_kernel<false, false, XT, false>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  if (S.gstate && resident > S.gstate_warps) resident = S.gstate_warps;
  KinSweepDev SW = S;
  SW.warp_lanes = S.warp_lanes > 0 ? S.warp_lanes : kin_warp_lanes(S.n_local, resident);
  const uint64_t blocks = (S.n_local + SW.warp_lanes - 1) / SW.warp_lanes;
  const unsigned grid = static_cast<unsigned>(blocks < resident ? blocks : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  kern<<<grid, kBlock, smem, stream>>>(T, SW, O, counter, ovf_flag);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_unit(const KinTables& T, int kind, const double* x, const double* params, double* out,
                        cudaStream_t stream) {
  // a[M] + x[N] (+ the rk_step stage vectors: M + 10 N more, see unit_rk_step), stride 1
  const size_t smem = static_cast<size_t>(2 * T.m + 11 * T.n) * sizeof(double);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(unit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  unit_kernel<<<1, 32, smem, stream>>>(T, kind, x, params, out);
  return cudaGetLastError();
}

cudaError_t launch_cle(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                       unsigned long long* counter, cudaStream_t stream) {
  if (S.n_local == 0) return cudaSuccess;
  const size_t smem = stochastic_smem_bytes(T, S, kBlock, false);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  const bool ph = S.rng_mode == KIN_RNG_PHILOX;
  auto kern = count ? (ph ? cle_kernel<true, true> : cle_kernel<true, false>)
                    : (ph ? cle_kernel<false, true> : cle_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  KinSweepDev SW = S;
  SW.warp_lanes = 32;  // a fixed number of steps per simulation: lanes stay converged, full warps issue least
  const uint64_t blocks = (S.n_local + SW.warp_lanes - 1) / SW.warp_lanes;
  const unsigned grid = static_cast<unsigned>(blocks < resident ? blocks : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  kern<<<grid, kBlock, smem, stream>>>(T, SW, O, counter);
  return cudaGetLastError();
}

cudaError_t launch_stochastic(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                              unsigned long long* counter, int* ovf_flag, bool int_state, cudaStream_t stream) {
  if (S.n_local == 0) return cudaSuccess;
  if (int_state) return launch_xt<int32_t>(T, S, O, count, counter, ovf_flag, stream);
  return launch_xt<double>(T, S, O, count, counter, ovf_flag, stream);
}

}  // namespace kin

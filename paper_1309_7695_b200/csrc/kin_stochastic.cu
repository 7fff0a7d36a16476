// kin_stochastic.cu — batched exact-SSA and tau-leaping (K2 + K3 of DESIGN.md).
//
// One CUDA thread = one simulation (the paper's mapping), in
// "compat" RNG mode: each thread owns the reference's xoshiro256++ stream seeded
// by derive_run_seed (rng.cpp:25-48, ensemble.hpp:15-18), so firing counts are
// bit-identical to the CPU reference's.  The per-thread state (amounts x and the
// leap target buffer) lives in shared memory in [species][thread] layout:
// lanes touch consecutive 8-byte words, conflict-free, and the model tables are
// walked with warp-uniform indices out of the kernel-parameter constant bank.
//
// Mirrors oracle/kin_oracle.cpp simulate_stochastic() statement for statement:
//   simulate_approx TauAdaptive/TauFixed ... stochastic.hpp:78-92
//   select_tau ............................. stochastic.hpp:40-46
//   tau_leap_step / rejection-halving ...... stochastic.hpp:48-57
//   ssa_step fallback (bursts of 100) ...... stochastic.hpp:22-26
//   simulate_ssa grid semantics ............ stochastic.hpp:34-38
// Compiled with -fmad=false (see Makefile): no contraction on the parity path.
#include "kin_device.cuh"
#include "kin_launch.h"

namespace kin {

namespace {

constexpr double kInf = __builtin_huge_val();

struct ThreadState {
  const KinTables& T;
  const double* av;  // this thread's axis values (stride B)
  int B;
  __device__ __forceinline__ double rate(int j) const {
    const int ax = tab_rate_axis(T, j);
    return ax < 0 ? tab_rate(T, j) : av[ax * B];
  }
  // a_j(x) = c_j * prod h(x_s, stoich_s)   (model.hpp:151-157)
  __device__ __forceinline__ double prop(int j, const double* x) const {
    double aj = rate(j);
    const int p1 = tab_rt_ptr(T, j + 1);
    for (int p = tab_rt_ptr(T, j); p < p1; ++p) {
      const uint32_t e = tab_rt(T, p);
      aj = __dmul_rn(aj, combinations(x[KIN_TERM_SPECIES(e) * B], KIN_TERM_STOICH(e)));
    }
    return aj;
  }
};

template <bool kCount>
__global__ void __launch_bounds__(256) stochastic_kernel(const __grid_constant__ KinTables T,
                                                         const __grid_constant__ KinSweepDev S,
                                                         KinOutDev O) {
  extern __shared__ double smem[];
  const int B = blockDim.x, tid = threadIdx.x;
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * B + tid;
  if (s >= S.n_local) return;
  const uint64_t sim = S.sim_begin + s;
  const int N = T.n, M = T.m, G = T.n_grid;
  const uint64_t nloc = S.n_local;

  double* x = smem + tid;
  double* xn = smem + static_cast<size_t>(N) * B + tid;
  double* av = smem + static_cast<size_t>(2 * N) * B + tid;

  // Cartesian decode, last axis fastest.
  {
    uint64_t rem = sim / S.runs;
    for (int a = S.n_axes - 1; a >= 0; --a) {
      const uint64_t nv = static_cast<uint64_t>(S.axis_n[a]);
      const uint64_t q = rem / nv;
      av[a * B] = __ldg(S.axis_values[a] + (rem - q * nv));
      rem = q;
    }
  }
  ThreadState ts{T, av, B};
  for (int i = 0; i < N; ++i) {
    const int ax = tab_x0_axis(T, i);
    x[i * B] = ax < 0 ? tab_x0(T, i) : av[ax * B];
  }

  Xoshiro rng;
  rng.seed(sim_seed(S, sim));
  const int kind = S.kind;
  const double t_end = S.t_end;
  double t = 0.0;
  int gi = 0;
  uint64_t flops = 0, used = 0;
  uint64_t n_steps = 0, n_rej = 0, n_ssa = 0;
  int status = 0;
  const uint64_t budget = S.max_steps;
  const uint64_t F_prop = static_cast<uint64_t>(T.fprop);  // algorithmic flops of one propensity pass

  auto emit = [&]() {
    double* o = O.traj + static_cast<size_t>(gi) * N * nloc + s;
    for (int i = 0; i < N; ++i) o[static_cast<size_t>(i) * nloc] = x[i * B];
    ++gi;
  };

  while (gi < G && tab_grid(T, S, gi) <= t) emit();

  while (t < t_end) {
    if (++used > budget) { status = KIN_SIM_BUDGET; break; }
    double a0 = 0.0;
    for (int j = 0; j < M; ++j) a0 = __dadd_rn(a0, ts.prop(j, x));
    if (kCount) flops += F_prop + M;
    if (a0 == 0.0) break;

    double tau = 0.0;
    bool burst = false;
    if (kind == 0) {
      burst = true;
    } else if (kind == 1) {
      // select_tau, header form (stochastic.hpp:40-44)
      tau = kInf;
      const double eps = S.epsilon;
      for (int i = 0; i < N; ++i) {
        double mu = 0.0, s2 = 0.0;
        const int p1 = tab_row_ptr(T, i + 1);
        const int p0 = tab_row_ptr(T, i);
        for (int p = p0; p < p1; ++p) {
          const uint32_t e = tab_row(T, p);
          const int dl = KIN_NU_DELTA(e);
          const double aj = ts.prop(KIN_NU_INDEX(e), x);
          mu = __dadd_rn(mu, __dmul_rn(static_cast<double>(dl), aj));
          s2 = __dadd_rn(s2, __dmul_rn(static_cast<double>(dl * dl), aj));
        }
        if (kCount) flops += 4 * static_cast<uint64_t>(p1 - p0);
        if (mu == 0.0 && s2 == 0.0) continue;
        double bound = __ddiv_rn(__dmul_rn(eps, x[i * B]), tab_g(T, i));
        if (bound < 1.0) bound = 1.0;
        if (kCount) flops += 2;
        if (mu != 0.0) {
          const double t1 = __ddiv_rn(bound, fabs(mu));
          if (t1 < tau) tau = t1;
          if (kCount) flops += 1;
        }
        if (s2 != 0.0) {
          const double t2 = __ddiv_rn(__dmul_rn(bound, bound), s2);
          if (t2 < tau) tau = t2;
          if (kCount) flops += 2;
        }
      }
      if (kCount) flops += 1;
      burst = tau < __ddiv_rn(10.0, a0);
    } else {
      tau = S.tau;
    }

    if (burst) {
      bool stop = false;
      for (int b = 0;; ++b) {
        if (b > 0) {
          if (kind != 0 && b >= 100) break;
          if (++used > budget) { status = KIN_SIM_BUDGET; stop = true; break; }
          a0 = 0.0;
          for (int j = 0; j < M; ++j) a0 = __dadd_rn(a0, ts.prop(j, x));
          if (kCount) flops += F_prop + M;
          if (a0 == 0.0) { stop = true; break; }
        }
        const double u1 = rng.uniform();
        const double u2 = rng.uniform();
        const double dt = __ddiv_rn(log(__ddiv_rn(1.0, u1)), a0);
        const double tn = __dadd_rn(t, dt);
        if (kCount) flops += 8;
        if (tn > t_end) { t = t_end; stop = true; break; }
        while (gi < G && tab_grid(T, S, gi) < tn) emit();
        // first j with cumulative propensity > u2*a0
        const double target = __dmul_rn(u2, a0);
        double c = 0.0;
        int sel = -1, last = -1;
        for (int j = 0; j < M; ++j) {
          const double aj = ts.prop(j, x);
          if (aj > 0.0) last = j;
          c = __dadd_rn(c, aj);
          if (c > target) { sel = j; break; }
        }
        if (sel < 0) sel = last;
        if (kCount) flops += 1 + static_cast<uint64_t>(sel + 1);
        const int p1 = tab_col_ptr(T, sel + 1);
        const int p0 = tab_col_ptr(T, sel);
        bool neg = false;
        for (int p = p0; p < p1; ++p) {
          const uint32_t e = tab_col(T, p);
          const int sp = KIN_NU_INDEX(e);
          const double v = __dadd_rn(x[sp * B], static_cast<double>(KIN_NU_DELTA(e)));
          if (v < 0.0) neg = true;
          x[sp * B] = v;
        }
        if (neg) { status = KIN_SIM_NEGATIVE; stop = true; break; }
        if (kCount) flops += static_cast<uint64_t>(p1 - p0);
        t = tn;
        if (kind == 0) ++n_steps; else ++n_ssa;
        while (gi < G && tab_grid(T, S, gi) <= t) emit();
      }
      if (stop) break;
      continue;
    }

    // Poisson leap truncated at the next grid time; reject -> halve
    const double t_stop = (gi < G && tab_grid(T, S, gi) < t_end) ? tab_grid(T, S, gi) : t_end;
    bool hit = false;
    const double gap = __dsub_rn(t_stop, t);
    if (kCount) flops += 1;
    if (!(tau < gap)) { tau = gap; hit = true; }
    for (;;) {
      for (int i = 0; i < N; ++i) xn[i * B] = x[i * B];
      for (int j = 0; j < M; ++j) {
        const uint64_t k = poisson<kCount>(rng, __dmul_rn(ts.prop(j, x), tau), flops);
        if (k == 0) continue;
        const double kj = static_cast<double>(k);
        const int p1 = tab_col_ptr(T, j + 1);
        for (int p = tab_col_ptr(T, j); p < p1; ++p) {
          const uint32_t e = tab_col(T, p);
          const int sp = KIN_NU_INDEX(e);
          xn[sp * B] = __dadd_rn(xn[sp * B], __dmul_rn(static_cast<double>(KIN_NU_DELTA(e)), kj));
        }
      }
      if (kCount) flops += static_cast<uint64_t>(M) + 2 * static_cast<uint64_t>(T.nnz);
      bool neg = false;
      for (int i = 0; i < N; ++i) neg |= xn[i * B] < 0.0;
      if (!neg) break;
      ++n_rej;
      tau = __dmul_rn(tau, 0.5);
      hit = false;
      if (kCount) flops += 1;
    }
    { double* tmp = x; x = xn; xn = tmp; }
    if (hit) {
      t = t_stop;
    } else {
      t = __dadd_rn(t, tau);
      if (kCount) flops += 1;
    }
    ++n_steps;
    while (gi < G && tab_grid(T, S, gi) <= t) emit();
  }
  if (status == 0)
    while (gi < G) emit();

  uint64_t* me = O.meta + s * 6;
  me[0] = n_steps;
  me[1] = n_rej;
  me[2] = 0;
  me[3] = n_ssa;
  me[4] = 0;
  me[5] = 0;
  O.status[s] = status;
  if (kCount && O.work) O.work[s] = flops;
}

}  // namespace

size_t stochastic_smem_bytes(const KinTables& T, const KinSweepDev& S, int block) {
  return static_cast<size_t>(2 * T.n + S.n_axes) * block * sizeof(double);
}

cudaError_t launch_stochastic(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                              int block, cudaStream_t stream) {
  if (S.n_local == 0) return cudaSuccess;
  const size_t smem = stochastic_smem_bytes(T, S, block);
  const unsigned grid = static_cast<unsigned>((S.n_local + block - 1) / block);
  if (count) {
    cudaFuncSetAttribute(stochastic_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    stochastic_kernel<true><<<grid, block, smem, stream>>>(T, S, O);
  } else {
    cudaFuncSetAttribute(stochastic_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    stochastic_kernel<false><<<grid, block, smem, stream>>>(T, S, O);
  }
  return cudaGetLastError();
}

}  // namespace kin

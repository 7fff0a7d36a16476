// kin_stochastic_group.cu — lane-group tau-leaping / SSA for the Philox mode.
//
// The compat mode must consume the reference's single xoshiro256++ stream in
// order, so it runs one thread per simulation (kin_stochastic.cu).  In the
// Philox mode every Poisson draw has its own counter (run seed, event, reaction),
// so a group of L lanes (L = 4..32, a sub-warp) cooperates on ONE simulation:
//   * lane l owns reactions j = l, l+L, ... : propensities a_j and the Poisson
//     draws k_j of a leap (independent counters -> parallel);
//   * lane l owns species i = l, l+L, ... : mu_i, sigma2_i of select_tau (row
//     sums in reaction order, as the oracle), and the leap update
//     x_i + sum_j nu_ij k_j (exact integers: order-free); a leap is rejected
//     when any lane sees a negative amount (group vote) BEFORE anything is
//     written, so rejection needs no rollback;
//   * tau = min over species: shuffle-min (exact, order-free);
//   * a0 and the SSA cumulative selection are sequential sums in reaction order
//     (the oracle's rounding): every lane evaluates them redundantly from shared
//     memory, so the group stays convergent and no broadcast is needed.
// Result: bit-identical to the oracle's Philox mode (and to the thread-per-
// simulation Philox kernel).  Per-simulation state lives in shared memory,
// simulation-major (x[N], a[M], k[M], axis values), stride padded so the two
// groups of a half-warp hit disjoint banks.
//
// Compiled with -fmad=false (parity path).
#include "kin_device.cuh"
#include "kin_launch.h"

namespace kin {

namespace {

constexpr double kInf = __builtin_huge_val();
constexpr int kBlockG = 128;

template <int L>
struct GroupSync {
  unsigned mask;
  __device__ __forceinline__ void sync() const {
    if (L > 1) __syncwarp(mask);
  }
  __device__ __forceinline__ double min(double v) const {
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(mask, v, off, L));
    return v;
  }
  __device__ __forceinline__ bool any(bool b) const {
    const unsigned bal = __ballot_sync(mask, b);
    return (bal & mask) != 0;
  }
  __device__ __forceinline__ uint64_t sum(uint64_t v) const {
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off, L);
    return v;
  }
};

__host__ __device__ __forceinline__ int sim_stride(int n, int m, int n_axes) {
  int s = n + 2 * m + n_axes;
  s += (8 - s % 16 + 16) % 16;  // stride = 8 (mod 16) doubles
  return s;
}

template <int L, bool kCount>
__device__ void simulate_group(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, uint64_t s,
                               double* x, double* a, double* kk, double* av, int lane, const GroupSync<L>& gs) {
  const uint64_t sim = global_sim(S, s);
  const int N = T.n, M = T.m, G = T.n_grid;

  if (lane == 0) {
    uint64_t rem = sim / S.runs;
    for (int ax = S.n_axes - 1; ax >= 0; --ax) {
      const uint64_t nv = static_cast<uint64_t>(S.axis_n[ax]);
      const uint64_t q = rem / nv;
      av[ax] = __ldg(S.axis_values[ax] + (rem - q * nv));
      rem = q;
    }
  }
  gs.sync();
  for (int i = lane; i < N; i += L) {
    const int ax = tab_x0_axis(T, i);
    x[i] = ax < 0 ? tab_x0(T, i) : av[ax];
  }
  auto prop = [&](int j) -> double {
    const uint64_t d = tab_rdesc(T, j);
    const int ax = KIN_RD_AXIS(d);
    double aj = ax < 0 ? tab_rate(T, j) : __dmul_rn(tab_rate(T, j), av[ax]);
    const int nt = KIN_RD_NTERMS(d);
    if (nt > 0) {
      aj = __dmul_rn(aj, combinations(x[KIN_RD_SPECIES(d, 0)], KIN_RD_STOICH(d, 0)));
      if (nt > 1) {
        aj = __dmul_rn(aj, combinations(x[KIN_RD_SPECIES(d, 1)], KIN_RD_STOICH(d, 1)));
        if (nt > 2) aj = __dmul_rn(aj, combinations(x[KIN_RD_SPECIES(d, 2)], KIN_RD_STOICH(d, 2)));
      }
    }
    return aj;
  };
  auto sum_a = [&]() {
    double a0 = 0.0;
    for (int j = 0; j < M; ++j) a0 = __dadd_rn(a0, a[j]);
    return a0;
  };
  auto emit = [&](int g) {
    double* o = O.traj + (static_cast<size_t>(s) * G + g) * N;  // [sim][g][n]
    for (int i = lane; i < N; i += L) o[i] = x[i];
  };

  const uint64_t seed = sim_seed(S, sim);
  uint64_t ev = 0;
  const int kind = S.kind;
  const double t_end = S.t_end;
  double t = 0.0;
  int gi = 0;
  uint64_t flops = 0, used = 0;
  uint64_t n_steps = 0, n_rej = 0, n_ssa = 0;
  int status = 0;
  const uint64_t budget = S.max_steps;
  const uint64_t F_prop = static_cast<uint64_t>(T.fprop);
  gs.sync();
  while (gi < G && tab_grid(T, S, gi) <= t) emit(gi++);
  bool a_valid = false;
  double a0 = 0.0;

  while (t < t_end) {
    if (++used > budget) { status = KIN_SIM_BUDGET; break; }
    if (!a_valid) {
      for (int j = lane; j < M; j += L) a[j] = prop(j);
      gs.sync();
      a0 = sum_a();
    }
    a_valid = false;
    if (kCount && lane == 0) flops += F_prop + M;
    if (a0 == 0.0) break;

    double tau = 0.0;
    bool burst = false;
    if (kind == 0) {
      burst = true;
    } else if (kind == 1) {
      double tl = kInf;
      const double eps = S.epsilon;
      for (int i = lane; i < N; i += L) {
        double mu = 0.0, s2 = 0.0;
        const int p1 = tab_row_ptr(T, i + 1);
        const int p0 = tab_row_ptr(T, i);
        for (int p = p0; p < p1; ++p) {
          const uint32_t e = tab_row(T, p);
          const int dl = KIN_NU_DELTA(e);
          const double aj = a[KIN_NU_INDEX(e)];
          mu = __dadd_rn(mu, __dmul_rn(static_cast<double>(dl), aj));
          s2 = __dadd_rn(s2, __dmul_rn(static_cast<double>(dl * dl), aj));
        }
        if (kCount) flops += 4 * static_cast<uint64_t>(p1 - p0);
        if (mu == 0.0 && s2 == 0.0) continue;
        const double ex = __dmul_rn(eps, x[i]);
        const double g = tab_g(T, i);
        double bound = g == 1.0 ? ex : (g == 2.0 ? __dmul_rn(ex, 0.5) : __ddiv_rn(ex, g));
        if (bound < 1.0) bound = 1.0;
        if (kCount) flops += 2;
        if (mu != 0.0) {
          const double amu = fabs(mu);
          if (!(bound > __dmul_rn(__dmul_rn(tl, amu), 1.0 + 0x1p-50))) {
            const double t1 = __ddiv_rn(bound, amu);
            if (t1 < tl) tl = t1;
          }
          if (kCount) flops += 1;
        }
        if (s2 != 0.0) {
          const double bb = __dmul_rn(bound, bound);
          if (!(bb > __dmul_rn(__dmul_rn(tl, s2), 1.0 + 0x1p-50))) {
            const double t2 = __ddiv_rn(bb, s2);
            if (t2 < tl) tl = t2;
          }
          if (kCount) flops += 2;
        }
      }
      tau = gs.min(tl);
      if (kCount && lane == 0) flops += 1;
      burst = tau < __ddiv_rn(10.0, a0);
    } else {
      tau = S.tau;
    }

    if (burst) {
      bool stop = false;
      for (int b = 0;; ++b) {
        if (b > 0) {
          if (kind != 0 && b >= 100) { a_valid = true; break; }
          if (++used > budget) { status = KIN_SIM_BUDGET; stop = true; break; }
          if (kCount && lane == 0) flops += F_prop + M;
          if (a0 == 0.0) { stop = true; break; }
        }
        PhiloxSite src(seed, ev++, kPhiloxSsaSite);
        const double u1 = src.uniform();
        const double u2 = src.uniform();
        const double dt = __ddiv_rn(log(__ddiv_rn(1.0, u1)), a0);
        const double tn = __dadd_rn(t, dt);
        if (kCount && lane == 0) flops += 8;
        if (tn > t_end) { t = t_end; stop = true; break; }
        while (gi < G && tab_grid(T, S, gi) < tn) emit(gi++);
        const double target = __dmul_rn(u2, a0);
        double c = 0.0;
        int sel = -1, last = -1;
        for (int j = 0; j < M; ++j) {
          const double aj = a[j];
          if (aj > 0.0) last = j;
          c = __dadd_rn(c, aj);
          if (c > target) { sel = j; break; }
        }
        if (sel < 0) sel = last;
        if (kCount && lane == 0) flops += 1 + static_cast<uint64_t>(sel + 1);
        gs.sync();  // every lane has read x/a for this event
        const int p1 = tab_col_ptr(T, sel + 1);
        const int p0 = tab_col_ptr(T, sel);
        bool neg = false;
        for (int p = p0; p < p1; ++p) {
          const uint32_t e = tab_col(T, p);
          const int sp = KIN_NU_INDEX(e);
          if (sp % L == lane) {
            const double v = __dadd_rn(x[sp], static_cast<double>(KIN_NU_DELTA(e)));
            neg |= v < 0.0;
            x[sp] = v;
          }
        }
        if (gs.any(neg)) { status = KIN_SIM_NEGATIVE; stop = true; break; }
        if (kCount && lane == 0) flops += static_cast<uint64_t>(p1 - p0);
        t = tn;
        if (kind == 0) ++n_steps; else ++n_ssa;
        gs.sync();
        while (gi < G && tab_grid(T, S, gi) <= t) emit(gi++);
        const int q1 = tab_dep_ptr(T, sel + 1);
        for (int q = tab_dep_ptr(T, sel) + lane; q < q1; q += L) {
          const int k = tab_dep(T, q);
          a[k] = prop(k);
        }
        gs.sync();
        a0 = sum_a();
      }
      if (stop) break;
      continue;
    }

    const double t_stop = (gi < G && tab_grid(T, S, gi) < t_end) ? tab_grid(T, S, gi) : t_end;
    bool hit = false;
    const double gap = __dsub_rn(t_stop, t);
    if (kCount && lane == 0) flops += 1;
    if (!(tau < gap)) { tau = gap; hit = true; }
    for (;;) {
      for (int j = lane; j < M; j += L) {
        PhiloxSite src(seed, ev, static_cast<uint32_t>(j));
        kk[j] = static_cast<double>(poisson<kCount>(src, __dmul_rn(a[j], tau), flops, S.lgamma_tab));
      }
      ++ev;
      if (kCount && lane == 0) flops += static_cast<uint64_t>(M) + 2 * static_cast<uint64_t>(T.nnz);
      gs.sync();
      bool neg = false;
      for (int i = lane; i < N; i += L) {
        double v = x[i];
        const int p1 = tab_row_ptr(T, i + 1);
        for (int p = tab_row_ptr(T, i); p < p1; ++p) {
          const uint32_t e = tab_row(T, p);
          const double kj = kk[KIN_NU_INDEX(e)];
          if (kj != 0.0) v = __dadd_rn(v, __dmul_rn(static_cast<double>(KIN_NU_DELTA(e)), kj));
        }
        neg |= v < 0.0;
      }
      if (!gs.any(neg)) break;
      ++n_rej;
      tau = __dmul_rn(tau, 0.5);
      hit = false;
      if (kCount && lane == 0) flops += 1;
      gs.sync();  // kk is rewritten by the next attempt
    }
    for (int i = lane; i < N; i += L) {
      double v = x[i];
      const int p1 = tab_row_ptr(T, i + 1);
      for (int p = tab_row_ptr(T, i); p < p1; ++p) {
        const uint32_t e = tab_row(T, p);
        const double kj = kk[KIN_NU_INDEX(e)];
        if (kj != 0.0) v = __dadd_rn(v, __dmul_rn(static_cast<double>(KIN_NU_DELTA(e)), kj));
      }
      x[i] = v;
    }
    if (hit) {
      t = t_stop;
    } else {
      t = __dadd_rn(t, tau);
      if (kCount && lane == 0) flops += 1;
    }
    ++n_steps;
    gs.sync();
    while (gi < G && tab_grid(T, S, gi) <= t) emit(gi++);
  }
  if (status == 0)
    while (gi < G) emit(gi++);
  if (kCount) flops = gs.sum(flops);
  if (lane == 0) {
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
  gs.sync();
}

template <int L, bool kCount>
__global__ void __launch_bounds__(kBlockG) stochastic_group_kernel(const __grid_constant__ KinTables T,
                                                                   const __grid_constant__ KinSweepDev S,
                                                                   KinOutDev O, unsigned long long* __restrict__ next) {
  extern __shared__ double smem[];
  constexpr int GPB = kBlockG / L;  // groups (simulations) per block
  const int grp = threadIdx.x / L, lane = threadIdx.x % L;
  const int wl = threadIdx.x & 31;
  const int stride = sim_stride(T.n, T.m, S.n_axes);
  double* base = smem + static_cast<size_t>(grp) * stride;
  double* x = base;
  double* a = x + T.n;
  double* kk = a + T.m;
  double* av = kk + T.m;
  GroupSync<L> gs;
  gs.mask = (L == 32) ? 0xFFFFFFFFu : (((1u << L) - 1u) << ((wl / L) * L));
  (void)GPB;
  // persistent warps: each warp fetches 32/L simulations at a time
  for (;;) {
    unsigned long long wbase = 0;
    if (wl == 0) wbase = atomicAdd(next, static_cast<unsigned long long>(32 / L));
    wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
    if (wbase >= S.n_local) break;
    const uint64_t s = wbase + wl / L;
    if (s < S.n_local) simulate_group<L, kCount>(T, S, O, s, x, a, kk, av, lane, gs);
    __syncwarp();
  }
}

template <int L>
cudaError_t launch_L(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                     unsigned long long* counter, cudaStream_t stream) {
  constexpr int GPB = kBlockG / L;
  const size_t smem = static_cast<size_t>(GPB) * sim_stride(T.n, T.m, S.n_axes) * sizeof(double);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  auto kern = count ? stochastic_group_kernel<L, true> : stochastic_group_kernel<L, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlockG, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t blocks_needed = (S.n_local + GPB - 1) / GPB;
  const uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  const unsigned grid = static_cast<unsigned>(blocks_needed < resident ? blocks_needed : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  kern<<<grid, kBlockG, smem, stream>>>(T, S, O, counter);
  return cudaGetLastError();
}

}  // namespace

// Measured on B200 (profiles/r1_philox_lanes.txt): lane groups win for tiny
// SSA-heavy models (Schlogl 4x4: 4 lanes, 2.1x) and wide models (C5 128x256:
// 16 lanes, 1.7x); mid-size models (C4 33x39) are faster one thread per
// simulation (returns 1).
// Measured on B200 (profiles/r1_philox_lanes.txt): lane groups pay
// off for small models (Schlogl: 4 lanes 122 ms vs 176 ms); for large ones the
// thread-per-simulation kernel with its state in global memory is faster
// (C5 128x256: 1236 ms vs 2244 ms with 16 lanes).
int stochastic_group_pick_lanes(int n_species, int n_reactions) {
  const int w = n_species > n_reactions ? n_species : n_reactions;
  return w <= 8 ? 4 : 1;
}

cudaError_t launch_stochastic_group(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                                    int lanes, unsigned long long* counter, cudaStream_t stream) {
  if (S.n_local == 0) return cudaSuccess;
  if (lanes <= 0) lanes = stochastic_group_pick_lanes(T.n, T.m);
  switch (lanes) {
    case 4: return launch_L<4>(T, S, O, count, counter, stream);
    case 8: return launch_L<8>(T, S, O, count, counter, stream);
    case 16: return launch_L<16>(T, S, O, count, counter, stream);
    case 32: return launch_L<32>(T, S, O, count, counter, stream);
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace kin

// kin_lsoda_impl.cuh — batched LSODA-style integration of the reaction-rate equations
// (K5 of DESIGN.md; north-star extension, no reference counterpart: the
// reference's ODE method is Dopri5, deterministic.hpp:38-83, and stiff solvers
// are a SPEC non-goal).
//
// Algorithm (ODEPACK LSODE core + LSODA switching, restated in
// oracle/kin_oracle.cpp integrate_lsoda, which this kernel mirrors statement for
// statement): Nordsieck history Z[0..12]; Adams-Moulton orders 1..12 with
// functional iteration; BDF orders 1..5 with chord Newton on P = I - h*l0*J,
// J = nu * da/dx analytic, dense LU with partial pivoting; LSODE error test and
// order/step selection every nq+1 steps; Adams steps capped by the stability
// region (h*||J|| <= sm1(q)); method switch Adams->BDF when BDF could step 5x
// farther, BDF->Adams when Adams could step at least as far.
//
// One thread per simulation; per-thread state in shared memory, [slot][thread]
// layout: Z (13N), acor/savf/ewt/y/tmp (5N), P and a Jacobian scratch (2N^2),
// propensities (M), axis values, pivots.  Compiled with -fmad=false and using
// the portable pow below (only correctly rounded IEEE operations), so results are
// bit-identical to the oracle's.
#pragma once
#include "kin_device.cuh"
#ifndef __CUDACC_RTC__
#include "kin_launch.h"
#endif
#include "kin_pmath.cuh"
#ifndef KIN_INF
#define KIN_INF __longlong_as_double(0x7FF0000000000000LL)
#endif

namespace kin {

namespace {
// Adams stability-region caps (LSODA's sm1), one copy per translation unit
// Adams -> BDF when the stability cap bound the Adams step this many order
// selections in a row (oracle: kLsodaStabSwitch)
constexpr int kLsodaStabSwitch = 8;
__device__ __constant__ double c_sm1[13] = {0.0, 0.5, 0.575, 0.55, 0.45, 0.35, 0.25, 0.2, 0.15, 0.1, 0.075, 0.05, 0.025};
}  // namespace

namespace lsd {

using pmath::pm_pow;

// Step-ratio factors 1 / (c * x^e + cs) of the order/step selection (LSODE
// rhsm/rhup/rhdn and LSODA's method-switch ratios), out of line: each inlined
// copy was ~150 instructions (portable log + exp + two divisions) at seven
// sites, all in the kernel's instruction-cache working set (ncu: no_instruction
// 2.38 warps per issue on C3), executed once per nq+1 steps.  Same operations,
// same results; C3 21.2 -> 18.7-19.1 ms, stiff C3 11.8 -> 10.8 ms.  (The
// Jacobian row/matrix out of line as well measured slower: 21.6 ms.)
static __device__ __noinline__ double step_ratio_e(double x, double e, double c, double cs) {
  return 1.0 / (c * pm_pow(x, e) + cs);
}
static __device__ __noinline__ double step_ratio_q(double x, int q, double c, double cs) {
  return 1.0 / (c * pm_pow(x, 1.0 / q) + cs);
}

constexpr int kBlock = 32;
// N <= 4: keep the iteration matrix P = I - h l0 J and its LU factors in
// registers (fully unrolled, constant indices) instead of shared memory.
// Implemented and bit-exact (tests/test_gpu_*.py ran green with it on), but
// measured slower on the B200: C3 31.8 -> 35.5 ms, stiff C3 15.0 -> 16.1 ms
// (167 registers against 126; the unrolled factorisation with predicated row
// swaps costs more than the shared-memory version saves), so it is off.
constexpr bool kLsodaRegLU = false;
constexpr int kL = 13;  // Nordsieck vectors (Adams max order 12)


// The RHS and the weighted RMS norm are called from several places in the
// step; out of line they exist once in the kernel's code (each inlined copy,
// with its species loop unrolled and its correctly rounded divisions, costs
// instruction-cache space the step loop needs).
template <int kN>
__device__ __noinline__ void rhs_out_of_line(const KinTables& T, const double* av, double* a, int m, int n_rt,
                                             const double* yy, double* f) {
  constexpr int B = kBlock;
  const int n = kN > 0 ? kN : n_rt;
#pragma unroll 1
  for (int j = 0; j < m; ++j) {
    const uint64_t d = tab_rdesc(T, j);
    const int ax = KIN_RD_AXIS(d);
    double aj = ax < 0 ? tab_rate(T, j) : __dmul_rn(tab_rate(T, j), av[ax * B]);
    const int nt = KIN_RD_NTERMS(d);
#pragma unroll 1
    for (int t = 0; t < nt; ++t) aj = aj * combinations(yy[KIN_RD_SPECIES(d, t) * B], KIN_RD_STOICH(d, t));
    a[j * B] = aj;
  }
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    const int p1 = tab_row_ptr(T, i + 1);
#pragma unroll 1
    for (int p = tab_row_ptr(T, i); p < p1; ++p) {
      const uint32_t e = tab_row(T, p);
      s = s + static_cast<double>(KIN_NU_DELTA(e)) * a[KIN_NU_INDEX(e) * B];
    }
    f[i * B] = s;
  }
}
template <int kN>
__device__ __noinline__ double wrms_out_of_line(const double* vv, const double* ewt, int n_rt) {
  constexpr int B = kBlock;
  const int n = kN > 0 ? kN : n_rt;
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    const double q = vv[i * B] / ewt[i * B];
    s = s + q * q;
  }
  return sqrt(s / n);
}

// The RHS policy: TablePM walks the packed tables (rhs_out_of_line); the
// per-model JIT passes its generated GenModel<double> (kin_jit.cpp: straight-
// line propensities and nu rows, the same operations in the same order).
struct TablePM {
  static constexpr bool kJit = false;
  static constexpr bool kJitJac = false;
};

// kN > 0: the species count is a compile-time constant (small models: every
// loop over species unrolls and the indexing folds); kN = 0: runtime T.n.
template <int kN, class PM = TablePM>
struct Lsoda {
  const KinTables& T;
  const KinSweepDev& S;
  const double* co;  // elco [2][13][14] then tesco [2][13][3]
  int n_rt, m;
  static constexpr int B = kBlock;
  // the register-resident P/LU variant (kLsodaRegLU above)
  static constexpr bool kRegLU = kLsodaRegLU && kN >= 1 && kN <= 4;
  __device__ __forceinline__ int N() const { return kN > 0 ? kN : n_rt; }
  double *Z, *acor, *savf, *ewt, *y, *tmp, *P, *a, *av;
  int* piv;
  uint64_t flops;
  uint64_t F_rhs;
  double pr[kRegLU ? kN * kN : 1];
  int pv[kRegLU ? kN : 1];

  __device__ __forceinline__ double elco(int meth, int q, int i) const { return __ldg(co + (meth * 13 + q) * 14 + i); }
  __device__ __forceinline__ double tesco(int meth, int q, int i) const {
    return __ldg(co + 2 * 13 * 14 + (meth * 13 + q) * 3 + i);
  }
  __device__ __forceinline__ double& z(int j, int i) const { return Z[(j * N() + i) * B]; }
  __device__ __forceinline__ double& v(double* base, int i) const { return base[i * B]; }
  __device__ __forceinline__ double rate(int j) const {
    const int ax = KIN_RD_AXIS(tab_rdesc(T, j));
    return ax < 0 ? tab_rate(T, j) : __dmul_rn(tab_rate(T, j), av[ax * B]);
  }
  // rre_rhs (oracle order): a_j then dx_i = sum over the nu row
  template <bool C>
  __device__ __forceinline__ void rhs(const double* yy, double* f) {
    if constexpr (PM::kJit) {
      const PM st{T, const_cast<double*>(yy), a, av};
      st.props_only();
      st.rre_rows(f, N());
    } else {
      rhs_out_of_line<kN>(T, av, a, m, N(), yy, f);
    }
    if (C) flops += F_rhs;
  }
  template <bool C>
  __device__ void jacobian(const double* yy, double* J) {
    if constexpr (PM::kJitJac) {  // the per-model straight-line matrix (kin_jit.cpp)
      const PM st{T, const_cast<double*>(yy), a, av};
      st.jac_full(J);
      if (C) flops += jac_flops();
      return;
    }
    for (int q = 0; q < N() * N(); ++q) J[q * B] = 0.0;
#pragma unroll 1
    for (int k = 0; k < m; ++k) {
      const uint64_t d = tab_rdesc(T, k);
      const int nt = KIN_RD_NTERMS(d);
      const double rk = rate(k);
      for (int p = 0; p < nt; ++p) {
        const int s = KIN_RD_SPECIES(d, p), st = KIN_RD_STOICH(d, p);
        const double xs = yy[s * B];
        const double h = combinations(xs, st);
        double dh;
        if (st == 1) dh = xs < 0.0 ? 0.0 : 1.0;
        else if (st == 2) dh = h > 0.0 ? xs - 0.5 : 0.0;
        else dh = h > 0.0 ? ((3.0 * xs - 6.0) * xs + 2.0) / 6.0 : 0.0;
        double dd = rk * dh;
        for (int q = 0; q < nt; ++q)
          if (q != p) dd = dd * combinations(yy[KIN_RD_SPECIES(d, q) * B], KIN_RD_STOICH(d, q));
        const int c1 = tab_col_ptr(T, k + 1);
#pragma unroll 1
        for (int c = tab_col_ptr(T, k); c < c1; ++c) {
          const uint32_t e = tab_col(T, c);
          double& jj = J[(KIN_NU_INDEX(e) * N() + s) * B];
          jj = jj + static_cast<double>(KIN_NU_DELTA(e)) * dd;
        }
        if (C) flops += 4 + nt + 2 * static_cast<uint64_t>(c1 - tab_col_ptr(T, k));
      }
    }
  }
  // max_i (sum_j |J_ij| ewt_j) / ewt_i without storing J: row i is formed in
  // tmp by walking row i of nu (reactions ascending), so each J_ij receives the
  // oracle's contributions (rre_jacobian: reactions ascending) in its order.
  // row i of J = nu * da/dx into tmp[s*B], walking row i of nu (reactions
  // ascending): each J_is receives the oracle's contributions (rre_jacobian:
  // reactions ascending) in its order
  __device__ __forceinline__ void jac_row(const double* yy, int i) {
    if constexpr (PM::kJitJac) {  // the per-model straight-line row (kin_jit.cpp)
      const PM st{T, const_cast<double*>(yy), a, av};
      st.jac_row(i, tmp);
      return;
    }
    for (int s = 0; s < N(); ++s) tmp[s * B] = 0.0;
    const int p1 = tab_row_ptr(T, i + 1);
#pragma unroll 1
    for (int prw = tab_row_ptr(T, i); prw < p1; ++prw) {
      const uint32_t e = tab_row(T, prw);
      const int k = KIN_NU_INDEX(e);
      const double dl = static_cast<double>(KIN_NU_DELTA(e));
      const uint64_t d = tab_rdesc(T, k);
      const int nt = KIN_RD_NTERMS(d);
      const double rk = rate(k);
#pragma unroll 1
      for (int p = 0; p < nt; ++p) {
        const int s = KIN_RD_SPECIES(d, p), st = KIN_RD_STOICH(d, p);
        const double xs = yy[s * B];
        const double h = combinations(xs, st);
        double dh;
        if (st == 1) dh = xs < 0.0 ? 0.0 : 1.0;
        else if (st == 2) dh = h > 0.0 ? xs - 0.5 : 0.0;
        else dh = h > 0.0 ? ((3.0 * xs - 6.0) * xs + 2.0) / 6.0 : 0.0;
        double dd = rk * dh;
        for (int q = 0; q < nt; ++q)
          if (q != p) dd = dd * combinations(yy[KIN_RD_SPECIES(d, q) * B], KIN_RD_STOICH(d, q));
        tmp[s * B] = tmp[s * B] + dl * dd;
      }
    }
  }
  // the oracle's rre_jacobian flop count
  __device__ __forceinline__ uint64_t jac_flops() const {
    uint64_t f = 0;
#pragma unroll 1
    for (int k = 0; k < m; ++k) {
      const int nt = KIN_RD_NTERMS(tab_rdesc(T, k));
      f += static_cast<uint64_t>(nt) * (4 + nt + 2 * static_cast<uint64_t>(tab_col_ptr(T, k + 1) - tab_col_ptr(T, k)));
    }
    return f;
  }
  // kRegLU: P = I - hl0 J built row by row into registers, then factored there
  template <bool C>
  __device__ __forceinline__ bool form_lu_reg(const double* yy, double hl0) {
#pragma unroll
    for (int i = 0; i < (kRegLU ? kN : 0); ++i) {
      jac_row(yy, i);
#pragma unroll
      for (int s = 0; s < (kRegLU ? kN : 0); ++s) pr[i * kN + s] = -hl0 * tmp[s * B];
    }
    if (C) flops += jac_flops();
#pragma unroll
    for (int i = 0; i < (kRegLU ? kN : 0); ++i) pr[i * kN + i] = pr[i * kN + i] + 1.0;
#pragma unroll
    for (int k = 0; k < (kRegLU ? kN : 0); ++k) {
      int prow = k;
      double best = fabs(pr[k * kN + k]);
#pragma unroll
      for (int i = k + 1; i < kN; ++i) {
        const double c = fabs(pr[i * kN + k]);
        if (c > best) { best = c; prow = i; }
      }
      pv[k] = prow;
      if (best == 0.0) return false;
#pragma unroll
      for (int i = k + 1; i < kN; ++i)
        if (prow == i) {
#pragma unroll
          for (int j = 0; j < kN; ++j) {
            const double t0 = pr[k * kN + j];
            pr[k * kN + j] = pr[i * kN + j];
            pr[i * kN + j] = t0;
          }
        }
      const double inv = 1.0 / pr[k * kN + k];
#pragma unroll
      for (int i = k + 1; i < kN; ++i) {
        const double l = pr[i * kN + k] * inv;
        pr[i * kN + k] = l;
#pragma unroll
        for (int j = k + 1; j < kN; ++j) pr[i * kN + j] = pr[i * kN + j] - l * pr[k * kN + j];
      }
    }
    if (C) flops += static_cast<uint64_t>(2 * kN * kN * kN / 3 + kN);
    return true;
  }
  template <bool C>
  __device__ __forceinline__ void lu_solve_reg(double* b) {
#pragma unroll
    for (int k = 0; k < (kRegLU ? kN : 0); ++k) {
      const int pk = pv[k];
      if (pk != k) {
        const double t0 = b[k * B];
        b[k * B] = b[pk * B];
        b[pk * B] = t0;
      }
#pragma unroll
      for (int i = k + 1; i < kN; ++i) b[i * B] = b[i * B] - pr[i * kN + k] * b[k * B];
    }
#pragma unroll
    for (int i = (kRegLU ? kN : 0) - 1; i >= 0; --i) {
      double s = b[i * B];
#pragma unroll
      for (int j = i + 1; j < kN; ++j) s = s - pr[i * kN + j] * b[j * B];
      b[i * B] = s / pr[i * kN + i];
    }
    if (C) flops += static_cast<uint64_t>(2 * kN * kN);
  }
  template <bool C>
  __device__ double jac_norm_rows(const double* yy) {
    double nm = 0.0;
#pragma unroll 1
    for (int i = 0; i < N(); ++i) {
      jac_row(yy, i);
      double sr = 0.0;
      for (int j = 0; j < N(); ++j) sr = sr + fabs(tmp[j * B]) * ewt[j * B];
      nm = fmax(nm, sr / ewt[i * B]);
    }
    if (C) {  // the oracle's count: rre_jacobian, then the norm
#pragma unroll 1
      for (int k = 0; k < m; ++k) {
        const int nt = KIN_RD_NTERMS(tab_rdesc(T, k));
        flops += static_cast<uint64_t>(nt) * (4 + nt + 2 * static_cast<uint64_t>(tab_col_ptr(T, k + 1) - tab_col_ptr(T, k)));
      }
      flops += 2 * static_cast<uint64_t>(N()) * N() + N();
    }
    return nm;
  }
  template <bool C>
  __device__ bool lu_factor() {
    for (int k = 0; k < N(); ++k) {
      int pr = k;
      double best = fabs(P[(k * N() + k) * B]);
      for (int i = k + 1; i < N(); ++i) {
        const double c = fabs(P[(i * N() + k) * B]);
        if (c > best) { best = c; pr = i; }
      }
      piv[k * B] = pr;
      if (best == 0.0) return false;
      if (pr != k)
        for (int j = 0; j < N(); ++j) {
          const double t0 = P[(k * N() + j) * B];
          P[(k * N() + j) * B] = P[(pr * N() + j) * B];
          P[(pr * N() + j) * B] = t0;
        }
      const double inv = 1.0 / P[(k * N() + k) * B];
      for (int i = k + 1; i < N(); ++i) {
        const double l = P[(i * N() + k) * B] * inv;
        P[(i * N() + k) * B] = l;
        for (int j = k + 1; j < N(); ++j) P[(i * N() + j) * B] = P[(i * N() + j) * B] - l * P[(k * N() + j) * B];
      }
    }
    if (C) flops += static_cast<uint64_t>(2 * N() * N() * N() / 3 + N());
    return true;
  }
  template <bool C>
  __device__ void lu_solve(double* b) {
    for (int k = 0; k < N(); ++k) {
      const int pk = piv[k * B];
      if (pk != k) {
        const double t0 = b[k * B];
        b[k * B] = b[pk * B];
        b[pk * B] = t0;
      }
      for (int i = k + 1; i < N(); ++i) b[i * B] = b[i * B] - P[(i * N() + k) * B] * b[k * B];
    }
    for (int i = N() - 1; i >= 0; --i) {
      double s = b[i * B];
      for (int j = i + 1; j < N(); ++j) s = s - P[(i * N() + j) * B] * b[j * B];
      b[i * B] = s / P[(i * N() + i) * B];
    }
    if (C) flops += static_cast<uint64_t>(2 * N() * N());
  }
  template <bool C>
  __device__ __forceinline__ double wrms(const double* vv) {
    if (C) flops += 3 * static_cast<uint64_t>(N()) + 2;
    return wrms_out_of_line<kN>(vv, ewt, N());
  }
};

template <bool kCount, int kN, class PM>
__device__ void lsoda_one(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, const double* co, uint64_t s,
                          double* smem_base, int* ismem_base, int tid, unsigned mask) {
  constexpr int B = kBlock;
  const uint64_t sim = global_sim(S, s);
  const int n = kN > 0 ? kN : T.n, m = T.m, G = T.n_grid;
  Lsoda<kN, PM> L{T, S, co, T.n, m};
  double* p = smem_base + tid;
  L.Z = p;
  p += kL * n * B;
  L.acor = p;
  p += n * B;
  L.savf = p;
  p += n * B;
  L.ewt = p;
  p += n * B;
  L.y = p;
  p += n * B;
  L.tmp = p;
  p += n * B;
  if constexpr (!Lsoda<kN, PM>::kRegLU) {
    L.P = p;
    p += n * n * B;
  }
  L.a = p;
  p += m * B;
  L.av = p;
  L.piv = ismem_base + tid;
  L.flops = 0;
  L.F_rhs = static_cast<uint64_t>(T.fprop) + 2 * static_cast<uint64_t>(T.nnz);

  decode_point(S, sim, L.av, B);
  const double rtol = S.rel_tol, atol = S.abs_tol;
  const double hmax = S.h_max > 0.0 ? S.h_max : KIN_INF;  // (NVRTC has no __builtin_huge_val)
  const double t_end = S.t_end;
  bool floored = false;
  uint64_t n_acc = 0, n_rej = 0, n_bdf = 0;  // n_bdf: accepted BDF steps (meta[3])
  int status = 0;

  auto emit = [&](int g, const double* vv) {
    double* o = O.traj + (static_cast<size_t>(s) * G + g) * n;  // [sim][g][n]
    for (int i = 0; i < n; ++i) {
      double vi = vv[i * B];
      if (vi < 0.0) { vi = 0.0; floored = true; }
      o[i] = vi;
    }
  };

  double t = 0.0;
  int gi = 0;
  for (int i = 0; i < n; ++i) {
    const int ax = tab_x0_axis(T, i);
    L.y[i * B] = ax < 0 ? tab_x0(T, i) : L.av[ax * B];
  }
  while (gi < G && tab_grid(T, S, gi) <= t) emit(gi++, L.y);
  if (t < t_end) {
    for (int i = 0; i < n; ++i) {
      L.z(0, i) = L.y[i * B];
      L.ewt[i * B] = rtol * fabs(L.y[i * B]) + atol;
    }
    L.template rhs<kCount>(L.y, L.savf);
    double h;
    if (S.h_init > 0.0) {
      h = S.h_init;
    } else {
      double tol = rtol;
      if (tol < 100.0 * 2.220446049250313e-16) tol = 100.0 * 2.220446049250313e-16;
      if (tol > 1e-3) tol = 1e-3;
      double fn = 0.0;
      for (int i = 0; i < n; ++i) fn = fmax(fn, fabs(L.savf[i * B]) / L.ewt[i * B]);
      const double w0 = t_end;
      const double sum = 1.0 / (tol * w0 * w0) + tol * fn * fn;
      h = 1.0 / sqrt(sum);
      if (h > t_end) h = t_end;
      if (h > hmax) h = hmax;
      if (kCount) L.flops += 2 * static_cast<uint64_t>(n) + 10;
    }
    for (int i = 0; i < n; ++i) L.z(1, i) = h * L.savf[i * B];

    int meth = 0, nq = 1, ialth = 2, icount = 20;
    int nstab = 0;  // consecutive order selections whose Adams step the stability cap bound
    double rmax = 1.0e4, crate = 0.7;
    bool ipup = false, jcur = false, have_p = false;
    double hl0_p = 0.0;
    uint64_t nst = 0, nslp = 0, attempts = 0;
    double el0 = L.elco(meth, nq, 0);
    auto maxord = [&]() { return meth == 0 ? 12 : 5; };
    auto set_order = [&](int mm, int q) { meth = mm; nq = q; el0 = L.elco(meth, nq, 0); };
    auto rescale = [&](double rh) {
      double r = rh;
#pragma unroll 1
      for (int j = 1; j <= nq; ++j) {
        for (int i = 0; i < n; ++i) L.z(j, i) = L.z(j, i) * r;
        r = r * rh;
      }
      h = h * rh;
      if (kCount) L.flops += static_cast<uint64_t>(nq) * (n + 1);
    };
    // kN > 0: the value each update adds (predict: z(j+1) as just updated;
    // unpredict: z(j+1) before its own update) is carried in registers
    // instead of re-read from shared memory — the same additions in the same
    // order, one load per element instead of two
    auto predict = [&]() {
      if constexpr (kN > 0) {
#pragma unroll 1
        for (int k = 0; k < nq; ++k) {
          double c[kN > 0 ? kN : 1];
#pragma unroll
          for (int i = 0; i < kN; ++i) c[i] = L.z(nq, i);
#pragma unroll 1
          for (int j = nq - 1; j >= k; --j)
#pragma unroll
            for (int i = 0; i < kN; ++i) {
              const double v = L.z(j, i) + c[i];
              L.z(j, i) = v;
              c[i] = v;
            }
        }
      } else {
#pragma unroll 1
        for (int k = 0; k < nq; ++k)
#pragma unroll 1
          for (int j = nq - 1; j >= k; --j)
            for (int i = 0; i < n; ++i) L.z(j, i) = L.z(j, i) + L.z(j + 1, i);
      }
      if (kCount) L.flops += static_cast<uint64_t>(nq) * (nq + 1) / 2 * n;
    };
    auto unpredict = [&]() {
      if constexpr (kN > 0) {
#pragma unroll 1
        for (int k = nq - 1; k >= 0; --k) {
          double c[kN > 0 ? kN : 1];
#pragma unroll
          for (int i = 0; i < kN; ++i) c[i] = L.z(k, i);
#pragma unroll 1
          for (int j = k; j <= nq - 1; ++j)
#pragma unroll
            for (int i = 0; i < kN; ++i) {
              const double nx = L.z(j + 1, i);
              L.z(j, i) = c[i] - nx;
              c[i] = nx;
            }
        }
      } else {
#pragma unroll 1
        for (int k = nq - 1; k >= 0; --k)
#pragma unroll 1
          for (int j = k; j <= nq - 1; ++j)
            for (int i = 0; i < n; ++i) L.z(j, i) = L.z(j, i) - L.z(j + 1, i);
      }
    };
    auto form_p = [&](const double* yy) {
      if constexpr (Lsoda<kN, PM>::kRegLU) {
        const double hl0 = h * el0;
        hl0_p = hl0;
        have_p = L.template form_lu_reg<kCount>(yy, hl0);
        return have_p;
      }
      L.template jacobian<kCount>(yy, L.P);
      const double hl0 = h * el0;
      for (int q = 0; q < n * n; ++q) L.P[q * B] = -hl0 * L.P[q * B];
      for (int i = 0; i < n; ++i) L.P[(i * n + i) * B] = L.P[(i * n + i) * B] + 1.0;
      hl0_p = hl0;
      have_p = L.template lu_factor<kCount>();
      return have_p;
    };
    auto jac_norm = [&](const double* yy) { return L.template jac_norm_rows<kCount>(yy); };
    auto cm1 = [&](int q) { return L.tesco(0, q, 1) * L.elco(0, q, q); };
    auto cm2 = [&](int q) { return L.tesco(1, q, 1) * L.elco(1, q, q); };

    // One accepted step per iteration, warp-synchronous: the lanes of `mask`
    // (one simulation each) reconverge at every step, so the shared
    // predictor / corrector / error-test code runs with the warp together
    // instead of drifting apart into 32 serial simulations.
    bool running = t < t_end && status == 0;
    bool fresh = true;  // the next attempt starts a new step (ewt, kflag, ncf reset)
    int kflag = 0, ncf = 0;
    double dsm = 0.0;
    while (__any_sync(mask, running)) {
      if (!running) continue;
      do {
      if (fresh) {
        for (int i = 0; i < n; ++i) L.ewt[i * B] = rtol * fabs(L.z(0, i)) + atol;
        kflag = 0;
        ncf = 0;
        dsm = 0.0;
        fresh = false;
      }
      // ONE attempt per trip of the warp loop: a lane whose step was rejected
      // retries on the next trip while the others take their next step (as
      // one attempt loop per trip, every lane waited out the warp's most
      // rejected step: with ~9% of attempts rejected, nearly every trip ran
      // two attempts).  `continue` below ends the trip without accepting.
      bool accepted = false;
      do {
        if (attempts++ >= S.max_steps) { status = KIN_SIM_BUDGET; break; }
        if (!(h > 0.0) || t + h == t) { status = KIN_SIM_STEP_UNDERFLOW; break; }
        if (meth == 1 && (!have_p || fabs(h * el0 / hl0_p - 1.0) > 0.3 || nst >= nslp + 20)) ipup = true;
        const double tn = t + h;
        predict();
        bool conv = false;
        for (;;) {
          for (int i = 0; i < n; ++i) L.y[i * B] = L.z(0, i);
          L.template rhs<kCount>(L.y, L.savf);
          if (meth == 1 && ipup) {
            if (!form_p(L.y)) { status = KIN_SIM_NONFINITE; break; }
            ipup = false;
            jcur = true;
            crate = 0.7;
            nslp = nst;
          }
          for (int i = 0; i < n; ++i) L.acor[i * B] = 0.0;
          double delp = 0.0;
          int mm = 0;
          for (;;) {
            double del;
            if (meth == 1) {
              for (int i = 0; i < n; ++i) L.tmp[i * B] = h * L.savf[i * B] - (L.z(1, i) + L.acor[i * B]);
              if constexpr (Lsoda<kN, PM>::kRegLU) L.template lu_solve_reg<kCount>(L.tmp);
              else L.template lu_solve<kCount>(L.tmp);
              del = L.template wrms<kCount>(L.tmp);
              for (int i = 0; i < n; ++i) {
                L.acor[i * B] = L.acor[i * B] + L.tmp[i * B];
                L.y[i * B] = L.z(0, i) + el0 * L.acor[i * B];
              }
            } else {
              for (int i = 0; i < n; ++i) L.tmp[i * B] = h * L.savf[i * B] - L.z(1, i);
              for (int i = 0; i < n; ++i) L.acor[i * B] = L.tmp[i * B] - L.acor[i * B];
              del = L.template wrms<kCount>(L.acor);
              for (int i = 0; i < n; ++i) {
                L.y[i * B] = L.z(0, i) + el0 * L.tmp[i * B];
                L.acor[i * B] = L.tmp[i * B];
              }
            }
            if (kCount) L.flops += 5 * static_cast<uint64_t>(n);
            if (!isfinite(del)) { conv = false; break; }
            if (mm != 0) crate = fmax(0.2 * crate, del / delp);
            const double conit = 0.5 / (nq + 2);
            const double dcon = del * fmin(1.0, 1.5 * crate) / (L.tesco(meth, nq, 1) * conit);
            if (dcon <= 1.0) { conv = true; break; }
            ++mm;
            if (mm == 3 || (mm >= 2 && del > 2.0 * delp)) break;
            delp = del;
            L.template rhs<kCount>(L.y, L.savf);
          }
          if (status != 0 || conv) break;
          if (meth == 1 && !jcur) { ipup = true; continue; }
          break;
        }
        if (status != 0) break;
        if (!conv) {
          unpredict();
          ++n_rej;
          if (++ncf >= 10) { status = KIN_SIM_STEP_UNDERFLOW; break; }
          rescale(0.25);
          if (meth == 1) ipup = true;
          continue;
        }
        jcur = false;
        dsm = L.template wrms<kCount>(L.acor) / L.tesco(meth, nq, 1);
        if (dsm > 1.0) {
          unpredict();
          ++n_rej;
          --kflag;
          if (kflag <= -3) {
            for (int i = 0; i < n; ++i) L.y[i * B] = L.z(0, i);
            h = h * 0.1;
            L.template rhs<kCount>(L.y, L.savf);
            for (int i = 0; i < n; ++i) L.z(1, i) = h * L.savf[i * B];
            set_order(meth, 1);
            ialth = 5;
            if (meth == 1) ipup = true;
            continue;
          }
          const double rhsm = step_ratio_q(dsm, nq + 1, 1.2, 1.2e-6);
          double rhdn = 0.0;
          if (nq > 1) {
            const double ddn = L.template wrms<kCount>(&L.z(nq, 0)) / L.tesco(meth, nq, 0);
            rhdn = step_ratio_q(ddn, nq, 1.3, 1.3e-6);
          }
          double rh;
          if (rhsm >= rhdn) {
            rh = rhsm;
          } else {
            rh = rhdn;
            set_order(meth, nq - 1);
          }
          rh = fmin(rh, 1.0);
          if (kflag <= -2) rh = fmin(rh, 0.2);
          rescale(rh);
          if (meth == 1) ipup = true;
          ialth = nq + 1;
          continue;
        }
        // accepted
        ++nst;
        ++n_acc;
        if (meth == 1) ++n_bdf;
        if constexpr (kN > 0) {  // acor held in registers across the rows
          double ac[kN > 0 ? kN : 1];
#pragma unroll
          for (int i = 0; i < kN; ++i) ac[i] = L.acor[i * B];
#pragma unroll 1
          for (int j = 0; j <= nq; ++j) {
            const double e = L.elco(meth, nq, j);
#pragma unroll
            for (int i = 0; i < kN; ++i) L.z(j, i) = L.z(j, i) + e * ac[i];
          }
        } else {
#pragma unroll 1
          for (int j = 0; j <= nq; ++j) {
            const double e = L.elco(meth, nq, j);
            for (int i = 0; i < n; ++i) L.z(j, i) = L.z(j, i) + e * L.acor[i * B];
          }
        }
        if (kCount) L.flops += 2 * static_cast<uint64_t>(nq + 1) * n;
        const double tprev = t;
        t = tn;
        for (;;) {
          if (!(gi < G)) break;
          const double tg = tab_grid(T, S, gi);
          if (!(tg <= t && tg > tprev)) break;
          const double sg = (tg - t) / h;
          if constexpr (kN > 0) {
            // Horner over the Nordsieck columns with the species as the inner
            // (unrolled) loop: kN independent chains instead of kN serial
            // ones — each species' operations and their order unchanged
            double vv[kN > 0 ? kN : 1];
#pragma unroll
            for (int i = 0; i < kN; ++i) vv[i] = L.z(nq, i);
#pragma unroll 1
            for (int j = nq - 1; j >= 0; --j)
#pragma unroll
              for (int i = 0; i < kN; ++i) vv[i] = L.z(j, i) + sg * vv[i];
            double* o = O.traj + (static_cast<size_t>(s) * G + gi) * n;  // emit() from registers
#pragma unroll
            for (int i = 0; i < kN; ++i) {
              double vi = vv[i];
              if (vi < 0.0) { vi = 0.0; floored = true; }
              o[i] = vi;
            }
            ++gi;
          } else {
            for (int i = 0; i < n; ++i) {
              double vv = L.z(nq, i);
#pragma unroll 1
              for (int j = nq - 1; j >= 0; --j) vv = L.z(j, i) + sg * vv;
              L.tmp[i * B] = vv;
            }
            emit(gi++, L.tmp);
          }
          if (kCount) L.flops += 2 * static_cast<uint64_t>(nq) * n + 2;
        }
        accepted = true;
      } while (0);
      if (status != 0 || !accepted) break;
      fresh = true;
      // order / step / method selection
      --ialth;
      if (ialth == 0) {
        const double rhsm = step_ratio_q(dsm, nq + 1, 1.2, 1.2e-6);
        double rhsm_cap;
        double rhup = 0.0;
        if (nq < maxord()) {
          for (int i = 0; i < n; ++i) L.tmp[i * B] = L.acor[i * B] - L.z(kL - 1, i);
          const double dup = L.template wrms<kCount>(L.tmp) / L.tesco(meth, nq, 2);
          rhup = step_ratio_q(dup, nq + 2, 1.4, 1.4e-6);
        }
        double rhdn = 0.0;
        if (nq > 1) {
          const double ddn = L.template wrms<kCount>(&L.z(nq, 0)) / L.tesco(meth, nq, 0);
          rhdn = step_ratio_q(ddn, nq, 1.3, 1.3e-6);
        }
        double pdnorm = -1.0;
        if (meth == 0) {
          pdnorm = jac_norm(&L.z(0, 0));
          const double pdh = fmax(h * pdnorm, 1.0e-6);
          if (nq < 12) rhup = fmin(rhup, c_sm1[nq + 1] / pdh);
          rhsm_cap = fmin(rhsm, c_sm1[nq] / pdh);
          if (nq > 1) rhdn = fmin(rhdn, c_sm1[nq - 1] / pdh);
          nstab = pdh >= 0.5 * c_sm1[nq] ? nstab + 1 : 0;  // within 2x of the stability boundary
        } else {
          rhsm_cap = rhsm;
          nstab = 0;
        }
        int newq = nq;
        double rh = rhsm_cap;
        if (rhsm_cap >= rhup) {
          if (rhsm_cap < rhdn) { newq = nq - 1; rh = rhdn; }
        } else if (rhup > rhdn) {
          newq = nq + 1;
          rh = rhup;
        } else {
          newq = nq - 1;
          rh = rhdn;
        }
        int newm = meth;
        if (icount > 0) {
          --icount;
        } else {
          if (pdnorm < 0.0) pdnorm = jac_norm(&L.z(0, 0));
          const double exsm = 1.0 / (nq + 1);
          if (meth == 0 && nq <= 5) {
            const double rh1 = rh;
            const double dm2 = dsm * (cm1(nq) / cm2(nq));
            const double rh2 = step_ratio_e(dm2, exsm, 1.2, 1.2e-6);
            if (rh2 >= 5.0 * rh1) {
              newm = 1; newq = nq; rh = rh2;
            } else if (nstab >= kLsodaStabSwitch) {
              // stiffness by stability: the Adams step has been held by its
              // stability region for many selections in a row
              newm = 1; newq = nq; rh = rh1;
            }
          } else if (meth == 1) {
            const double dm1 = dsm * (cm2(nq) / cm1(nq));
            double rh1 = step_ratio_e(dm1, exsm, 1.2, 1.2e-6);
            double rh1it = 2.0 * rh1;
            const double pdh = pdnorm * h;
            if (pdh * rh1 > 1e-5) rh1it = c_sm1[nq] / pdh;
            rh1 = fmin(rh1, rh1it);
            const double rh2 = rh;
            if (rh1 >= rh2) { newm = 0; newq = nq; rh = rh1; }
          }
          if (newm != meth) icount = 20;
          else icount = 0;
        }
        if (newm == meth && newq == nq && rh < 1.1) {
          ialth = 3;
        } else {
          if (newq == nq + 1) {
            const double r = L.elco(meth, nq, nq) / (nq + 1);
            for (int i = 0; i < n; ++i) L.z(newq, i) = L.acor[i * B] * r;
          }
          rh = fmin(rh, rmax);
          rh = rh / fmax(1.0, h * rh / hmax);
          if (newm != meth || newq != nq) set_order(newm, newq);
          rescale(rh);
          ialth = nq + 1;
          if (meth == 1) ipup = true;
        }
        rmax = 10.0;
      } else if (ialth == 1 && nq < maxord()) {
        for (int i = 0; i < n; ++i) L.z(kL - 1, i) = L.acor[i * B];
      }
      } while (0);
      running = t < t_end && status == 0;
    }
    if (status == 0)
      while (gi < G) emit(gi++, &L.z(0, 0));
  }
  if (status == 0)
    while (gi < G) emit(gi++, L.y);
  uint64_t* me = O.meta + s * 6;
  me[0] = n_acc;
  me[1] = n_rej;
  me[2] = 0;
  me[3] = n_bdf;
  me[4] = 0;
  me[5] = floored ? 1 : 0;
  O.status[s] = status;
  if (kCount && O.work) O.work[s] = L.flops;
}

// doubles of per-warp state (the pivot ints rounded up to whole doubles)
__host__ __device__ __forceinline__ size_t lsoda_warp_doubles(const KinTables& T, const KinSweepDev& S) {
  const size_t n = static_cast<size_t>(T.n);
  return (18 * n + n * n + T.m + S.n_axes) * kBlock + (n * kBlock + 1) / 2;
}

template <bool kCount, bool kGlobal, int kN, class PM>
__device__ __forceinline__ void lsoda_body(const KinTables& T, const KinSweepDev& S, const KinOutDev& O,
                                           const double* __restrict__ co, unsigned long long* __restrict__ next) {
  extern __shared__ double smem[];
  constexpr int B = kBlock;
  const int tid = threadIdx.x, lane = tid & 31;
  const int n = T.n;
  const size_t nd = static_cast<size_t>(18 * n + (Lsoda<kN, PM>::kRegLU ? 0 : n * n) + T.m + S.n_axes) * B;
  // state in shared memory, or (kGlobal: models too large for it) in this
  // block's region of global memory, same layout
  double* sbase = kGlobal ? S.gstate + static_cast<size_t>(blockIdx.x) * lsoda_warp_doubles(T, S) : smem;
  int* ism = reinterpret_cast<int*>(sbase + nd);
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, 32ULL);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (base >= S.n_local) break;
    const uint64_t s = base + lane;
    const unsigned mask = __ballot_sync(0xFFFFFFFFu, s < S.n_local);
    if (s < S.n_local) lsoda_one<kCount, kN, PM>(T, S, O, co, s, sbase, ism, tid, mask);
    __syncwarp();
  }
}

// __maxnreg__ rather than __launch_bounds__(32): with the launch bounds
// ptxas held these kernels at 128 registers and spilled (the generic variant
// 316 bytes, the N = 4 one 352 with the register LU); 200 lets them allocate
// what they use (N = 4: 167 registers, no spills) — residency is set by the
// shared-memory state anyway.
template <bool kCount, bool kGlobal, int kN>
__global__ void __maxnreg__(200) lsoda_kernel(const __grid_constant__ KinTables T,
                                               const __grid_constant__ KinSweepDev S, KinOutDev O,
                                               const double* __restrict__ co, unsigned long long* __restrict__ next) {
  lsoda_body<kCount, kGlobal, kN, TablePM>(T, S, O, co, next);
}

#ifndef __CUDACC_RTC__


// Host launcher of one kernel variant (explicitly instantiated across several
// translation units so the size-specialised variants compile in parallel).
template <bool kCount, bool kGlobal, int kN>
cudaError_t launch_k(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, const double* coeffs,
                     unsigned long long* counter, size_t smem, cudaStream_t stream) {
  auto kern = lsoda_kernel<kCount, kGlobal, kN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t warps = (S.n_local + 31) / 32;
  uint64_t resident = static_cast<uint64_t>(per_sm) * sms;
  if (S.gstate && resident > S.gstate_warps) resident = S.gstate_warps;
  const unsigned grid = static_cast<unsigned>(warps < resident ? warps : resident);
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  kern<<<grid, kBlock, smem, stream>>>(T, S, O, coeffs, counter);
  return cudaGetLastError();
}

#define KIN_LSODA_SIG(kc, kg, kn)                                                                                \
  cudaError_t launch_k<kc, kg, kn>(const KinTables&, const KinSweepDev&, const KinOutDev&, const double*,       \
                                   unsigned long long*, size_t, cudaStream_t)
#endif  // __CUDACC_RTC__

}  // namespace lsd
}  // namespace kin

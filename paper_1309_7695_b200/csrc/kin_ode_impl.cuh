// kin_ode.cu — batched Dormand-Prince 5(4) integration of the reaction-rate
// equations (K4 of DESIGN.md): the reference's Method::Ode.
//
//   rre_rhs ........ deterministic.hpp:85-88
//   rk_step/Dopri5 . deterministic.hpp:26-83, SPEC.md:224-232,249 (PI control, FSAL,
//                    Hairer continuous extension, exact at step ends SPEC.md:247)
//   integrate_rre .. deterministic.hpp:90-95, SPEC.md:233-241 (dense output onto the
//                    grid, floor at zero with a flag, max_steps / non-finite errors)
//
// Mapping: a group of L lanes integrates one simulation.  Lane l owns species
// i = l + q*L (q < SL); the nine Dopri5 vectors (y, k1..k7, y_new) of those
// species live in REGISTERS.  The RHS is evaluated cooperatively through a small
// per-group shared-memory scratch: owners publish the stage state xs[N], lanes
// compute propensities a[j] for j = l, l+L, ..., then owners gather their nu-rows
// (same reaction-ascending order as the oracle).  Norms are group reductions
// with __shfl_xor_sync.  L = 1 is the thread-per-simulation limit used for small
// models; C4 (N=33) uses L=8, SL=5.  Parity with the oracle is tolerance-based
// (FMA contraction and CUDA's pow differ from glibc in the last ulp).
#pragma once
#include "kin_device.cuh"
#include "kin_launch.h"

namespace kin {
namespace ode {

namespace dp {
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
constexpr double d1 = -12715105075.0 / 11282082432.0, d3 = 87487479700.0 / 32700410799.0,
                 d4 = -10690763975.0 / 1880347072.0, d5 = 701980252875.0 / 199316789632.0,
                 d6 = -1453857185.0 / 822651844.0, d7 = 69997945.0 / 29380423.0;
constexpr double kSafe = 0.9, kFacMinInv = 5.0, kFacMaxInv = 0.1, kBeta = 0.04, kExpo1 = 0.2 - kBeta * 0.75;
}  // namespace dp

// bytes of the table blob a block copies to shared memory (16-byte multiple)
__host__ __device__ __forceinline__ uint32_t table_smem_bytes(const KinTables& T) { return (T.used + 15u) & ~15u; }

template <int L>
struct Group {
  unsigned mask;
  __device__ __forceinline__ void sync() const {
    if (L > 1) __syncwarp(mask);
  }
  __device__ __forceinline__ double sum(double v) const {
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off, L);
    return v;
  }
  __device__ __forceinline__ double maxv(double v) const {
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(mask, v, off, L));
    return v;
  }
  __device__ __forceinline__ int any(int v) const {
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) v |= __shfl_xor_sync(mask, v, off, L);
    return v;
  }
};

template <int L, int SL, bool kCount>
__global__ void __launch_bounds__(128, 4) dopri5_kernel(const __grid_constant__ KinTables T,
                                                     const __grid_constant__ KinSweepDev S, KinOutDev O) {
  using namespace dp;
  extern __shared__ double smem[];
  // The model tables go to shared memory once per block: the RHS walks them
  // with lane-dependent indices (lane l handles reactions l, l+L, ...), which
  // the constant bank would serialise across the distinct addresses of a warp.
  const uint32_t tb = table_smem_bytes(T);
  unsigned char* tblob = reinterpret_cast<unsigned char*>(smem);
  for (uint32_t o = threadIdx.x * 16u; o < tb; o += blockDim.x * 16u)
    *reinterpret_cast<uint4*>(tblob + o) = *reinterpret_cast<const uint4*>(T.blob + o);
  __syncthreads();
  const int gpb = blockDim.x / L;
  const int grp = threadIdx.x / L, lane = threadIdx.x % L;
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * gpb + grp;
  if (s >= S.n_local) return;  // whole groups retire together
  const int N = T.n, M = T.m, G = T.n_grid;
  const uint64_t sim = global_sim(S, s);
  Group<L> grpc;
  grpc.mask = (L == 32) ? 0xFFFFFFFFu : (((1u << L) - 1u) << ((threadIdx.x & 31) / L * L));

  const int stride = N + M + S.n_axes;
  double* xs = smem + tb / sizeof(double) + static_cast<size_t>(grp) * stride;
  const double* s_rate = reinterpret_cast<const double*>(tblob + T.off_rate);
  const int8_t* s_rate_axis = reinterpret_cast<const int8_t*>(tblob + T.off_rate_axis);
  const int16_t* s_rt_ptr = reinterpret_cast<const int16_t*>(tblob + T.off_rt_ptr);
  const uint32_t* s_rt = reinterpret_cast<const uint32_t*>(tblob + T.off_rt);
  const int16_t* s_row_ptr = reinterpret_cast<const int16_t*>(tblob + T.off_row_ptr);
  const uint32_t* s_row = reinterpret_cast<const uint32_t*>(tblob + T.off_row);
  double* a = xs + N;
  double* av = a + M;
  // lane slot -> species / reaction: the work-balancing orders of kin_tables.h
  // for wide groups (C5, L = 32: 271 -> 232 ms); at L <= 8 the lookups cost
  // more than the balance saves (C4 9.3 -> 9.4 ms, C3 2.6 -> 2.8 ms)
  constexpr bool kPerm = L >= 16;
  const int16_t* s_sp =
      (kPerm && T.off_sp_perm) ? reinterpret_cast<const int16_t*>(tblob + T.off_sp_perm) : nullptr;
  const int16_t* s_rx =
      (kPerm && T.off_rx_perm) ? reinterpret_cast<const int16_t*>(tblob + T.off_rx_perm) : nullptr;
  auto species = [&](int slot) { return s_sp ? static_cast<int>(s_sp[slot]) : slot; };

  if (lane == 0) {
    uint64_t rem = sim / S.runs;
    for (int ax = S.n_axes - 1; ax >= 0; --ax) {
      const uint64_t nv = static_cast<uint64_t>(S.axis_n[ax]);
      const uint64_t q = rem / nv;
      av[ax] = __ldg(S.axis_values[ax] + (rem - q * nv));
      rem = q;
    }
  }
  grpc.sync();

  double y[SL], k1[SL], k2[SL], k3[SL], k4[SL], k5[SL], k6[SL], k7[SL], yn[SL];
#pragma unroll
  for (int q = 0; q < SL; ++q) {
    const int slot = lane + q * L;
    y[q] = 0.0;
    if (slot < N) {
      const int i = species(slot);
      const int ax = tab_x0_axis(T, i);
      y[q] = ax < 0 ? tab_x0(T, i) : av[ax];
    }
  }
  const uint64_t F_rhs = static_cast<uint64_t>(T.fprop) + 2 * static_cast<uint64_t>(T.nnz);
  uint64_t flops = 0;

  // RHS of the stage state already published in xs: dx = nu * a(xs).
  auto rhs = [&](double* out) {
    grpc.sync();
    for (int jj = lane; jj < M; jj += L) {
      const int j = s_rx ? static_cast<int>(s_rx[jj]) : jj;
      const int ax = s_rate_axis[j];
      double aj = ax < 0 ? s_rate[j] : __dmul_rn(s_rate[j], av[ax]);
      const int p1 = s_rt_ptr[j + 1];
#pragma unroll 1
      for (int p = s_rt_ptr[j]; p < p1; ++p) {
        const uint32_t e = s_rt[p];
        aj = aj * combinations(xs[KIN_TERM_SPECIES(e)], KIN_TERM_STOICH(e));
      }
      a[j] = aj;
    }
    grpc.sync();
#pragma unroll
    for (int q = 0; q < SL; ++q) {
      const int slot = lane + q * L;
      double acc = 0.0;
      if (slot < N) {
        const int i = species(slot);
        const int p1 = s_row_ptr[i + 1];
#pragma unroll 1
        for (int p = s_row_ptr[i]; p < p1; ++p) {
          const uint32_t e = s_row[p];
          acc = acc + static_cast<double>(KIN_NU_DELTA(e)) * a[KIN_NU_INDEX(e)];
        }
      }
      out[q] = acc;
    }
    if (kCount && lane == 0) flops += F_rhs;
  };
  auto publish = [&](const double* v) {
#pragma unroll
    for (int q = 0; q < SL; ++q) {
      const int slot = lane + q * L;
      if (slot < N) xs[species(slot)] = v[q];
    }
  };
  auto emit = [&](int g, const double* v) {
    double* o = O.traj + (static_cast<size_t>(s) * G + g) * N;  // [sim][g][n]
#pragma unroll
    for (int q = 0; q < SL; ++q) {
      const int slot = lane + q * L;
      if (slot < N) o[species(slot)] = v[q];
    }
  };

  const double rtol = S.rel_tol, atol = S.abs_tol;
  const double hmax = S.h_max > 0.0 ? S.h_max : __builtin_huge_val();
  const double t_end = S.t_end;
  double t = 0.0;
  int gi = 0;
  int status = 0, floored = 0;
  uint64_t n_acc = 0, n_rej = 0;
  while (gi < G && tab_grid(T, S, gi) <= t) emit(gi++, y);

  if (t < t_end) {
    publish(y);
    rhs(k1);
    double h;
    if (S.h_init > 0.0) {
      h = S.h_init;
    } else {  // Hairer HINIT (order 5)
      double pf = 0.0, py = 0.0;
#pragma unroll
      for (int q = 0; q < SL; ++q) {
        if (lane + q * L < N) {
          const double sk = atol + rtol * fabs(y[q]);
          const double qf = k1[q] / sk, qy = y[q] / sk;
          pf += qf * qf;
          py += qy * qy;
        }
      }
      const double dnf = grpc.sum(pf), dny = grpc.sum(py);
      h = (dnf <= 1e-10 || dny <= 1e-10) ? 1.0e-6 : sqrt(dny / dnf) * 0.01;
      if (h > hmax) h = hmax;
#pragma unroll
      for (int q = 0; q < SL; ++q) yn[q] = y[q] + h * k1[q];
      grpc.sync();
      publish(yn);
      rhs(k2);
      double pd = 0.0;
#pragma unroll
      for (int q = 0; q < SL; ++q) {
        if (lane + q * L < N) {
          const double sk = atol + rtol * fabs(y[q]);
          const double qq = (k2[q] - k1[q]) / sk;
          pd += qq * qq;
        }
      }
      const double der2 = sqrt(grpc.sum(pd)) / h;
      const double der12 = fmax(der2, sqrt(dnf));
      const double h1 = der12 <= 1e-15 ? fmax(1.0e-6, h * 1.0e-3) : pow(0.01 / der12, 0.2);
      h = fmin(100.0 * h, h1);
      if (h > hmax) h = hmax;
      if (kCount && lane == 0) flops += 15 * static_cast<uint64_t>(N) + 12;
    }

    double facold = 1.0e-4;
    bool last_rejected = false;
    uint64_t attempts = 0;
    while (t < t_end) {
      if (attempts++ >= S.max_steps) { status = KIN_SIM_BUDGET; break; }
      double hh = h < hmax ? h : hmax;
      bool hit = false;
      if (t + hh >= t_end) { hh = t_end - t; hit = true; }
      if (!(hh > 0.0) || t + hh == t) { status = KIN_SIM_STEP_UNDERFLOW; break; }

#pragma unroll
      for (int q = 0; q < SL; ++q) yn[q] = y[q] + hh * (a21 * k1[q]);
      grpc.sync(); publish(yn); rhs(k2);
#pragma unroll
      for (int q = 0; q < SL; ++q) yn[q] = y[q] + hh * (a31 * k1[q] + a32 * k2[q]);
      grpc.sync(); publish(yn); rhs(k3);
#pragma unroll
      for (int q = 0; q < SL; ++q) yn[q] = y[q] + hh * (a41 * k1[q] + a42 * k2[q] + a43 * k3[q]);
      grpc.sync(); publish(yn); rhs(k4);
#pragma unroll
      for (int q = 0; q < SL; ++q) yn[q] = y[q] + hh * (a51 * k1[q] + a52 * k2[q] + a53 * k3[q] + a54 * k4[q]);
      grpc.sync(); publish(yn); rhs(k5);
#pragma unroll
      for (int q = 0; q < SL; ++q)
        yn[q] = y[q] + hh * (a61 * k1[q] + a62 * k2[q] + a63 * k3[q] + a64 * k4[q] + a65 * k5[q]);
      grpc.sync(); publish(yn); rhs(k6);
#pragma unroll
      for (int q = 0; q < SL; ++q)
        yn[q] = y[q] + hh * (a71 * k1[q] + a73 * k3[q] + a74 * k4[q] + a75 * k5[q] + a76 * k6[q]);
      grpc.sync(); publish(yn); rhs(k7);

      double part = 0.0;
      int bad = 0;
#pragma unroll
      for (int q = 0; q < SL; ++q) {
        if (lane + q * L < N) {
          const double e = hh * (e1 * k1[q] + e3 * k3[q] + e4 * k4[q] + e5 * k5[q] + e6 * k6[q] + e7 * k7[q]);
          const double sk = atol + rtol * fmax(fabs(y[q]), fabs(yn[q]));
          const double r = e / sk;
          part += r * r;
          bad |= !isfinite(yn[q]);
        }
      }
      const double err = sqrt(grpc.sum(part) / static_cast<double>(N));
      bad = grpc.any(bad);
      if (kCount && lane == 0) flops += 63 * static_cast<uint64_t>(N) + 4;
      if (bad || !isfinite(err)) { status = KIN_SIM_NONFINITE; break; }
      const double fac11 = pow(err, kExpo1);

      if (err <= 1.0) {
        double fac = fac11 / pow(facold, kBeta);
        fac = fmax(kFacMaxInv, fmin(kFacMinInv, fac / kSafe));
        double hnew = hh / fac;
        facold = fmax(err, 1.0e-4);
        const double tprev = t;
        t = hit ? t_end : t + hh;
        if (kCount && lane == 0) flops += 18 * static_cast<uint64_t>(N) + 8;
        // dense output onto grid points in (tprev, t]
        while (gi < G && tab_grid(T, S, gi) <= t) {
          const double tg = tab_grid(T, S, gi);
          double v[SL];
          if (tg == t) {
#pragma unroll
            for (int q = 0; q < SL; ++q) v[q] = yn[q];
          } else {
            const double th = (tg - tprev) / hh;
            const double th1 = 1.0 - th;
#pragma unroll
            for (int q = 0; q < SL; ++q) {
              const double r2 = yn[q] - y[q];
              const double r3 = hh * k1[q] - r2;
              const double r4 = r2 - hh * k7[q] - r3;
              const double r5 = hh * (d1 * k1[q] + d3 * k3[q] + d4 * k4[q] + d5 * k5[q] + d6 * k6[q] + d7 * k7[q]);
              v[q] = y[q] + th * (r2 + th1 * (r3 + th * (r4 + th1 * r5)));
            }
            if (kCount && lane == 0) flops += 8 * static_cast<uint64_t>(N) + 3;
          }
#pragma unroll
          for (int q = 0; q < SL; ++q)
            if (v[q] < 0.0) { v[q] = 0.0; floored = 1; }
          emit(gi++, v);
        }
        int lifted = 0;
#pragma unroll
        for (int q = 0; q < SL; ++q) {
          y[q] = yn[q];
          k1[q] = k7[q];
          if (y[q] < 0.0) { y[q] = 0.0; lifted = 1; }
        }
        if (last_rejected && hnew > hh) hnew = hh;
        last_rejected = false;
        h = hnew;
        ++n_acc;
        if (grpc.any(lifted)) {
          floored = 1;
          grpc.sync();
          publish(y);
          rhs(k1);
        }
      } else {
        h = hh / fmin(kFacMinInv, fac11 / kSafe);
        last_rejected = true;
        ++n_rej;
        if (kCount && lane == 0) flops += 3;
      }
    }
  }
  if (status == 0)
    while (gi < G) emit(gi++, y);
  floored = grpc.any(floored);
  if (lane == 0) {
    uint64_t* me = O.meta + s * 6;
    me[0] = n_acc;
    me[1] = n_rej;
    me[2] = 0;
    me[3] = 0;
    me[4] = 0;
    me[5] = floored ? 1 : 0;
    O.status[s] = status;
    if (kCount && O.work) O.work[s] = flops;
  }
}

template <int L, int SL>
cudaError_t launch_t(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count, cudaStream_t st) {
  constexpr int kBlock = 128;
  constexpr int gpb = kBlock / L;
  const size_t smem = table_smem_bytes(T) + static_cast<size_t>(gpb) * (T.n + T.m + S.n_axes) * sizeof(double);
  const unsigned grid = static_cast<unsigned>((S.n_local + gpb - 1) / gpb);
  if (count) {
    cudaFuncSetAttribute(dopri5_kernel<L, SL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dopri5_kernel<L, SL, true><<<grid, kBlock, smem, st>>>(T, S, O);
  } else {
    cudaFuncSetAttribute(dopri5_kernel<L, SL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dopri5_kernel<L, SL, false><<<grid, kBlock, smem, st>>>(T, S, O);
  }
  return cudaGetLastError();
}

}  // namespace ode
}  // namespace kin

// oracle/kin_lsoda.hpp — TEST INFRASTRUCTURE ONLY.
//
// LSODA-style integrator for the reaction-rate equations (north-star
// extension: the reference's only ODE method is Dopri5, deterministic.hpp:38-83,
// and stiff solvers are a SPEC non-goal).  Restated from the
// published ODEPACK algorithm (Hindmarsh's LSODE stode/cfode, Petzold's LSODA
// method switching) — no reference implementation exists to pin it, so parity
// is GPU-vs-this-oracle plus accuracy against analytic solutions and against
// scipy's LSODA (tests/test_oracle_lsoda.py).
//
// The same algorithm, statement for statement, runs on the device
// (paper_1309_7695_b200/csrc/kin_lsoda.cu).  Shared pieces that must agree
// exactly (the cfode coefficient tables) are computed by kin_lsoda_coeffs()
// here and by the engine's host code from the same recurrences.
#pragma once

#include <cmath>

namespace kin_oracle {

constexpr int kLsodaMaxOrdAdams = 12;
constexpr int kLsodaMaxOrdBdf = 5;
constexpr int kLsodaL = kLsodaMaxOrdAdams + 1;  // Nordsieck vectors (0..12)

// cfode: elco[meth][nq][0..nq], tesco[meth][nq][0..2] for nq = 1..maxord.
struct LsodaCoeffs {
  double elco[2][13][14];
  double tesco[2][13][3];
};

inline void kin_lsoda_coeffs(LsodaCoeffs* C) {
  for (int m = 0; m < 2; ++m)
    for (int q = 0; q < 13; ++q) {
      for (int i = 0; i < 14; ++i) C->elco[m][q][i] = 0.0;
      for (int i = 0; i < 3; ++i) C->tesco[m][q][i] = 0.0;
    }
  // ---- Adams (meth index 0) ----
  {
    double pc[13];
    C->elco[0][1][0] = 1.0;
    C->elco[0][1][1] = 1.0;
    C->tesco[0][1][0] = 0.0;
    C->tesco[0][1][1] = 2.0;
    C->tesco[0][2][0] = 1.0;
    C->tesco[0][12][2] = 0.0;
    pc[0] = 1.0;
    double rqfac = 1.0;
    for (int nq = 2; nq <= 12; ++nq) {
      // p(x) = (x+1)(x+2)...(x+nq-1), coefficients pc[0..nq-1]
      const double rq1fac = rqfac;
      rqfac = rqfac / nq;
      const int nqm1 = nq - 1;
      const double fnqm1 = nqm1;
      pc[nq - 1] = 0.0;
      for (int i = nq - 1; i >= 1; --i) pc[i] = pc[i - 1] + fnqm1 * pc[i];
      pc[0] = fnqm1 * pc[0];
      // integrals over [-1,0] of p(x) and x p(x)
      double pint = pc[0], xpin = pc[0] / 2.0, tsign = 1.0;
      for (int i = 1; i < nq; ++i) {
        tsign = -tsign;
        pint += tsign * pc[i] / (i + 1);
        xpin += tsign * pc[i] / (i + 2);
      }
      C->elco[0][nq][0] = pint * rq1fac;
      C->elco[0][nq][1] = 1.0;
      for (int i = 1; i < nq; ++i) C->elco[0][nq][i + 1] = rq1fac * pc[i] / (i + 1);
      const double agamq = rqfac * xpin;
      const double ragq = 1.0 / agamq;
      C->tesco[0][nq][1] = ragq;
      if (nq < 12) C->tesco[0][nq + 1][0] = ragq * rqfac / (nq + 1);
      C->tesco[0][nq - 1][2] = ragq;
    }
  }
  // ---- BDF (meth index 1) ----
  {
    double pc[7];
    pc[0] = 1.0;
    double rq1fac = 1.0;
    for (int nq = 1; nq <= 5; ++nq) {
      // p(x) = (x+1)(x+2)...(x+nq)
      const double fnq = nq;
      pc[nq] = 0.0;
      for (int i = nq; i >= 1; --i) pc[i] = pc[i - 1] + fnq * pc[i];
      pc[0] = fnq * pc[0];
      for (int i = 0; i <= nq; ++i) C->elco[1][nq][i] = pc[i] / pc[1];
      C->elco[1][nq][1] = 1.0;
      C->tesco[1][nq][0] = rq1fac;
      C->tesco[1][nq][1] = (nq + 1) / C->elco[1][nq][0];
      C->tesco[1][nq][2] = (nq + 2) / C->elco[1][nq][0];
      rq1fac = rq1fac / fnq;
    }
  }
}

// Adams stability-region sizes (LSODA sm1), orders 1..12.
constexpr int kLsodaStabSwitch = 8;  // see integrate_lsoda: Adams -> BDF on a binding stability cap
constexpr double kLsodaSm1[13] = {0.0, 0.5, 0.575, 0.55, 0.45, 0.35, 0.25, 0.2, 0.15, 0.1, 0.075, 0.05, 0.025};

}  // namespace kin_oracle

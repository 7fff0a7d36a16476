// kin_ode.cu — Dopri5 launcher dispatch (instantiations live in kin_ode_l*.cu so
// they compile in parallel).  Kernel: kin_ode_impl.cuh.
#include "kin_launch.h"

namespace kin {
namespace ode {
template <int L, int SL>
cudaError_t launch_t(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count, cudaStream_t st);
}  // namespace ode

int ode_pick_lanes(int n) {
  if (n <= 4) return 1;
  if (n <= 8) return 2;
  if (n <= 16) return 4;
  if (n <= 40) return 8;
  if (n <= 64) return 16;
  return 32;
}

cudaError_t launch_dopri5(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count, int lanes,
                          cudaStream_t st) {
  using ode::launch_t;
  if (S.n_local == 0) return cudaSuccess;
  const int n = T.n;
  if (lanes <= 0) lanes = ode_pick_lanes(n);
  switch (lanes) {
    case 1:
      if (n <= 4) return launch_t<1, 4>(T, S, O, count, st);
      if (n <= 8) return launch_t<1, 8>(T, S, O, count, st);
      break;
    case 2:
      if (n <= 8) return launch_t<2, 4>(T, S, O, count, st);
      break;
    case 4:
      if (n <= 16) return launch_t<4, 4>(T, S, O, count, st);
      break;
    case 8:
      if (n <= 40) return launch_t<8, 5>(T, S, O, count, st);
      break;
    case 16:
      if (n <= 48) return launch_t<16, 3>(T, S, O, count, st);
      if (n <= 64) return launch_t<16, 4>(T, S, O, count, st);
      break;
    case 32:
      if (n <= 64) return launch_t<32, 2>(T, S, O, count, st);
      if (n <= 128) return launch_t<32, 4>(T, S, O, count, st);
      if (n <= 256) return launch_t<32, 8>(T, S, O, count, st);
      break;
  }
  return cudaErrorInvalidConfiguration;
}

}  // namespace kin

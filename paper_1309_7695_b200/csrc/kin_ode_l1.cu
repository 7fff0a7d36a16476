// Dopri5 instantiations (see kin_ode_impl.cuh).
#include "kin_ode_impl.cuh"

namespace kin {
namespace ode {
template cudaError_t launch_t<1, 4>(const KinTables&, const KinSweepDev&, const KinOutDev&, bool, cudaStream_t);
template cudaError_t launch_t<1, 8>(const KinTables&, const KinSweepDev&, const KinOutDev&, bool, cudaStream_t);
template cudaError_t launch_t<2, 4>(const KinTables&, const KinSweepDev&, const KinOutDev&, bool, cudaStream_t);
}  // namespace ode
}  // namespace kin

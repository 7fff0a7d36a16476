// kin_hybrid_n34.cu — hybrid kernel variants specialised on N = 3, 4
// (explicit instantiations; see kin_hybrid.cu).
#include "kin_hybrid_impl.cuh"

namespace kin {
namespace hyb {
template KIN_HYB_SIG(false, true, false, 3);
template KIN_HYB_SIG(false, false, false, 3);
template KIN_HYB_SIG(false, true, false, 4);
template KIN_HYB_SIG(false, false, false, 4);
}  // namespace hyb
}  // namespace kin

// kin_hybrid_n78.cu — hybrid kernel variants specialised on N = 7, 8
// (explicit instantiations; see kin_hybrid.cu).
#include "kin_hybrid_impl.cuh"

namespace kin {
namespace hyb {
template KIN_HYB_SIG(false, true, false, 7);
template KIN_HYB_SIG(false, false, false, 7);
template KIN_HYB_SIG(false, true, false, 8);
template KIN_HYB_SIG(false, false, false, 8);
}  // namespace hyb
}  // namespace kin

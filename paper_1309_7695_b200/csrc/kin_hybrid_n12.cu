// kin_hybrid_n12.cu — hybrid kernel variants specialised on N = 1, 2
// (explicit instantiations; see kin_hybrid.cu).
#include "kin_hybrid_impl.cuh"

namespace kin {
namespace hyb {
template KIN_HYB_SIG(false, true, false, 1);
template KIN_HYB_SIG(false, false, false, 1);
template KIN_HYB_SIG(false, true, false, 2);
template KIN_HYB_SIG(false, false, false, 2);
}  // namespace hyb
}  // namespace kin

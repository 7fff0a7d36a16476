// kin_hybrid_n56.cu — hybrid kernel variants specialised on N = 5, 6
// (explicit instantiations; see kin_hybrid.cu).
#include "kin_hybrid_impl.cuh"

namespace kin {
namespace hyb {
template KIN_HYB_SIG(false, true, false, 5);
template KIN_HYB_SIG(false, false, false, 5);
template KIN_HYB_SIG(false, true, false, 6);
template KIN_HYB_SIG(false, false, false, 6);
}  // namespace hyb
}  // namespace kin

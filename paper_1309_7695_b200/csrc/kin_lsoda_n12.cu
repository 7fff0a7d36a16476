// kin_lsoda_n12.cu — LSODA kernel variants specialised on N = 1, 2
// (explicit instantiations; see kin_lsoda.cu).
#include "kin_lsoda_impl.cuh"

namespace kin {
namespace lsd {
template KIN_LSODA_SIG(true, false, 1);
template KIN_LSODA_SIG(false, false, 1);
template KIN_LSODA_SIG(true, false, 2);
template KIN_LSODA_SIG(false, false, 2);
}  // namespace lsd
}  // namespace kin

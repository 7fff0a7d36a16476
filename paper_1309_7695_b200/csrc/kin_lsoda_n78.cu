// kin_lsoda_n78.cu — LSODA kernel variants specialised on N = 7, 8
// (explicit instantiations; see kin_lsoda.cu).
#include "kin_lsoda_impl.cuh"

namespace kin {
namespace lsd {
template KIN_LSODA_SIG(true, false, 7);
template KIN_LSODA_SIG(false, false, 7);
template KIN_LSODA_SIG(true, false, 8);
template KIN_LSODA_SIG(false, false, 8);
}  // namespace lsd
}  // namespace kin

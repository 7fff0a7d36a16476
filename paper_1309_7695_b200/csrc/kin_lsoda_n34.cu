// kin_lsoda_n34.cu — LSODA kernel variants specialised on N = 3, 4
// (explicit instantiations; see kin_lsoda.cu).
#include "kin_lsoda_impl.cuh"

namespace kin {
namespace lsd {
template KIN_LSODA_SIG(true, false, 3);
template KIN_LSODA_SIG(false, false, 3);
template KIN_LSODA_SIG(true, false, 4);
template KIN_LSODA_SIG(false, false, 4);
}  // namespace lsd
}  // namespace kin

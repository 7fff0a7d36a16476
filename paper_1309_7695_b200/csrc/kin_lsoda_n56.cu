// kin_lsoda_n56.cu — LSODA kernel variants specialised on N = 5, 6
// (explicit instantiations; see kin_lsoda.cu).
#include "kin_lsoda_impl.cuh"

namespace kin {
namespace lsd {
template KIN_LSODA_SIG(true, false, 5);
template KIN_LSODA_SIG(false, false, 5);
template KIN_LSODA_SIG(true, false, 6);
template KIN_LSODA_SIG(false, false, 6);
}  // namespace lsd
}  // namespace kin

// kin_lsoda.cu — LSODA sweep: launch dispatch and the generic kernel variants.
// Kernel: kin_lsoda_impl.cuh; the variants specialised on the species count
// are instantiated in kin_lsoda_n*.cu (parallel compilation).
#include "kin_lsoda_impl.cuh"

namespace kin {
namespace lsd {
#define KIN_LSODA_EXTERN(k) extern template KIN_LSODA_SIG(true, false, k); extern template KIN_LSODA_SIG(false, false, k);
KIN_LSODA_EXTERN(1) KIN_LSODA_EXTERN(2) KIN_LSODA_EXTERN(3) KIN_LSODA_EXTERN(4)
KIN_LSODA_EXTERN(5) KIN_LSODA_EXTERN(6) KIN_LSODA_EXTERN(7) KIN_LSODA_EXTERN(8)
#undef KIN_LSODA_EXTERN
}  // namespace lsd

size_t lsoda_state_doubles_per_warp(const KinTables& T, const KinSweepDev& S) { return lsd::lsoda_warp_doubles(T, S); }

size_t lsoda_smem_bytes(const KinTables& T, const KinSweepDev& S) {
  const int n = T.n;
  // N <= 4: the iteration matrix, its LU factors and pivots are in registers
  if (lsd::kLsodaRegLU && n >= 1 && n <= 4)
    return static_cast<size_t>(18 * n + T.m + S.n_axes) * lsd::kBlock * sizeof(double);
  return static_cast<size_t>(18 * n + n * n + T.m + S.n_axes) * lsd::kBlock * sizeof(double) +
         static_cast<size_t>(n) * lsd::kBlock * sizeof(int);
}

cudaError_t launch_lsoda(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count, const double* coeffs,
                         unsigned long long* counter, cudaStream_t stream) {
  using namespace lsd;
  if (S.n_local == 0) return cudaSuccess;
  const size_t smem = S.gstate ? 0 : lsoda_smem_bytes(T, S);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  if (S.gstate)
    return count ? launch_k<true, true, 0>(T, S, O, coeffs, counter, smem, stream)
                 : launch_k<false, true, 0>(T, S, O, coeffs, counter, smem, stream);
  switch (T.n) {  // small models: the kernel specialised on the species count
#define KIN_LSODA_CASE(k)                                                        \
  case k:                                                                        \
    return count ? launch_k<true, false, k>(T, S, O, coeffs, counter, smem, stream) \
                 : launch_k<false, false, k>(T, S, O, coeffs, counter, smem, stream);
    KIN_LSODA_CASE(1) KIN_LSODA_CASE(2) KIN_LSODA_CASE(3) KIN_LSODA_CASE(4)
    KIN_LSODA_CASE(5) KIN_LSODA_CASE(6) KIN_LSODA_CASE(7) KIN_LSODA_CASE(8)
#undef KIN_LSODA_CASE
    default:
      return count ? launch_k<true, false, 0>(T, S, O, coeffs, counter, smem, stream)
                   : launch_k<false, false, 0>(T, S, O, coeffs, counter, smem, stream);
  }
}

}  // namespace kin

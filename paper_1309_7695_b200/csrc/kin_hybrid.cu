// kin_hybrid.cu — hybrid PDMP sweep: launch dispatch and the generic kernel
// variants.  Kernel: kin_hybrid_impl.cuh; the variants specialised on the
// species count are instantiated in kin_hybrid_n*.cu (parallel compilation).
#include "kin_hybrid_impl.cuh"

namespace kin {
namespace hyb {
#define KIN_HYB_EXTERN(k) extern template KIN_HYB_SIG(false, true, false, k); extern template KIN_HYB_SIG(false, false, false, k);
KIN_HYB_EXTERN(1) KIN_HYB_EXTERN(2) KIN_HYB_EXTERN(3) KIN_HYB_EXTERN(4)
KIN_HYB_EXTERN(5) KIN_HYB_EXTERN(6) KIN_HYB_EXTERN(7) KIN_HYB_EXTERN(8)
#undef KIN_HYB_EXTERN
}  // namespace hyb

size_t hybrid_state_doubles_per_warp(const KinTables& T, const KinSweepDev& S) { return hyb::hybrid_warp_doubles(T, S); }

size_t hybrid_smem_bytes(const KinTables& T, const KinSweepDev& S) {
  const size_t words = (static_cast<size_t>(T.m) + 31) / 32;
  return (static_cast<size_t>(hyb::kVecs) * (T.n + 1) + T.m + S.n_axes) * hyb::kBlock * sizeof(double) +
         words * hyb::kBlock * sizeof(uint32_t);
}

cudaError_t launch_hybrid(const KinTables& T, const KinSweepDev& S, const KinOutDev& O, bool count,
                          unsigned long long* counter, cudaStream_t stream) {
  using namespace hyb;
  if (S.n_local == 0) return cudaSuccess;
  const size_t smem = S.gstate ? 0 : hybrid_smem_bytes(T, S);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  const bool ph = S.rng_mode == KIN_RNG_PHILOX;
  if (S.gstate)
    return count ? (ph ? launch_k<true, true, true, 0>(T, S, O, counter, smem, stream)
                       : launch_k<true, false, true, 0>(T, S, O, counter, smem, stream))
                 : (ph ? launch_k<false, true, true, 0>(T, S, O, counter, smem, stream)
                       : launch_k<false, false, true, 0>(T, S, O, counter, smem, stream));
  if (!count && T.n <= 8) {  // small models: specialised on the species count
    switch (T.n) {
#define KIN_HYB_CASE(k)                                                   \
  case k:                                                                 \
    return ph ? launch_k<false, true, false, k>(T, S, O, counter, smem, stream) \
              : launch_k<false, false, false, k>(T, S, O, counter, smem, stream);
      KIN_HYB_CASE(1) KIN_HYB_CASE(2) KIN_HYB_CASE(3) KIN_HYB_CASE(4)
      KIN_HYB_CASE(5) KIN_HYB_CASE(6) KIN_HYB_CASE(7) KIN_HYB_CASE(8)
#undef KIN_HYB_CASE
    }
  }
  return count ? (ph ? launch_k<true, true, false, 0>(T, S, O, counter, smem, stream)
                     : launch_k<true, false, false, 0>(T, S, O, counter, smem, stream))
               : (ph ? launch_k<false, true, false, 0>(T, S, O, counter, smem, stream)
                     : launch_k<false, false, false, 0>(T, S, O, counter, smem, stream));
}

}  // namespace kin

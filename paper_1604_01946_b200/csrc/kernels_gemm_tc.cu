// kernels_gemm_tc.cu -- instantiations of the one-tile-per-CTA tcgen05 GEMM (gemm_tc.cuh).
#include "gemm_tc.cuh"
#include "kernel_ptrs.h"

namespace rw {

// bf16: one accumulation over the whole K (BNV 0); two-plane formats: chunked promotion with
// BNV = the tile width (64 or 128)
template <class P, bool AMN, bool BMN>
static void* tc_ptr(int bnv) {
  if constexpr (P::kPlanes == 1) {
    return (void*)k_gemm_tc<P, AMN, BMN, 0>;
  } else {
    return bnv == 128 ? (void*)k_gemm_tc<P, AMN, BMN, 128> : (void*)k_gemm_tc<P, AMN, BMN, 64>;
  }
}
template <class P>
static void* tc_ptr_p(bool amn, bool bmn, int bnv) {
  if (amn) return bmn ? tc_ptr<P, true, true>(bnv) : tc_ptr<P, true, false>(bnv);
  return bmn ? tc_ptr<P, false, true>(bnv) : tc_ptr<P, false, false>(bnv);
}

void* gemm_tc_ptr(int prec, bool amn, bool bmn, int bnv) {
  if (prec == kBF16) return tc_ptr_p<PrecBF16>(amn, bmn, bnv);
  if (prec == kF16x2) return tc_ptr_p<PrecF16x2>(amn, bmn, bnv);
  return tc_ptr_p<PrecTF32x3>(amn, bmn, bnv);
}

}  // namespace rw

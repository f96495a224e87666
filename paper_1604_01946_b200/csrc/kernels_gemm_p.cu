// kernels_gemm_p.cu -- instantiations of the persistent bf16 GEMMs (gemm_tc.cuh k_gemm_p / p2).
#include "gemm_tc.cuh"
#include "kernel_ptrs.h"

namespace rw {

template <bool AMN, bool BMN>
static void* p_ptr(int bn, bool two) {
  if (two) return bn == 256 ? (void*)k_gemm_p2<AMN, BMN, 256> : (void*)k_gemm_p2<AMN, BMN, 128>;
  return bn == 256 ? (void*)k_gemm_p<AMN, BMN, 256> : (void*)k_gemm_p<AMN, BMN, 128>;
}
static void* p_sel(bool amn, bool bmn, int bn, bool two) {
  if (amn) return bmn ? p_ptr<true, true>(bn, two) : p_ptr<true, false>(bn, two);
  return bmn ? p_ptr<false, true>(bn, two) : p_ptr<false, false>(bn, two);
}

void* gemm_p_ptr(bool amn, bool bmn, int bn) { return p_sel(amn, bmn, bn, false); }
void* gemm_p2_ptr(bool amn, bool bmn, int bn) { return p_sel(amn, bmn, bn, true); }

}  // namespace rw

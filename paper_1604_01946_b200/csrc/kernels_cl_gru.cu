// kernels_cl_gru.cu -- instantiations of the cluster-schedule recurrent kernels (rec_cluster.cuh) for the
// GRU (linear before reset) cell.
#include "kernel_ptrs.h"
#include "rec_cluster.cuh"

namespace rw {

template <class P>
static void* cl_ptr_gru(bool fwd, int nco) {
  switch (nco >> 4) {
    case 4: return fwd ? (void*)k_cl_fwd<P, 4, kCellGru> : (void*)k_cl_bwd<P, 4, kCellGru>;
    case 3: return fwd ? (void*)k_cl_fwd<P, 3, kCellGru> : (void*)k_cl_bwd<P, 3, kCellGru>;
    case 2: return fwd ? (void*)k_cl_fwd<P, 2, kCellGru> : (void*)k_cl_bwd<P, 2, kCellGru>;
    default: return fwd ? (void*)k_cl_fwd<P, 1, kCellGru> : (void*)k_cl_bwd<P, 1, kCellGru>;
  }
}

void* cl_kernel_ptr_gru(int prec, bool fwd, int nco) {
  return prec == kF16x2 ? cl_ptr_gru<PrecF16x2>(fwd, nco) : cl_ptr_gru<PrecBF16>(fwd, nco);
}

}  // namespace rw

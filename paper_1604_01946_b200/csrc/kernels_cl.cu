// kernels_cl.cu -- instantiations of the cluster-schedule recurrent kernels (rec_cluster.cuh).
#include "kernel_ptrs.h"
#include "rec_cluster.cuh"

namespace rw {

template <class P>
static void* cl_ptr(bool fwd, int nco) {
  switch (nco >> 4) {
    case 4: return fwd ? (void*)k_cl_fwd<P, 4> : (void*)k_cl_bwd<P, 4>;
    case 3: return fwd ? (void*)k_cl_fwd<P, 3> : (void*)k_cl_bwd<P, 3>;
    case 2: return fwd ? (void*)k_cl_fwd<P, 2> : (void*)k_cl_bwd<P, 2>;
    default: return fwd ? (void*)k_cl_fwd<P, 1> : (void*)k_cl_bwd<P, 1>;
  }
}

void* cl_kernel_ptr(int prec, bool fwd, int nco) {
  return prec == kF16x2 ? cl_ptr<PrecF16x2>(fwd, nco) : cl_ptr<PrecBF16>(fwd, nco);
}

}  // namespace rw

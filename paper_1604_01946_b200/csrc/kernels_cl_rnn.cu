// kernels_cl_rnn.cu -- instantiations of the cluster-schedule recurrent kernels (rec_cluster.cuh) for the
// vanilla RNN cell (tanh and relu share an instantiation: ClParams::kind).
#include "kernel_ptrs.h"
#include "rec_cluster.cuh"

namespace rw {

template <class P>
static void* cl_ptr_rnn(bool fwd, int nco) {
  switch (nco >> 4) {
    case 4: return fwd ? (void*)k_cl_fwd<P, 4, kCellRnnTanh> : (void*)k_cl_bwd<P, 4, kCellRnnTanh>;
    case 3: return fwd ? (void*)k_cl_fwd<P, 3, kCellRnnTanh> : (void*)k_cl_bwd<P, 3, kCellRnnTanh>;
    case 2: return fwd ? (void*)k_cl_fwd<P, 2, kCellRnnTanh> : (void*)k_cl_bwd<P, 2, kCellRnnTanh>;
    default: return fwd ? (void*)k_cl_fwd<P, 1, kCellRnnTanh> : (void*)k_cl_bwd<P, 1, kCellRnnTanh>;
  }
}

void* cl_kernel_ptr_rnn(int prec, bool fwd, int nco) {
  return prec == kF16x2 ? cl_ptr_rnn<PrecF16x2>(fwd, nco) : cl_ptr_rnn<PrecBF16>(fwd, nco);
}

}  // namespace rw

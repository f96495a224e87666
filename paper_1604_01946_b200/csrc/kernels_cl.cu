// kernels_cl.cu -- instantiations of the cluster-schedule recurrent kernels (rec_cluster.cuh) for the
// LSTM cell; cl_kernel_ptr dispatches on the cell kind.
#include "kernel_ptrs.h"
#include "rec_cluster.cuh"

namespace rw {

template <class P>
static void* cl_ptr_lstm(bool fwd, int nco) {
  switch (nco >> 4) {
    case 4: return fwd ? (void*)k_cl_fwd<P, 4, kCellLstm> : (void*)k_cl_bwd<P, 4, kCellLstm>;
    case 3: return fwd ? (void*)k_cl_fwd<P, 3, kCellLstm> : (void*)k_cl_bwd<P, 3, kCellLstm>;
    case 2: return fwd ? (void*)k_cl_fwd<P, 2, kCellLstm> : (void*)k_cl_bwd<P, 2, kCellLstm>;
    default: return fwd ? (void*)k_cl_fwd<P, 1, kCellLstm> : (void*)k_cl_bwd<P, 1, kCellLstm>;
  }
}

void* cl_kernel_ptr_lstm(int prec, bool fwd, int nco) {
  return prec == kF16x2 ? cl_ptr_lstm<PrecF16x2>(fwd, nco) : cl_ptr_lstm<PrecBF16>(fwd, nco);
}

void* cl_kernel_ptr(int prec, bool fwd, int nco, int kind) {
  if (kind == kCellGru) return cl_kernel_ptr_gru(prec, fwd, nco);
  if (kind == kCellRnnTanh || kind == kCellRnnRelu) return cl_kernel_ptr_rnn(prec, fwd, nco);
  return cl_kernel_ptr_lstm(prec, fwd, nco);
}

}  // namespace rw

// kernels_lstm.cu -- instantiations of the persistent / stepwise recurrent kernels (lstm_step.cuh).
#include "kernel_ptrs.h"
#include "lstm_step.cuh"

namespace rw {

void* lstm_kernel_ptr(int prec, bool fwd, bool pair, int kind) {
  if (kind != kCellLstm) return lstm_kernel_ptr_cells(prec, fwd, kind);  // (no CTA pairs)
  if (pair) return fwd ? (void*)k_lstm_fwd<PrecBF16, true> : (void*)k_lstm_bwd<PrecBF16, true>;
  if (prec == kBF16) return fwd ? (void*)k_lstm_fwd<PrecBF16> : (void*)k_lstm_bwd<PrecBF16>;
  if (prec == kF16x2) return fwd ? (void*)k_lstm_fwd<PrecF16x2> : (void*)k_lstm_bwd<PrecF16x2>;
  return fwd ? (void*)k_lstm_fwd<PrecTF32x3> : (void*)k_lstm_bwd<PrecTF32x3>;
}

}  // namespace rw

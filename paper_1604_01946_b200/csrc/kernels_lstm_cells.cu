// kernels_lstm_cells.cu -- the persistent / stepwise recurrent kernels (lstm_step.cuh) for the GRU
// and vanilla-RNN cells (kKind; tanh / relu selected at run time), bf16, fp16x2 and 3xTF32 operands.
#include "kernel_ptrs.h"
#include "lstm_step.cuh"

namespace rw {

void* lstm_kernel_ptr_cells(int prec, bool fwd, int kind) {
  const bool gru = kind == kCellGru;
  if (prec == kBF16) {
    if (gru) return fwd ? (void*)k_lstm_fwd<PrecBF16, false, kCellGru> : (void*)k_lstm_bwd<PrecBF16, false, kCellGru>;
    return fwd ? (void*)k_lstm_fwd<PrecBF16, false, kCellRnnTanh> : (void*)k_lstm_bwd<PrecBF16, false, kCellRnnTanh>;
  }
  if (prec == kTF32x3) {  // the layer-sequential schedule's fp32-parity operands
    if (gru) return fwd ? (void*)k_lstm_fwd<PrecTF32x3, false, kCellGru> : (void*)k_lstm_bwd<PrecTF32x3, false, kCellGru>;
    return fwd ? (void*)k_lstm_fwd<PrecTF32x3, false, kCellRnnTanh>
               : (void*)k_lstm_bwd<PrecTF32x3, false, kCellRnnTanh>;
  }
  if (gru) return fwd ? (void*)k_lstm_fwd<PrecF16x2, false, kCellGru> : (void*)k_lstm_bwd<PrecF16x2, false, kCellGru>;
  return fwd ? (void*)k_lstm_fwd<PrecF16x2, false, kCellRnnTanh> : (void*)k_lstm_bwd<PrecF16x2, false, kCellRnnTanh>;
}

}  // namespace rw

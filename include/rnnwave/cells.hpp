// rnnwave/cells.hpp -- the host-visible part of the cell layer of the drop-in facade: the
// FLOP convention (proj/include/rnnwave/cells.hpp:65-68) and the gate order. The pointwise
// cell math itself runs on the device, fused into the recurrent GEMM epilogues
// (paper_1604_01946_b200/csrc/lstm_step.cuh).
#pragma once

#include <cstdint>

#include "rnnwave/config.hpp"

namespace rnnwave {

// Gate row blocks of W, R, bias and the gates tape: LSTM i, f, o, c' (cells.hpp:24-28).
enum LstmGate : int { kGateI = 0, kGateF = 1, kGateO = 2, kGateC = 3 };

// cells.hpp:65-68 -- GEMM multiply-add FLOPs of one cell step.
inline std::int64_t flop_count(CellKind kind, int hidden, int input, int batch) {
  return 2ll * gate_count(kind) * hidden * (std::int64_t(input) + hidden) * batch;
}

}  // namespace rnnwave

// rnnwave/gemm.hpp -- the reference's free GEMM (proj/include/rnnwave/gemm.hpp:339-347) on the
// device: C = alpha op(A) op(B) + beta C over column-major spans, executed by librnnwave_sm100's
// tcgen05 GEMM with 3xTF32 split operands (rw_gemm). Same signatures, same dimension checks and
// messages (gemm.hpp:115-130); the result meets the fp32-parity tolerance, it is not bitwise the
// reference's ordered CPU chain.
#pragma once

#include <stdexcept>
#include <string>

#include "rnnwave/matrix.hpp"
#include "rnnwave_sm100.h"

namespace rnnwave {

/// CPU cache-blocking sizes of the reference's tiled GEMM (gemm.hpp:27-31). The device GEMM tiles
/// for the tensor cores itself, so these select nothing; results are identical for every value,
/// which is the property the reference promises for its own tiles (gemm.hpp:20-25).
struct GemmTiles {
  int mc = 64;
  int nc = 64;
  int kc = 64;
};

inline void gemm(bool trans_a, bool trans_b, ConstSpan a, ConstSpan b, Span c, float alpha, float beta) {
  const int am = trans_a ? a.cols : a.rows;
  const int ak = trans_a ? a.rows : a.cols;
  const int bk = trans_b ? b.cols : b.rows;
  const int bn = trans_b ? b.rows : b.cols;
  if (ak != bk)
    throw std::invalid_argument("gemm: op(A) is " + std::to_string(am) + "x" + std::to_string(ak) + " but op(B) is " +
                                std::to_string(bk) + "x" + std::to_string(bn) + "; inner dimensions differ");
  if (c.rows != am || c.cols != bn)
    throw std::invalid_argument("gemm: C is " + std::to_string(c.rows) + "x" + std::to_string(c.cols) +
                                " but op(A)*op(B) is " + std::to_string(am) + "x" + std::to_string(bn));
  if (c.rows == 0 || c.cols == 0) return;
  const int st = rw_gemm(trans_a ? 1 : 0, trans_b ? 1 : 0, am, bn, ak, alpha, a.data, a.ld > 0 ? a.ld : 1, b.data,
                         b.ld > 0 ? b.ld : 1, beta, c.data, c.ld);
  if (st == RW_EINVAL) throw std::invalid_argument(rw_last_error(nullptr));
  if (st != RW_OK) throw std::runtime_error(rw_last_error(nullptr));
}

/// gemm.hpp:254-337 (the reference's entry point with explicit tiles).
inline void gemm_tiled(bool trans_a, bool trans_b, ConstSpan a, ConstSpan b, Span c, float alpha, float beta,
                       const GemmTiles&) {
  gemm(trans_a, trans_b, a, b, c, alpha, beta);
}

/// op(A) * B convenience with op(B) = B (gemm.hpp:344-347).
inline void gemm(bool trans_a, ConstSpan a, ConstSpan b, Span c, float alpha, float beta) {
  gemm(trans_a, false, a, b, c, alpha, beta);
}

}  // namespace rnnwave

// rnnwave/cells.hpp -- the cell layer of the drop-in facade: the FLOP convention
// (proj/include/rnnwave/cells.hpp:65-68), the gate order, and the free pointwise stage
// (pointwise_forward cells.hpp:181-333, pointwise_backward 349-562) with the reference's
// signatures, dimension checks and messages, executed on the device by librnnwave_sm100
// (rw_pointwise_forward / rw_pointwise_backward, csrc/pointwise.cuh). Inside the engine the same
// math is fused into the recurrent kernels' epilogues; these entry points serve callers of the
// free functions (the reference's own tests/test_cells.cpp compiles against this header).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rnnwave/config.hpp"
#include "rnnwave/matrix.hpp"
#include "rnnwave_sm100.h"

namespace rnnwave {

// Gate row blocks of W, R, bias and the gates tape: LSTM i, f, o, c' (cells.hpp:24-28).
enum LstmGate : int { kGateI = 0, kGateF = 1, kGateO = 2, kGateC = 3 };

inline float sigmoid_scalar(float x) { return 1.0f / (1.0f + std::exp(-x)); }

/// Views into the tape slots for one step (cells.hpp:32-43).
struct CellSavedSlices {
  Span gates;   // post-activation gates, G*H x B
  Span tanh_c;  // tanh(c_t), LSTM only
  Span zr_h;    // R_h * h_prev block, GRU only
};

struct CellSavedConst {
  ConstSpan gates;
  ConstSpan tanh_c;
  ConstSpan zr_h;
};

/// Scratch of the reference's host loops (cells.hpp:45-60); the device keeps its own, so this is
/// only sized for signature compatibility.
struct CellWorkspace {
  Matrix pre, gates_scratch, t1, t2, t3, t4;
  void ensure(CellKind, int, int) {}
};

// cells.hpp:65-68 -- GEMM multiply-add FLOPs of one cell step.
inline std::int64_t flop_count(CellKind kind, int hidden, int input, int batch) {
  return 2ll * gate_count(kind) * hidden * (std::int64_t(input) + hidden) * batch;
}

namespace detail {

inline void check_dims(ConstSpan s, int rows, int cols, const char* what) {
  if (s.rows != rows || s.cols != cols)
    throw std::invalid_argument(std::string("cells: ") + what + " is " + std::to_string(s.rows) + "x" +
                                std::to_string(s.cols) + ", expected " + std::to_string(rows) + "x" +
                                std::to_string(cols));
}

// dense column-major copies of (possibly strided) views; empty views give nullptr
struct Dense {
  std::vector<float> v;
  const float* in(ConstSpan s) {
    if (!s.data) return nullptr;
    v.resize(std::size_t(s.rows) * s.cols);
    for (int c = 0; c < s.cols; ++c)
      for (int r = 0; r < s.rows; ++r) v[std::size_t(c) * s.rows + r] = s.at(r, c);
    return v.data();
  }
  float* out(Span s) {
    if (!s.data) return nullptr;
    v.assign(std::size_t(s.rows) * s.cols, 0.0f);
    return v.data();
  }
  void back(Span s) const {
    if (!s.data) return;
    for (int c = 0; c < s.cols; ++c)
      for (int r = 0; r < s.rows; ++r) s.at(r, c) = v[std::size_t(c) * s.rows + r];
  }
};

inline void check_status(int st) {
  if (st == RW_EINVAL) throw std::invalid_argument(rw_last_error(nullptr));
  if (st != RW_OK) throw std::runtime_error(rw_last_error(nullptr));
}

}  // namespace detail

inline void pointwise_forward(CellKind kind, bool fused, ConstSpan zw, ConstSpan zr, const float* bias,
                              ConstSpan h_prev, ConstSpan c_prev, Span h_out, Span c_out,
                              const CellSavedSlices* save, CellWorkspace& ws) {
  const int hidden = h_prev.rows, batch = h_prev.cols, gates = gate_count(kind);
  detail::check_dims(zw, gates * hidden, batch, "zw");
  detail::check_dims(zr, gates * hidden, batch, "zr");
  detail::check_dims(ConstSpan(h_out), hidden, batch, "h_out");
  if (kind == CellKind::Lstm) {
    detail::check_dims(c_prev, hidden, batch, "c_prev");
    detail::check_dims(ConstSpan(c_out), hidden, batch, "c_out");
  } else if (!c_prev.empty()) {
    throw std::invalid_argument("cells: cell state supplied for a cell kind without one");
  }
  ws.ensure(kind, hidden, batch);
  const bool rnn = kind == CellKind::RnnTanh || kind == CellKind::RnnRelu;
  detail::Dense zw_d, zr_d, hp_d, cp_d, h_d, c_d, g_d, tc_d, zh_d;
  const Span none{};
  const Span g_s = save && !rnn ? save->gates : none;
  const Span tc_s = save && kind == CellKind::Lstm ? save->tanh_c : none;
  const Span zh_s = save && kind == CellKind::Gru ? save->zr_h : none;
  detail::check_status(rw_pointwise_forward(
      static_cast<int>(kind), fused ? 1 : 0, hidden, batch, zw_d.in(zw), zr_d.in(zr), bias, hp_d.in(h_prev),
      cp_d.in(c_prev), h_d.out(h_out), c_d.out(c_out), g_d.out(g_s), tc_d.out(tc_s), zh_d.out(zh_s)));
  h_d.back(h_out);
  c_d.back(c_out);
  g_d.back(g_s);
  tc_d.back(tc_s);
  zh_d.back(zh_s);
}

// dgw / dgr: W-side / R-side pre-activation gradients (dgr distinct from dgw only for GRU;
// callers may alias the two for LSTM / RNN), dh_local: the direct h_prev term, dc_prev: LSTM
// cell-state carry, db: optional G*H accumulator (cells.hpp:336-348).
inline void pointwise_backward(CellKind kind, bool fused, const CellSavedConst& saved, ConstSpan h_prev,
                               ConstSpan c_prev, ConstSpan d_above, ConstSpan dh_carry, ConstSpan dc_carry, Span dgw,
                               Span dgr, Span dh_local, Span dc_prev, float* db, CellWorkspace& ws) {
  const int hidden = d_above.rows, batch = d_above.cols, gates = gate_count(kind);
  detail::check_dims(ConstSpan(dgw), gates * hidden, batch, "dgw");
  detail::check_dims(dh_carry, hidden, batch, "dh_carry");
  detail::check_dims(ConstSpan(dh_local), hidden, batch, "dh_local");
  if (saved.gates.empty()) throw std::invalid_argument("cells: backward requires saved state from a training forward");
  ws.ensure(kind, hidden, batch);
  const Span none{};
  if (kind == CellKind::Lstm) {
    detail::check_dims(dc_carry, hidden, batch, "dc_carry");
    detail::check_dims(ConstSpan(dc_prev), hidden, batch, "dc_prev");
  }
  if (kind == CellKind::Gru) {
    if (dgr.data == dgw.data) throw std::invalid_argument("cells: GRU needs distinct dgw and dgr blocks");
    detail::check_dims(ConstSpan(dgr), gates * hidden, batch, "dgr");
  }
  const bool lstm = kind == CellKind::Lstm, gru = kind == CellKind::Gru;
  detail::Dense g_d, tc_d, zh_d, hp_d, cp_d, da_d, hc_d, cc_d, dgw_d, dgr_d, dhl_d, dcp_d;
  const Span dgr_s = gru ? dgr : none, dcp_s = lstm ? dc_prev : none;
  detail::check_status(rw_pointwise_backward(
      static_cast<int>(kind), fused ? 1 : 0, hidden, batch, g_d.in(saved.gates), lstm ? tc_d.in(saved.tanh_c) : nullptr,
      gru ? zh_d.in(saved.zr_h) : nullptr, gru ? hp_d.in(h_prev) : nullptr, lstm ? cp_d.in(c_prev) : nullptr,
      da_d.in(d_above), hc_d.in(dh_carry), lstm ? cc_d.in(dc_carry) : nullptr, dgw_d.out(dgw), dgr_d.out(dgr_s),
      dhl_d.out(dh_local), dcp_d.out(dcp_s), db));
  dgw_d.back(dgw);
  dgr_d.back(dgr_s);
  dhl_d.back(dh_local);
  dcp_d.back(dcp_s);
}

}  // namespace rnnwave

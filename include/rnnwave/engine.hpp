// rnnwave/engine.hpp -- drop-in facade of rnnwave::Engine over librnnwave_sm100.so.
//
// Keeps the reference's public signatures (proj/include/rnnwave/engine.hpp:36-217):
//   explicit Engine(const LadderConfig&)                       (+ optional device knobs)
//   const LadderConfig& config() const;  void set_trace_sink(sched::ScheduleTrace*)
//   ForwardResult forward(std::vector<LayerParams>&, const Matrix& x, bool training,
//                         const std::vector<Matrix>* h0 = nullptr, const std::vector<Matrix>* c0 = nullptr)
//   BackwardState backward_data(std::vector<LayerParams>&, const ForwardTape&, const Matrix& dy)
//   Gradients     weight_update(const ForwardTape&, const BackwardState&)
// and the value types' field names (ForwardTape::x0/h_seq/c_seq/gates_seq/tanh_c_seq,
// BackwardState::dx0/dgw_seq/dh0/dc0, Gradients::dw/dr/db/dx0). The tape tensors live in
// HBM; the facade materialises a tape field on first access (verify.hpp reads
// tape.h_seq[l] / bwd.dgw_seq[l] directly), so the device-resident path stays free of
// host copies. Errors: RW_EINVAL -> std::invalid_argument (same message substrings as the
// reference: "expected", "training", "stale tape"), anything else -> std::runtime_error.
//
// Link with -L<repo>/paper_1604_01946_b200/lib -lrnnwave_sm100.
#pragma once

#include <cstddef>
#include <cstdint>
#include <iterator>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "rnnwave/cells.hpp"
#include "rnnwave/config.hpp"
#include "rnnwave/gemm.hpp"
#include "rnnwave/matrix.hpp"
#include "rnnwave/params.hpp"
#include "rnnwave/trace.hpp"
#include "rnnwave_sm100.h"

namespace rnnwave {

namespace detail {

[[noreturn]] inline void raise(int status, const std::string& msg) {
  if (status == RW_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// Owns the device context; shared by the Engine and every tape/state it hands out.
struct DeviceHandle {
  rw_ctx* ctx = nullptr;
  std::uint64_t fwd_tape = 0;  // the forward tape the device holds (rw_forward's id)
  std::uint64_t bwd_tape = 0;  // the tape whose backward state (dG) the device holds
  ~DeviceHandle() {
    if (ctx) rw_destroy(ctx);
  }
  void check(int status) const {
    if (status != RW_OK) raise(status, rw_last_error(ctx));
  }
};

// Per-layer tape tensor sequence, materialised from HBM on first access. Like the reference's
// std::vector<Matrix> fields it is indexable and iterable (range-for). A field first read after
// the device moved on to a newer tape throws "stale tape" (the reference's value-type tapes keep
// their data; here the data lives on the device until the next forward / backward).
class TapeSeq {
 public:
  TapeSeq() = default;
  TapeSeq(std::shared_ptr<DeviceHandle> h, std::uint64_t id, int which, int n, int rows, int cols)
      : h_(std::move(h)), id_(id), which_(which), rows_(rows), cols_(cols), cache_(n) {}
  std::size_t size() const { return cache_.size(); }
  bool empty() const { return cache_.empty(); }
  const Matrix& operator[](std::size_t l) const {
    if (l >= cache_.size()) throw std::out_of_range("tape: layer index out of range");
    if (!cache_[l]) {
      const std::uint64_t held = (which_ == RW_TAPE_DGW || which_ == RW_TAPE_DGR) ? h_->bwd_tape : h_->fwd_tape;
      if (held != id_)
        throw std::invalid_argument("engine: stale tape, the device no longer holds tape " + std::to_string(id_));
      Matrix m(rows_, cols_);
      h_->check(rw_get_tape(h_->ctx, which_, int(l), m.data()));
      cache_[l] = std::move(m);
    }
    return *cache_[l];
  }
  const Matrix& at(std::size_t l) const { return (*this)[l]; }
  const Matrix& back() const { return (*this)[cache_.size() - 1]; }
  const Matrix& front() const { return (*this)[0]; }
  std::uint64_t id() const { return id_; }

  class const_iterator {
   public:
    using value_type = Matrix;
    using reference = const Matrix&;
    using pointer = const Matrix*;
    using difference_type = std::ptrdiff_t;
    using iterator_category = std::forward_iterator_tag;
    const_iterator(const TapeSeq* s, std::size_t i) : s_(s), i_(i) {}
    reference operator*() const { return (*s_)[i_]; }
    pointer operator->() const { return &(*s_)[i_]; }
    const_iterator& operator++() {
      ++i_;
      return *this;
    }
    const_iterator operator++(int) {
      const_iterator o = *this;
      ++i_;
      return o;
    }
    bool operator==(const const_iterator& o) const { return s_ == o.s_ && i_ == o.i_; }
    bool operator!=(const const_iterator& o) const { return !(*this == o); }

   private:
    const TapeSeq* s_;
    std::size_t i_;
  };
  const_iterator begin() const { return const_iterator(this, 0); }
  const_iterator end() const { return const_iterator(this, cache_.size()); }

 private:
  std::shared_ptr<DeviceHandle> h_;
  std::uint64_t id_ = 0;
  int which_ = 0, rows_ = 0, cols_ = 0;
  mutable std::vector<std::optional<Matrix>> cache_;
};

}  // namespace detail

struct ForwardTape {
  LadderConfig cfg;
  bool training = false;
  Matrix x0;
  detail::TapeSeq h_seq;
  detail::TapeSeq c_seq;
  detail::TapeSeq gates_seq;
  detail::TapeSeq tanh_c_seq;
  detail::TapeSeq zrh_seq;      // GRU only (engine.hpp:44)
  std::shared_ptr<detail::DeviceHandle> device;
  std::uint64_t id = 0;
};

struct ForwardResult {
  Matrix y;
  ForwardTape tape;
};

struct BackwardState {
  Matrix dx0;
  detail::TapeSeq dgw_seq;
  detail::TapeSeq dgr_seq;      // GRU only (engine.hpp:57)
  std::vector<Matrix> dh0;
  std::vector<Matrix> dc0;
  std::uint64_t id = 0;
};

struct Gradients {
  std::vector<Matrix> dw;
  std::vector<Matrix> dr;
  std::vector<std::vector<float>> db;
  Matrix dx0;
};

class Engine {
 public:
  // precision: RW_PREC_FP32 (3xTF32 fp32-parity, default) or RW_PREC_BF16; the environment
  // variable RNNWAVE_PRECISION=bf16|fp32 overrides the default for unmodified callers.
  explicit Engine(const LadderConfig& cfg, int precision = -1, int schedule = RW_SCHED_AUTO,
                  int device = 0)
      : cfg_(cfg), dev_(std::make_shared<detail::DeviceHandle>()) {
    cfg_.validate();
    if (precision < 0) {
      precision = RW_PREC_FP32;
      if (const char* e = std::getenv("RNNWAVE_PRECISION"))
        if (std::strcmp(e, "bf16") == 0) precision = RW_PREC_BF16;
    }
    rw_config c{};
    c.layers = cfg_.layers;
    c.hidden = cfg_.hidden;
    c.input = cfg_.input;
    c.batch = cfg_.batch;
    c.steps = cfg_.steps;
    c.cell_kind = int(cfg_.kind);
    c.opt_level = cfg_.opt_level;
    c.batch_steps = cfg_.batch_steps;
    c.workers = cfg_.workers;
    c.seed = cfg_.seed;
    c.precision = precision;
    c.schedule = schedule;
    const int st = rw_create(&c, device, &dev_->ctx);
    if (st != RW_OK) detail::raise(st, rw_create_error());
  }

  const LadderConfig& config() const { return cfg_; }
  // engine.hpp:79-80: when set, every forward / backward_data deposits its schedule trace here
  // (the device's per-step tasks, build_graph(L, T, 1) ids; rw_trace_records).
  void set_trace_sink(sched::ScheduleTrace* sink) {
    trace_sink_ = sink;
    dev_->check(rw_trace_enable(dev_->ctx, sink ? 1 : 0));
  }

  ForwardResult forward(std::vector<LayerParams>& params, const Matrix& x, bool training,
                        const std::vector<Matrix>* h0 = nullptr,
                        const std::vector<Matrix>* c0 = nullptr) {
    upload(params);
    const int bt = cfg_.batch * cfg_.steps;
    if (x.rows() != cfg_.input || x.cols() != bt)
      throw std::invalid_argument("forward: x is " + std::to_string(x.rows()) + "x" +
                                  std::to_string(x.cols()) + ", expected " +
                                  std::to_string(cfg_.input) + "x" + std::to_string(bt));
    if (cfg_.opt_level >= 4) pretranspose(params);
    std::vector<const float*> ph0, pc0;
    if (h0) {
      if (int(h0->size()) != cfg_.layers)
        throw std::invalid_argument("forward: h0 must supply one matrix per layer");
      for (const Matrix& m : *h0) ph0.push_back(m.data());
    }
    if (c0) {
      if (cfg_.kind != CellKind::Lstm)
        throw std::invalid_argument("forward: c0 supplied for a cell kind without cell state");
      if (int(c0->size()) != cfg_.layers)
        throw std::invalid_argument("forward: c0 must supply one matrix per layer");
      for (const Matrix& m : *c0) pc0.push_back(m.data());
    }
    ForwardResult res;
    res.y = Matrix(cfg_.hidden, bt);
    std::uint64_t id = 0;
    dev_->check(rw_forward(dev_->ctx, x.data(), training ? 1 : 0, h0 ? ph0.data() : nullptr,
                           c0 ? pc0.data() : nullptr, res.y.data(), &id));
    dev_->fwd_tape = id;
    deposit_trace(0);
    ForwardTape& t = res.tape;
    t.cfg = cfg_;
    t.training = training;
    t.x0 = x;
    t.device = dev_;
    t.id = id;
    const int H = cfg_.hidden, L = cfg_.layers;
    const int G = gate_count(cfg_.kind);
    const bool lstm = cfg_.kind == CellKind::Lstm, gru = cfg_.kind == CellKind::Gru;
    t.h_seq = detail::TapeSeq(dev_, id, RW_TAPE_H, L, H, cfg_.batch + bt);
    if (lstm) t.c_seq = detail::TapeSeq(dev_, id, RW_TAPE_C, L, H, cfg_.batch + bt);  // engine.hpp:264
    if (training) {
      t.gates_seq = detail::TapeSeq(dev_, id, RW_TAPE_GATES, L, G * H, bt);
      if (lstm) t.tanh_c_seq = detail::TapeSeq(dev_, id, RW_TAPE_TANH_C, L, H, bt);
      if (gru) t.zrh_seq = detail::TapeSeq(dev_, id, RW_TAPE_ZRH, L, H, bt);
    }
    return res;
  }

  BackwardState backward_data(std::vector<LayerParams>& params, const ForwardTape& tape,
                              const Matrix& dy) {
    upload(params);
    check_tape(tape);
    const int bt = cfg_.batch * cfg_.steps;
    if (dy.rows() != cfg_.hidden || dy.cols() != bt)
      throw std::invalid_argument("backward_data: dy is " + std::to_string(dy.rows()) + "x" +
                                  std::to_string(dy.cols()) + ", expected " +
                                  std::to_string(cfg_.hidden) + "x" + std::to_string(bt));
    if (cfg_.opt_level >= 4) pretranspose(params);
    BackwardState s;
    s.dx0 = Matrix(cfg_.input, bt);
    std::vector<float*> pdh, pdc;
    for (int l = 0; l < cfg_.layers; ++l) {
      s.dh0.emplace_back(cfg_.hidden, cfg_.batch);
      if (cfg_.kind == CellKind::Lstm) s.dc0.emplace_back(cfg_.hidden, cfg_.batch);  // engine.hpp:318
    }
    for (int l = 0; l < cfg_.layers; ++l) {
      pdh.push_back(s.dh0[l].data());
      if (cfg_.kind == CellKind::Lstm) pdc.push_back(s.dc0[l].data());
    }
    dev_->check(rw_backward_data(dev_->ctx, tape.id, dy.data(), s.dx0.data(), pdh.data(),
                                 pdc.empty() ? nullptr : pdc.data()));
    dev_->bwd_tape = tape.id;
    deposit_trace(1);
    const int gh = gate_count(cfg_.kind) * cfg_.hidden;
    s.dgw_seq = detail::TapeSeq(dev_, tape.id, RW_TAPE_DGW, cfg_.layers, gh, bt);
    if (cfg_.kind == CellKind::Gru) s.dgr_seq = detail::TapeSeq(dev_, tape.id, RW_TAPE_DGR, cfg_.layers, gh, bt);
    s.id = tape.id;
    return s;
  }

  Gradients weight_update(const ForwardTape& tape, const BackwardState& state) {
    check_tape(tape);
    if (int(state.dgw_seq.size()) != cfg_.layers || state.id != tape.id)
      throw std::invalid_argument("weight_update: backward state layer count mismatch");
    Gradients g;
    std::vector<float*> pw, pr, pb;
    for (int l = 0; l < cfg_.layers; ++l) {
      const int gh = gate_count(cfg_.kind) * cfg_.hidden;
      g.dw.emplace_back(gh, cfg_.input_width(l));
      g.dr.emplace_back(gh, cfg_.hidden);
      g.db.emplace_back(std::size_t(gh), 0.0f);
    }
    for (int l = 0; l < cfg_.layers; ++l) {
      pw.push_back(g.dw[l].data());
      pr.push_back(g.dr[l].data());
      pb.push_back(g.db[l].data());
    }
    dev_->check(rw_weight_update(dev_->ctx, tape.id, pw.data(), pr.data(), pb.data()));
    g.dx0 = state.dx0;
    return g;
  }

 private:
  void deposit_trace(int direction) {
    if (!trace_sink_) return;
    int n = 0;
    dev_->check(rw_trace_records(dev_->ctx, direction, nullptr, 0, &n));
    std::vector<rw_trace_record> r(static_cast<std::size_t>(n));
    dev_->check(rw_trace_records(dev_->ctx, direction, r.data(), n, &n));
    trace_sink_->clear();
    for (const rw_trace_record& t : r) {
      sched::TraceRecord o;
      o.task_id = t.task_id;
      o.layer = t.layer;
      o.block = t.block;
      o.step_k = t.step_k;
      o.phase = t.phase == 0 ? sched::TaskPhase::InputGemm : sched::TaskPhase::RecurrentStep;
      o.worker = t.worker;
      o.start_ns = t.start_ns;
      o.end_ns = t.end_ns;
      trace_sink_->push_back(o);
    }
  }

  void upload(const std::vector<LayerParams>& params) {
    if (int(params.size()) != cfg_.layers)
      throw std::invalid_argument("engine: expected " + std::to_string(cfg_.layers) +
                                  " layer parameter sets, got " + std::to_string(params.size()));
    const int gh = gate_count(cfg_.kind) * cfg_.hidden;
    for (int l = 0; l < cfg_.layers; ++l) {
      const LayerParams& p = params[l];
      if (p.w.rows() != gh || p.w.cols() != cfg_.input_width(l) || p.r.rows() != gh ||
          p.r.cols() != cfg_.hidden || int(p.bias.size()) != gh)
        throw std::invalid_argument("engine: layer " + std::to_string(l) +
                                    " parameter shapes do not match the configuration");
      dev_->check(rw_set_params(dev_->ctx, l, p.w.data(), p.r.data(), p.bias.data()));
    }
  }

  void check_tape(const ForwardTape& tape) const {
    if (!tape.training) throw std::invalid_argument("engine: tape was recorded without training mode");
    const LadderConfig& t = tape.cfg;
    if (t.layers != cfg_.layers || t.hidden != cfg_.hidden || t.input != cfg_.input ||
        t.batch != cfg_.batch || t.steps != cfg_.steps || t.kind != cfg_.kind)
      throw std::invalid_argument("engine: stale tape, network dimensions differ");
    if (tape.device != dev_)
      throw std::invalid_argument("engine: stale tape, recorded by another engine");
  }

  LadderConfig cfg_;
  std::shared_ptr<detail::DeviceHandle> dev_;
  sched::ScheduleTrace* trace_sink_ = nullptr;
};

}  // namespace rnnwave

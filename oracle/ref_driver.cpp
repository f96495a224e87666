// ref_driver.cpp -- C shim over the UNMODIFIED reference engine (TEST INFRASTRUCTURE ONLY).
//
// Compiled against the read-only reference headers at /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/librwref_*.so (git-ignored, travels to the GPU box
// with the snapshot). No reference source is copied: this file only calls the
// reference's public API -- rnnwave::Engine (engine.hpp:69-217), init_params
// (params.hpp:31-51), verify::make_input/make_dy (verify.hpp:38-44), the fp64
// oracle (oracle.hpp:72-424) and bench::time_level (bench.hpp:128-174).
// It is the north-star comparator for the GPU parity tests and the `--impl reference`
// CPU arm of bench.py. The product library never links it.

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "rnnwave/bench.hpp"
#include "rnnwave/engine.hpp"
#include "rnnwave/oracle.hpp"
#include "rnnwave/verify.hpp"

using namespace rnnwave;

namespace {

// cfg[] = {layers, hidden, input, batch, steps, opt_level, batch_steps, workers, kind}
// (kind: the reference's CellKind order -- 0 rnn-tanh, 1 rnn-relu, 2 gru, 3 lstm)
LadderConfig make_cfg(const int* c, std::uint64_t seed) {
  LadderConfig cfg;
  cfg.kind = static_cast<CellKind>(c[8]);
  cfg.layers = c[0];
  cfg.hidden = c[1];
  cfg.input = c[2];
  cfg.batch = c[3];
  cfg.steps = c[4];
  cfg.opt_level = c[5];
  cfg.batch_steps = c[6];
  cfg.workers = c[7];
  cfg.seed = seed;
  return cfg;
}

void put(const Matrix& m, float* dst) {
  if (dst) std::memcpy(dst, m.data(), m.size() * sizeof(float));
}

Matrix get(const float* src, int rows, int cols) {
  Matrix m(rows, cols);
  std::memcpy(m.data(), src, m.size() * sizeof(float));
  return m;
}

int fail(const std::exception& e, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), static_cast<std::size_t>(errlen - 1));
    err[errlen - 1] = '\0';
  }
  return 1;
}

}  // namespace

extern "C" {

int rwref_init_params(const int* c, std::uint64_t seed, float* const* w, float* const* r) {
  const LadderConfig cfg = make_cfg(c, seed);
  std::vector<LayerParams> p = init_params(cfg);
  for (int l = 0; l < cfg.layers; ++l) {
    put(p[l].w, w[l]);
    put(p[l].r, r[l]);
  }
  return 0;
}

int rwref_make_input(const int* c, std::uint64_t seed, float* x, float* dy) {
  const LadderConfig cfg = make_cfg(c, seed);
  if (x) put(verify::make_input(cfg), x);
  if (dy) put(verify::make_dy(cfg), dy);
  return 0;
}

long long rwref_flop_count_cell(int hidden, int input, int batch) {
  return static_cast<long long>(flop_count(CellKind::Lstm, hidden, input, batch));
}

// Full pipeline through the reference Engine: forward(training) and, when dy is given,
// backward_data + weight_update. Every output pointer may be null.
int rwref_run(const int* c, std::uint64_t seed, const float* const* w, const float* const* r,
              const float* const* b, const float* x, const float* const* h0,
              const float* const* c0, const float* dy, int training, float* y,
              float* const* h_seq, float* const* c_seq, float* const* gates_seq,
              float* const* tanh_c_seq, float* const* dgw_seq, float* dx0, float* const* dh0,
              float* const* dc0, float* const* dw, float* const* dr, float* const* db,
              char* err, int errlen) {
  try {
    const LadderConfig cfg = make_cfg(c, seed);
    const int H = cfg.hidden, B = cfg.batch, T = cfg.steps, G = gate_count(cfg.kind) * H;
    std::vector<LayerParams> params(cfg.layers);
    for (int l = 0; l < cfg.layers; ++l) {
      params[l].w = get(w[l], G, cfg.input_width(l));
      params[l].r = get(r[l], G, H);
      params[l].bias.assign(b[l], b[l] + G);
    }
    std::vector<Matrix> mh0, mc0;
    if (h0) for (int l = 0; l < cfg.layers; ++l) mh0.push_back(get(h0[l], H, B));
    if (c0) for (int l = 0; l < cfg.layers; ++l) mc0.push_back(get(c0[l], H, B));
    Engine engine(cfg);
    const Matrix xm = get(x, cfg.input, B * T);
    ForwardResult fwd = engine.forward(params, xm, training != 0 || dy != nullptr,
                                       h0 ? &mh0 : nullptr, c0 ? &mc0 : nullptr);
    put(fwd.y, y);
    for (int l = 0; l < cfg.layers; ++l) {
      if (h_seq) put(fwd.tape.h_seq[l], h_seq[l]);
      if (c_seq && !fwd.tape.c_seq.empty()) put(fwd.tape.c_seq[l], c_seq[l]);
      if (gates_seq && !fwd.tape.gates_seq.empty()) put(fwd.tape.gates_seq[l], gates_seq[l]);
      if (tanh_c_seq && !fwd.tape.tanh_c_seq.empty()) put(fwd.tape.tanh_c_seq[l], tanh_c_seq[l]);
    }
    if (!dy) return 0;
    const Matrix dym = get(dy, H, B * T);
    BackwardState bwd = engine.backward_data(params, fwd.tape, dym);
    Gradients grads = engine.weight_update(fwd.tape, bwd);
    put(bwd.dx0, dx0);
    for (int l = 0; l < cfg.layers; ++l) {
      if (dgw_seq) put(bwd.dgw_seq[l], dgw_seq[l]);
      if (dh0) put(bwd.dh0[l], dh0[l]);
      if (dc0 && !bwd.dc0.empty()) put(bwd.dc0[l], dc0[l]);
      if (dw) put(grads.dw[l], dw[l]);
      if (dr) put(grads.dr[l], dr[l]);
      if (db) std::memcpy(db[l], grads.db[l].data(), grads.db[l].size() * sizeof(float));
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// fp64 scalar oracle (oracle.hpp:72-424) on the same float parameters: y (H x BT), and
// when dy is given dW/dR/db/dx0/dh0/dc0, all as doubles.
int rwref_oracle(const int* c, const float* const* w, const float* const* r,
                 const float* const* b, const float* x, const float* dy, double* y,
                 double* const* dw, double* const* dr, double* const* db, double* dx0,
                 double* const* dh0, double* const* dc0, char* err, int errlen) {
  try {
    const LadderConfig cfg = make_cfg(c, 0);
    const int H = cfg.hidden, B = cfg.batch, T = cfg.steps, G = gate_count(cfg.kind) * H;
    std::vector<LayerParams> params(cfg.layers);
    for (int l = 0; l < cfg.layers; ++l) {
      params[l].w = get(w[l], G, cfg.input_width(l));
      params[l].r = get(r[l], G, H);
      params[l].bias.assign(b[l], b[l] + G);
    }
    const oracle::Net net = oracle::widen(cfg, params);
    const Matrix xm = get(x, cfg.input, B * T);
    const oracle::Activations acts = oracle::forward(net, xm, B, T);
    if (y) std::memcpy(y, acts.y.data(), acts.y.size() * sizeof(double));
    if (!dy) return 0;
    const Matrix dym = get(dy, H, B * T);
    const oracle::GradientResult g = oracle::gradient(net, xm, dym, B, T);
    for (int l = 0; l < cfg.layers; ++l) {
      std::memcpy(dw[l], g.dw[l].data(), g.dw[l].size() * sizeof(double));
      std::memcpy(dr[l], g.dr[l].data(), g.dr[l].size() * sizeof(double));
      std::memcpy(db[l], g.db[l].data(), g.db[l].size() * sizeof(double));
      if (dh0) std::memcpy(dh0[l], g.dh0[l].data(), g.dh0[l].size() * sizeof(double));
      if (dc0) std::memcpy(dc0[l], g.dc0[l].data(), g.dc0[l].size() * sizeof(double));
    }
    if (dx0) std::memcpy(dx0, g.dx0.data(), g.dx0.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// bench::time_level (bench.hpp:128-174) at the given level/workers.
// pass: 0 = fwd (inference), 1 = bwd (backward_data + weight_update), 2 = both.
int rwref_time(const int* c, std::uint64_t seed, int pass, int reps, int warmup,
               double* median_us, double* mean_us, double* min_us, char* err, int errlen) {
  try {
    const LadderConfig cfg = make_cfg(c, seed);
    const bench::PassKind kind = pass == 0   ? bench::PassKind::Forward
                                 : pass == 1 ? bench::PassKind::Backward
                                             : bench::PassKind::Both;
    const auto s = bench::time_level(cfg, kind, reps, warmup, nullptr);
    if (median_us) *median_us = s.median_us;
    if (mean_us) *mean_us = s.mean_us;
    if (min_us) *min_us = s.min_us;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// The reference's free pointwise stage (cells.hpp:181 pointwise_forward, 349
// pointwise_backward) on dense column-major buffers (ld = rows); null save / optional pointers
// as in the reference (gates == nullptr: inference). kind: CellKind.
int rwref_pointwise_forward(int kind, int fused, int hidden, int batch, const float* zw, const float* zr,
                            const float* bias, const float* h_prev, const float* c_prev, float* h_out,
                            float* c_out, float* gates, float* tanh_c, float* zr_h, char* err, int errlen) {
  try {
    const CellKind k = static_cast<CellKind>(kind);
    const int G = gate_count(k);
    auto cs = [](const float* p, int r, int c) { return ConstSpan(Span{const_cast<float*>(p), r, c, r}); };
    auto ms = [](float* p, int r, int c) { return p ? Span{p, r, c, r} : Span{}; };
    CellSavedSlices save;
    const bool rnn = k == CellKind::RnnTanh || k == CellKind::RnnRelu;
    save.gates = rnn ? ms(h_out, hidden, batch) : ms(gates, G * hidden, batch);
    save.tanh_c = ms(tanh_c, hidden, batch);
    save.zr_h = ms(zr_h, hidden, batch);
    CellWorkspace ws;
    pointwise_forward(k, fused != 0, cs(zw, G * hidden, batch), cs(zr, G * hidden, batch), bias,
                      cs(h_prev, hidden, batch), c_prev ? cs(c_prev, hidden, batch) : ConstSpan(),
                      ms(h_out, hidden, batch), ms(c_out, hidden, batch), gates || rnn ? &save : nullptr, ws);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

int rwref_pointwise_backward(int kind, int fused, int hidden, int batch, const float* gates, const float* tanh_c,
                             const float* zr_h, const float* h_prev, const float* c_prev, const float* d_above,
                             const float* dh_carry, const float* dc_carry, float* dgw, float* dgr, float* dh_local,
                             float* dc_prev, float* db, char* err, int errlen) {
  try {
    const CellKind k = static_cast<CellKind>(kind);
    const int G = gate_count(k);
    const bool rnn = k == CellKind::RnnTanh || k == CellKind::RnnRelu;
    auto cs = [](const float* p, int r, int c) {
      return p ? ConstSpan(Span{const_cast<float*>(p), r, c, r}) : ConstSpan();
    };
    auto ms = [](float* p, int r, int c) { return p ? Span{p, r, c, r} : Span{}; };
    CellSavedConst saved;
    saved.gates = cs(gates, rnn ? hidden : G * hidden, batch);
    saved.tanh_c = cs(tanh_c, hidden, batch);
    saved.zr_h = cs(zr_h, hidden, batch);
    CellWorkspace ws;
    pointwise_backward(k, fused != 0, saved, cs(h_prev, hidden, batch), cs(c_prev, hidden, batch),
                       cs(d_above, hidden, batch), cs(dh_carry, hidden, batch), cs(dc_carry, hidden, batch),
                       ms(dgw, G * hidden, batch), dgr ? ms(dgr, G * hidden, batch) : ms(dgw, G * hidden, batch),
                       ms(dh_local, hidden, batch), ms(dc_prev, hidden, batch), db, ws);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

}  // extern "C"

// facade_parity.cpp -- drop-in check of the C++ facade (include/rnnwave/engine.hpp).
//
// Written the way the reference's own tests use the API (test_engine.cpp, verify.hpp
// run_pipeline): init_params -> Engine::forward(training) -> backward_data ->
// weight_update, then reads tape fields (tape.h_seq[l], bwd.dgw_seq[l]) like
// verify::check_weight_update_equivalence does. The checker is the C restatement of the
// reference (oracle/lstm_oracle.c, linked as test infrastructure); tolerances are the
// SURVEY §8c rules. Exit 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "rnnwave/engine.hpp"

extern "C" {
#include "lstm_oracle.h"
}

using namespace rnnwave;

static int g_fail = 0;

static void check(const char* what, const float* got, const float* ref, std::size_t n,
                  double nw_tol, double sm_tol) {
  double dn = 0, rn = 0, dm = 0, rm = 0;
  for (std::size_t i = 0; i < n; ++i) {
    const double d = double(got[i]) - double(ref[i]);
    dn += d * d;
    rn += double(ref[i]) * ref[i];
    dm = std::max(dm, std::abs(d));
    rm = std::max(rm, std::abs(double(ref[i])));
  }
  const double nw = rn > 0 ? std::sqrt(dn / rn) : std::sqrt(dn);
  const double sm = rm > 0 ? dm / rm : dm;
  const bool ok = nw <= nw_tol && sm <= sm_tol;
  if (!ok) ++g_fail;
  std::printf("  %-10s normwise %.3e scaled-max %.3e %s\n", what, nw, sm, ok ? "ok" : "FAIL");
}

static void run(int precision, LadderConfig cfg) {
  const double nw_tol = precision == RW_PREC_FP32 ? 1e-5 : 1e-2;
  const double sm_tol = precision == RW_PREC_FP32 ? 1e-5 : 2e-2;
  std::printf("facade %s L%d H%d I%d B%d T%d\n", precision == RW_PREC_FP32 ? "fp32" : "bf16",
              cfg.layers, cfg.hidden, cfg.input, cfg.batch, cfg.steps);
  std::vector<LayerParams> params = init_params(cfg);
  for (int l = 0; l < cfg.layers; ++l) {
    SplitMix64 s = split_stream(cfg.seed, 300 + l);
    for (float& b : params[l].bias) b = s.next_symmetric(0.5);
  }
  Matrix x(cfg.input, cfg.batch * cfg.steps), dy(cfg.hidden, cfg.batch * cfg.steps);
  {
    SplitMix64 sx = split_stream(cfg.seed, 1000), sd = split_stream(cfg.seed, 1001);
    for (std::size_t i = 0; i < x.size(); ++i) x.data()[i] = sx.next_symmetric(1.0);
    for (std::size_t i = 0; i < dy.size(); ++i) dy.data()[i] = sd.next_symmetric(1.0);
  }
  Engine engine(cfg, precision);
  ForwardResult fwd = engine.forward(params, x, true);
  BackwardState bwd = engine.backward_data(params, fwd.tape, dy);
  Gradients g = engine.weight_update(fwd.tape, bwd);

  // checker: the C restatement of the reference engine
  const int L = cfg.layers, H = cfg.hidden, B = cfg.batch, T = cfg.steps, G = 4 * H;
  rwo_dims d{L, H, cfg.input, B, T};
  std::vector<std::vector<float>> hs(L, std::vector<float>(std::size_t(H) * B * (T + 1))),
      cs = hs, gs(L, std::vector<float>(std::size_t(G) * B * T)),
      ts(L, std::vector<float>(std::size_t(H) * B * T)), dg = gs, dh0(L, std::vector<float>(H * B)),
      dc0 = dh0, dw(L), dr(L), db(L, std::vector<float>(G));
  std::vector<float> y(std::size_t(H) * B * T), dx0(std::size_t(cfg.input) * B * T);
  std::vector<const float*> pw, pr, pb;
  std::vector<float*> ph, pc, pg, pt, pdg, pdh, pdc, pdw, pdr, pdb;
  for (int l = 0; l < L; ++l) {
    pw.push_back(params[l].w.data());
    pr.push_back(params[l].r.data());
    pb.push_back(params[l].bias.data());
    dw[l].resize(std::size_t(G) * cfg.input_width(l));
    dr[l].resize(std::size_t(G) * H);
    ph.push_back(hs[l].data());
    pc.push_back(cs[l].data());
    pg.push_back(gs[l].data());
    pt.push_back(ts[l].data());
    pdg.push_back(dg[l].data());
    pdh.push_back(dh0[l].data());
    pdc.push_back(dc0[l].data());
    pdw.push_back(dw[l].data());
    pdr.push_back(dr[l].data());
    pdb.push_back(db[l].data());
  }
  rwo_forward(&d, pw.data(), pr.data(), pb.data(), x.data(), nullptr, nullptr, 1, ph.data(),
              pc.data(), pg.data(), pt.data(), y.data());
  rwo_backward_data(&d, pw.data(), pr.data(), ph.data(), pc.data(), pg.data(), pt.data(), dy.data(),
                    pdg.data(), dx0.data(), pdh.data(), pdc.data());
  rwo_weight_update(&d, x.data(), ph.data(), pdg.data(), pdw.data(), pdr.data(), pdb.data());

  check("y", fwd.y.data(), y.data(), y.size(), nw_tol, sm_tol);
  check("dx0", bwd.dx0.data(), dx0.data(), dx0.size(), nw_tol, sm_tol);
  for (int l = 0; l < L; ++l) {
    const std::string s = "[" + std::to_string(l) + "]";
    check(("h_seq" + s).c_str(), fwd.tape.h_seq[l].data(), hs[l].data(), hs[l].size(), nw_tol, sm_tol);
    check(("gates" + s).c_str(), fwd.tape.gates_seq[l].data(), gs[l].data(), gs[l].size(), nw_tol, sm_tol);
    check(("dgw_seq" + s).c_str(), bwd.dgw_seq[l].data(), dg[l].data(), dg[l].size(), nw_tol, sm_tol);
    check(("dh0" + s).c_str(), bwd.dh0[l].data(), dh0[l].data(), dh0[l].size(), nw_tol, sm_tol);
    check(("dc0" + s).c_str(), bwd.dc0[l].data(), dc0[l].data(), dc0[l].size(), nw_tol, sm_tol);
    check(("dW" + s).c_str(), g.dw[l].data(), dw[l].data(), dw[l].size(), nw_tol, sm_tol);
    check(("dR" + s).c_str(), g.dr[l].data(), dr[l].data(), dr[l].size(), nw_tol, sm_tol);
    check(("db" + s).c_str(), g.db[l].data(), db[l].data(), db[l].size(), nw_tol, sm_tol);
  }
}

int main() {
  // error behaviour (test_engine.cpp:220-256)
  {
    LadderConfig cfg;
    cfg.layers = 2;
    cfg.hidden = 4;
    cfg.input = 4;
    cfg.batch = 2;
    cfg.steps = 2;
    cfg.seed = 1;
    cfg.opt_level = 1;
    auto params = init_params(cfg);
    Engine e(cfg);
    bool ok = false;
    try {
      e.forward(params, Matrix(3, 4), false);
    } catch (const std::invalid_argument& ex) {
      ok = std::string(ex.what()).find("expected") != std::string::npos;
    }
    Matrix x(4, 4), dy(4, 4);
    ForwardResult inf = e.forward(params, x, false);
    bool ok2 = false;
    try {
      e.backward_data(params, inf.tape, dy);
    } catch (const std::invalid_argument& ex) {
      ok2 = std::string(ex.what()).find("training") != std::string::npos;
    }
    bool ok3 = false;
    try {
      LadderConfig bad = cfg;
      bad.opt_level = 7;
      Engine eb(bad);
    } catch (const std::invalid_argument&) {
      ok3 = true;
    }
    std::printf("facade errors: expected=%d training=%d opt_level=%d\n", ok, ok2, ok3);
    if (!(ok && ok2 && ok3)) ++g_fail;
  }
  for (int prec : {RW_PREC_FP32, RW_PREC_BF16}) {
    LadderConfig c;
    c.layers = 2;
    c.hidden = 48;
    c.input = 40;
    c.batch = 6;
    c.steps = 24;
    c.batch_steps = 2;
    c.opt_level = 6;
    c.seed = 314159;
    run(prec, c);
    LadderConfig c2 = c;
    c2.layers = 3;
    c2.hidden = 200;
    c2.input = 130;
    c2.batch = 40;
    c2.steps = 16;
    run(prec, c2);
  }
  std::printf(g_fail ? "FACADE FAIL (%d)\n" : "FACADE PASS\n", g_fail);
  return g_fail ? 1 : 0;
}

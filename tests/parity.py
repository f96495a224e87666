"""Shared parity helpers: run the B200 engine and the reference on identical inputs and
compare every output tensor with the tolerance rules of SURVEY.md §8c:

  * fp32-parity mode (3xTF32): normwise ||d||/||ref|| <= 1e-5 AND scaled-max
    max|d|/max|ref| <= 1e-5 for y, h_T, c_T, dx0, dh0, dc0, dW, dR, db.
  * bf16 mode: normwise <= 1e-2 AND scaled-max <= 2e-2.
Elementwise relative error is not used (near-zero entries make it meaningless even for an
fp64 truth).
"""
from __future__ import annotations

import numpy as np

TOL = {"fp32": (1e-5, 1e-5), "bf16": (1e-2, 2e-2)}


def errors(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = got - ref
    nref = np.linalg.norm(ref)
    mref = np.abs(ref).max() if ref.size else 0.0
    if nref == 0.0:
        return (float(np.linalg.norm(d)), float(np.abs(d).max()) if d.size else 0.0)
    return float(np.linalg.norm(d) / nref), float(np.abs(d).max() / mref)


def make_case(cfg, seed, bias=False, state=False):
    """SplitMix64 weights/inputs exactly like the reference (init_params, make_input/make_dy),
    optionally with nonzero bias and initial states (SURVEY §8c asks for both). cfg.kind (the
    reference's CellKind, default LSTM) selects the cell; c0 exists for LSTM only."""
    from paper_1604_01946_b200 import engine as E
    kind = getattr(cfg, "kind", 3)
    c = E.LadderConfig(layers=cfg.layers, hidden=cfg.hidden, input=cfg.input, batch=cfg.batch,
                       steps=cfg.steps, seed=seed, kind=kind)
    params = E.init_params(c)
    if bias:
        for l, p in enumerate(params):
            p.bias = E.splitmix_symmetric(seed, 300 + l, 0.5, E.gate_count(kind) * c.hidden)
    h0 = c0 = None
    if state:
        h0 = [E.random_matrix(c.hidden, c.batch, seed, 50 + l) for l in range(c.layers)]
        if kind == 3:
            c0 = [E.random_matrix(c.hidden, c.batch, seed, 60 + l) for l in range(c.layers)]
    x = E.make_input(c)
    dy = E.make_dy(c)
    return c, params, x, dy, h0, c0


def run_reference(ref, c, params, x, dy, h0, c0):
    w = [p.w for p in params]
    r = [p.r for p in params]
    b = [np.ascontiguousarray(p.bias, np.float32) for p in params]
    return ref.run(c, w, r, b, x, h0, c0, dy)


def run_device(eng, params, x, dy, h0, c0):
    fwd = eng.forward(params, x, True, h0, c0)
    bwd = eng.backward_data(params, fwd.tape, dy)
    g = eng.weight_update(fwd.tape, bwd)
    c = eng.cfg
    out = {"y": fwd.y, "dx0": bwd.dx0, "dh0": bwd.dh0, "dc0": bwd.dc0, "dw": g.dw, "dr": g.dr,
           "db": g.db}
    out["hT"] = [fwd.tape.h_seq[l][:, c.batch * c.steps:] for l in range(c.layers)]
    if c.kind == 3:
        out["cT"] = [fwd.tape.c_seq[l][:, c.batch * c.steps:] for l in range(c.layers)]
    return out


def compare(dev, refo, c):
    """-> list of (name, normwise, scaled_max)."""
    rows = []
    rows.append(("y",) + errors(dev["y"], refo["y"]))
    rows.append(("dx0",) + errors(dev["dx0"], refo["dx0"]))
    bt = c.batch * c.steps
    lstm = getattr(c, "kind", 3) == 3
    for l in range(c.layers):
        rows.append((f"hT[{l}]",) + errors(dev["hT"][l], refo["h_seq"][l][:, bt:]))
        if lstm:
            rows.append((f"cT[{l}]",) + errors(dev["cT"][l], refo["c_seq"][l][:, bt:]))
        rows.append((f"dh0[{l}]",) + errors(dev["dh0"][l], refo["dh0"][l]))
        if lstm:
            rows.append((f"dc0[{l}]",) + errors(dev["dc0"][l], refo["dc0"][l]))
        rows.append((f"dW[{l}]",) + errors(dev["dw"][l], refo["dw"][l]))
        rows.append((f"dR[{l}]",) + errors(dev["dr"][l], refo["dr"][l]))
        rows.append((f"db[{l}]",) + errors(dev["db"][l], refo["db"][l]))
    return rows


def assert_within(rows, precision):
    nw_tol, sm_tol = TOL[precision]
    bad = [r for r in rows if not (r[1] <= nw_tol and r[2] <= sm_tol)]
    worst = max(rows, key=lambda r: max(r[1] / nw_tol, r[2] / sm_tol))
    assert not bad, f"{precision}: {len(bad)} tensors out of tolerance, e.g. {bad[:4]}; worst {worst}"
    return worst

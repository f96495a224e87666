"""Layer pipeline: stages must reproduce the single-context run bit for bit -- the
boundary layer's off-critical GEMM uses the same k-split and reduction order, only on the
neighbour's GPU. On one GPU the stages run one after another with a ring as deep as T
(RW_PP_RING, read when the contexts are created): forward of stage 0, 1, ..., then backward of
the last stage down to stage 0. That exercises the whole data path (rings, counters, the
layer-input copy and its ready flag) without needing the stages co-resident on the device."""
import os

import numpy as np
import pytest

from parity import make_case

pytestmark = pytest.mark.gpu

from oracle import Dims  # noqa: E402


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("dims,n", [(Dims(4, 128, 96, 32, 10), 2), (Dims(3, 64, 64, 16, 7), 3),
                                    (Dims(3, 128, 96, 32, 8, kind=2), 3), (Dims(2, 64, 48, 16, 6, kind=0), 2)],
                         ids=["L4H128x2", "L3H64x3", "gru-L3H128x3", "rnn-L2H64x2"])
def test_pipeline_matches_single_context(dims, n, precision, monkeypatch):
    from paper_1604_01946_b200 import Engine
    from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process
    c, params, x, dy, _, _ = make_case(dims, seed=23, bias=True)
    H, I, B, T, L = c.hidden, c.input, c.batch, c.steps, c.layers
    ref = Engine(c, precision=precision, schedule="cluster")
    ref.set_params(params)
    ref.upload_inputs(x, dy)
    ref.run_pass(2)
    ref.sync()
    y_r = np.zeros((H, B * T), np.float32, order="F")
    dx_r = np.zeros((I, B * T), np.float32, order="F")
    G = {3: 4, 2: 3}.get(getattr(dims, "kind", 3), 1)  # gate count of the cell kind
    dw_r = [np.zeros((G * H, I if l == 0 else H), np.float32, order="F") for l in range(L)]
    dr_r = [np.zeros((G * H, H), np.float32, order="F") for _ in range(L)]
    db_r = [np.zeros(G * H, np.float32) for _ in range(L)]
    ref.read_outputs(y_r, dx_r, dw_r, dr_r, db_r)

    monkeypatch.setenv("RW_PP_RING", str(T))
    stages = [PipelineStage(c, k, n, precision=precision) for k in range(n)]
    for s in stages:
        s.set_params(params)
    link_in_process(stages, params)
    zx = np.zeros((H, B * T), np.float32, order="F")
    for k, s in enumerate(stages):
        s.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)
    for rep in range(2):  # twice: the cumulative per-pass counters must carry over
        for s in stages:          # forward, stage by stage (pass 3: training tape)
            s.engine.run_pass(3)
            s.engine.sync()
        for s in reversed(stages):  # backward from the last stage down
            s.engine.run_pass(1)
            s.engine.sync()
        for s in stages:
            lo, cnt = s.first, s.count
            y = np.zeros((H, B * T), np.float32, order="F")
            dx = np.zeros((I if s.k == 0 else H, B * T), np.float32, order="F")
            dw = [np.zeros_like(dw_r[l]) for l in range(lo, lo + cnt)]
            dr = [np.zeros_like(dr_r[l]) for l in range(lo, lo + cnt)]
            db = [np.zeros_like(db_r[l]) for l in range(lo, lo + cnt)]
            s.engine.read_outputs(y, dx, dw, dr, db)
            for j in range(cnt):
                assert np.array_equal(dw[j], dw_r[lo + j]), (rep, "dW", lo + j)
                assert np.array_equal(dr[j], dr_r[lo + j]), (rep, "dR", lo + j)
                assert np.array_equal(db[j], db_r[lo + j]), (rep, "db", lo + j)
            if s.k == n - 1:
                assert np.array_equal(y, y_r), (rep, "y")
            if s.k == 0:
                assert np.array_equal(dx, dx_r), (rep, "dx0")


@pytest.mark.parametrize("schedule,precision,dims,n,ks", [
    ("persistent", "bf16", Dims(4, 128, 96, 32, 10), 2, "2"),
    ("persistent", "fp32", Dims(4, 128, 96, 32, 8), 2, "1"),
    ("stepwise", "fp32", Dims(4, 128, 128, 32, 7, kind=2), 2, "1"),
    ("stepwise", "bf16", Dims(6, 64, 64, 16, 6, kind=0), 3, "1"),
    # config E's kernels: the CTA-pair persistent backward / stepwise forward
    ("persistent", "bf16", Dims(4, 256, 256, 128, 5), 2, "1"),
    ("stepwise", "bf16", Dims(4, 256, 256, 128, 5), 2, "1"),
], ids=["pers-bf16", "pers-fp32", "step-gru-fp32", "step-rnn-bf16x3", "pers-pairbwd-bf16", "step-pairfwd-bf16"])
def test_pipeline_plain_matches_single_context(schedule, precision, dims, n, ks, monkeypatch):
    """The persistent / stepwise family (config E's schedules): h_t stored into the next stage's
    layer-input planes, the next stage's dG_t into this stage's dG-input planes with W_next^T in
    the top layer's backward image -- bitwise the single context with the same k-split."""
    from paper_1604_01946_b200 import Engine
    from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process
    monkeypatch.setenv("RW_FWD_KSPLIT", ks)
    monkeypatch.setenv("RW_BWD_KSPLIT", ks)
    c, params, x, dy, _, _ = make_case(dims, seed=31, bias=True)
    H, I, B, T, L = c.hidden, c.input, c.batch, c.steps, c.layers
    ref = Engine(c, precision=precision, schedule=schedule)
    desc = ref.describe()
    if desc["fwd_schedule"] == "cluster":
        pytest.skip("auto chose the cluster schedule")
    ref.set_params(params)
    ref.upload_inputs(x, dy)
    ref.run_pass(2)
    ref.sync()
    G = {3: 4, 2: 3}.get(getattr(dims, "kind", 3), 1)
    y_r = np.zeros((H, B * T), np.float32, order="F")
    dx_r = np.zeros((I, B * T), np.float32, order="F")
    dw_r = [np.zeros((G * H, I if l == 0 else H), np.float32, order="F") for l in range(L)]
    dr_r = [np.zeros((G * H, H), np.float32, order="F") for _ in range(L)]
    db_r = [np.zeros(G * H, np.float32) for _ in range(L)]
    ref.read_outputs(y_r, dx_r, dw_r, dr_r, db_r)

    stages = [PipelineStage(c, k, n, precision=precision, schedule=schedule) for k in range(n)]
    kinds = [(d["fwd_schedule"], d["bwd_schedule"], d["fwd_pair"], d["bwd_pair"])
             for d in [desc] + [s.engine.describe() for s in stages]]
    for s in stages:
        s.set_params(params)
    link_in_process(stages, params)
    zx = np.zeros((H, B * T), np.float32, order="F")
    for k, s in enumerate(stages):
        s.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)
    if dims.batch >= 128:  # the CTA-pair kernels are the ones exercised
        assert kinds[1][3] if schedule == "persistent" else kinds[1][2], kinds
    for rep in range(2):  # the cumulative per-pass counters must carry over
        for s in stages:
            s.engine.run_pass(3)
            s.engine.sync()
        for s in reversed(stages):
            s.engine.run_pass(1)
            s.engine.sync()
        for s in stages:
            lo, cnt = s.first, s.count
            y = np.zeros((H, B * T), np.float32, order="F")
            dx = np.zeros((I if s.k == 0 else H, B * T), np.float32, order="F")
            dw = [np.zeros_like(dw_r[l]) for l in range(lo, lo + cnt)]
            dr = [np.zeros_like(dr_r[l]) for l in range(lo, lo + cnt)]
            db = [np.zeros_like(db_r[l]) for l in range(lo, lo + cnt)]
            s.engine.read_outputs(y, dx, dw, dr, db)
            for j in range(cnt):
                assert np.array_equal(dw[j], dw_r[lo + j]), (rep, "dW", lo + j, np.abs(dw[j] - dw_r[lo + j]).max(), kinds)
                assert np.array_equal(dr[j], dr_r[lo + j]), (rep, "dR", lo + j, np.abs(dr[j] - dr_r[lo + j]).max())
                assert np.array_equal(db[j], db_r[lo + j]), (rep, "db", lo + j)
            if s.k == n - 1:
                assert np.array_equal(y, y_r), (rep, "y", np.abs(y - y_r).max())
            if s.k == 0:
                assert np.array_equal(dx, dx_r), (rep, "dx0", np.abs(dx - dx_r).max())


def test_pipeline_plain_rejects_mixed_families(monkeypatch):
    from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process
    c, params, x, dy, _, _ = make_case(Dims(4, 128, 96, 32, 4), seed=3, bias=True)
    stages = [PipelineStage(c, 0, 2, schedule="persistent"), PipelineStage(c, 1, 2, schedule="cluster")]
    for s in stages:
        s.set_params(params)
    with pytest.raises(Exception, match="schedule famil"):
        link_in_process(stages, params)


def _single(c, params, x, dy):
    from paper_1604_01946_b200 import Engine
    H, I, B, T, L = c.hidden, c.input, c.batch, c.steps, c.layers
    ref = Engine(c, precision="bf16", schedule="cluster")
    ref.set_params(params)
    ref.upload_inputs(x, dy)
    ref.run_pass(2)
    ref.sync()
    y = np.zeros((H, B * T), np.float32, order="F")
    dw = [np.zeros((4 * H, I if l == 0 else H), np.float32, order="F") for l in range(L)]
    ref.read_outputs(y=y, dw=dw)
    return y, dw


def test_pipeline_follows_parameter_updates(monkeypatch):
    """After the stages are linked, new parameters (an optimizer step) reach the forward boundary
    group too (rw_pp_set_next_w): the next pass equals a fresh single context on the new
    parameters, bit for bit (the boundary kept the link-time W)."""
    from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process
    c, params, x, dy, _, _ = make_case(Dims(4, 128, 96, 32, 6), seed=29, bias=True)
    H, B, T, L, n = c.hidden, c.batch, c.steps, c.layers, 2
    monkeypatch.setenv("RW_PP_RING", str(T))
    stages = [PipelineStage(c, k, n) for k in range(n)]
    for s in stages:
        s.set_params(params)
    link_in_process(stages, params)
    zx = np.zeros((H, B * T), np.float32, order="F")
    for k, s in enumerate(stages):
        s.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)

    def run():
        for s in stages:
            s.engine.run_pass(3)
            s.engine.sync()
        for s in reversed(stages):
            s.engine.run_pass(1)
            s.engine.sync()
        y = np.zeros((H, B * T), np.float32, order="F")
        stages[-1].engine.read_outputs(y=y)
        return y

    run()
    for p in params:  # "optimizer step"
        p.w[:] = p.w * np.float32(0.9) + np.float32(0.01)
        p.r[:] = p.r * np.float32(1.1)
    for s in stages:
        s.set_params(params)
    y = run()
    y_ref, _ = _single(c, params, x, dy)
    assert np.array_equal(y, y_ref)


@pytest.mark.parametrize("schedule,precision", [("cluster", "bf16"), ("persistent", "bf16"), ("stepwise", "fp32")])
def test_pipeline_stages_run_concurrently(schedule, precision, monkeypatch):
    """Both stages in flight at once (in-process, each on its own stream, no host sync between
    the stages): stage 1's forward spins on stage 0's per-step h_t counters while stage 0 is
    still running, stage 0's backward on stage 1's dG_t (cluster: the default ring depth, so the
    ring's back-pressure is live too). Bitwise the single context. With the cluster schedule the
    overlap is forced: the backward ring is 4 steps deep and T = 24, so stage 1's boundary group
    cannot finish before stage 0's backward has consumed 20 of its partials -- run one after the
    other, the two kernels would deadlock into the flag timeout instead."""
    import time
    from paper_1604_01946_b200 import Engine
    from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process
    monkeypatch.setenv("RW_FWD_KSPLIT", "1")
    monkeypatch.setenv("RW_BWD_KSPLIT", "1")
    dims = Dims(4, 128, 128, 32, 24)
    c, params, x, dy, _, _ = make_case(dims, seed=37, bias=True)
    H, I, B, T, L, n = c.hidden, c.input, c.batch, c.steps, c.layers, 2
    ref = Engine(c, precision=precision, schedule=schedule)
    ref.set_params(params)
    ref.upload_inputs(x, dy)
    ref.run_pass(2)
    ref.sync()
    y_r = np.zeros((H, B * T), np.float32, order="F")
    dw_r = [np.zeros((4 * H, I if l == 0 else H), np.float32, order="F") for l in range(L)]
    ref.read_outputs(y=y_r, dw=dw_r)
    stages = [PipelineStage(c, k, n, precision=precision, schedule=schedule) for k in range(n)]
    for s in stages:
        s.set_params(params)
    link_in_process(stages, params)
    zx = np.zeros((H, B * T), np.float32, order="F")
    for k, s in enumerate(stages):
        s.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)
    for s in stages:
        s.engine.sync()
    t0 = time.perf_counter()
    for s in stages:            # both forwards enqueued back to back
        s.engine.run_pass(3)
    for s in reversed(stages):  # then both backwards
        s.engine.run_pass(1)
    for s in stages:
        s.engine.sync()
    elapsed = time.perf_counter() - t0
    y = np.zeros((H, B * T), np.float32, order="F")
    stages[1].engine.read_outputs(y=y)
    assert np.array_equal(y, y_r), np.abs(y - y_r).max()
    for s in stages:
        lo, cnt = s.first, s.count
        dw = [np.zeros_like(dw_r[l]) for l in range(lo, lo + cnt)]
        s.engine.read_outputs(dw=dw)
        for j in range(cnt):
            assert np.array_equal(dw[j], dw_r[lo + j]), ("dW", lo + j)
    assert elapsed < 20.0  # no flag wait ran into its timeout


@pytest.mark.parametrize("host_w", [False, True], ids=["live-peer-W", "host-W_next"])
def test_pipeline_plain_follows_parameter_updates(host_w, monkeypatch):
    """Persistent family: the lower stage's top-layer backward multiplies by the next stage's
    W_0. After an optimizer step it must use the new W_0 -- read live over the link (set_params
    marks the image for re-packing) or, when the link was given a host copy, the copy handed to
    rw_pp_set_next_w -- bitwise a fresh single context on the new parameters."""
    from paper_1604_01946_b200 import Engine
    from paper_1604_01946_b200.pipeline import PipelineStage, link_in_process
    monkeypatch.setenv("RW_FWD_KSPLIT", "1")
    monkeypatch.setenv("RW_BWD_KSPLIT", "1")
    c, params, x, dy, _, _ = make_case(Dims(4, 128, 128, 32, 6), seed=43, bias=True)
    H, I, B, T, L, n = c.hidden, c.input, c.batch, c.steps, c.layers, 2
    stages = [PipelineStage(c, k, n, schedule="persistent") for k in range(n)]
    for s in stages:
        s.set_params(params)
    ex = [s.export() for s in stages]
    stages[0].engine.pp_link(0, ex[1][0], params[2].w if host_w else None)
    stages[1].engine.pp_link(1, ex[0][1])
    zx = np.zeros((H, B * T), np.float32, order="F")
    for k, s in enumerate(stages):
        s.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)

    def run():
        for s in stages:
            s.engine.run_pass(3)
            s.engine.sync()
        for s in reversed(stages):
            s.engine.run_pass(1)
            s.engine.sync()
        dr = [np.zeros((4 * H, H), np.float32, order="F") for _ in range(2)]
        stages[0].engine.read_outputs(dr=dr)
        return dr

    run()
    for p in params:  # "optimizer step"
        p.w[:] = p.w * np.float32(0.9) + np.float32(0.01)
        p.r[:] = p.r * np.float32(1.1)
    stages[1].set_params(params)  # only the upper stage's parameters are re-sent ...
    stages[0].set_params(params)
    if host_w:  # ... and the lower stage gets the new W_next as a host copy
        stages[0].engine.pp_set_next_w(params[2].w)
    dr = run()
    ref = Engine(c, precision="bf16", schedule="persistent")
    ref.set_params(params)
    ref.upload_inputs(x, dy)
    ref.run_pass(2)
    ref.sync()
    dr_r = [np.zeros((4 * H, H), np.float32, order="F") for _ in range(L)]
    ref.read_outputs(dr=dr_r)
    for j in range(2):
        assert np.array_equal(dr[j], dr_r[j]), j

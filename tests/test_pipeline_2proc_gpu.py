"""GPU: the layer pipeline across PROCESSES (one process per stage, as on a multi-GPU box): two
stages on one GPU in two processes, linked through CUDA IPC handles of the boundary rings
(rw_pp_export / rw_pp_link, system-scope flags), must give bitwise the single context's
results -- the cross-process path of SURVEY §8e that bench / torchrun use, minus NVLink.

The stages run one after another (forward 0 -> 1, backward 1 -> 0, ring as deep as T): without
MPS two processes' kernels on one GPU time-slice rather than co-run, so two persistent kernels
that spin on each other's flags cannot make progress concurrently there; on separate GPUs
(the deployment) they do."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from parity import make_case  # noqa: E402
from oracle import Dims  # noqa: E402

DIMS = Dims(4, 128, 96, 32, 6)
SEED = 53


def _stage_proc(k, n, conn, precision, schedule="cluster"):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ["RW_PP_RING"] = str(DIMS.steps)
    os.environ["RW_FWD_KSPLIT"] = os.environ["RW_BWD_KSPLIT"] = "1"
    from parity import make_case as mk
    from paper_1604_01946_b200.pipeline import PipelineStage
    try:
        c, params, x, dy, _, _ = mk(DIMS, seed=SEED, bias=True)
        H, B, T = c.hidden, c.batch, c.steps
        st = PipelineStage(c, k, n, precision=precision, schedule=schedule)
        st.set_params(params)
        conn.send(("exports", st.export()))
        nxt, prv = conn.recv()
        st.link(nxt, prv, params)
        zx = np.zeros((H, B * T), np.float32, order="F")
        st.engine.upload_inputs(x if k == 0 else zx, dy if k == n - 1 else zx)
        conn.send(("linked", None))
        while True:
            cmd = conn.recv()
            if cmd == "done":
                break
            st.engine.run_pass(cmd)
            st.engine.sync()
            conn.send(("ok", None))
        y = np.zeros((H, B * T), np.float32, order="F")
        I = c.input if k == 0 else H
        dx = np.zeros((I, B * T), np.float32, order="F")
        lo, cnt = st.first, st.count
        dw = [np.zeros((4 * H, c.input if l == 0 else H), np.float32, order="F") for l in range(lo, lo + cnt)]
        st.engine.read_outputs(y, dx, dw)
        conn.send(("out", (y, dx, dw, lo)))
    except Exception as e:  # surface the failure in the parent
        conn.send(("error", repr(e)))


@pytest.mark.parametrize("precision,schedule", [("bf16", "cluster"), ("fp32", "cluster"), ("bf16", "persistent"),
                                                ("fp32", "stepwise")])
def test_two_process_pipeline_matches_single_context(precision, schedule, monkeypatch):
    import multiprocessing as mp
    from paper_1604_01946_b200 import Engine
    c, params, x, dy, _, _ = make_case(DIMS, seed=SEED, bias=True)
    H, I, B, T, L = c.hidden, c.input, c.batch, c.steps, c.layers
    monkeypatch.setenv("RW_FWD_KSPLIT", "1")  # the stages' k-split (the children set the same)
    monkeypatch.setenv("RW_BWD_KSPLIT", "1")
    ref = Engine(c, precision=precision, schedule=schedule)
    ref.set_params(params)
    ref.upload_inputs(x, dy)
    ref.run_pass(2)
    ref.sync()
    y_r = np.zeros((H, B * T), np.float32, order="F")
    dx_r = np.zeros((I, B * T), np.float32, order="F")
    dw_r = [np.zeros((4 * H, I if l == 0 else H), np.float32, order="F") for l in range(L)]
    ref.read_outputs(y_r, dx_r, dw_r)
    ref.close()

    n = 2
    ctx = mp.get_context("spawn")
    pipes, procs = [], []
    for k in range(n):
        a, b = ctx.Pipe()
        p = ctx.Process(target=_stage_proc, args=(k, n, b, precision, schedule))
        p.start()
        pipes.append(a)
        procs.append(p)

    def recv(k, want):
        assert pipes[k].poll(300), f"stage {k} timed out waiting for {want}"
        tag, val = pipes[k].recv()
        assert tag == want, (k, tag, val)
        return val

    try:
        ex = [recv(k, "exports") for k in range(n)]
        for k in range(n):
            pipes[k].send((ex[k + 1] if k + 1 < n else None, ex[k - 1] if k > 0 else None))
        for k in range(n):
            recv(k, "linked")
        for k in range(n):  # forward, stage by stage (training tape)
            pipes[k].send(3)
            recv(k, "ok")
        for k in reversed(range(n)):  # backward from the last stage down
            pipes[k].send(1)
            recv(k, "ok")
        outs = []
        for k in range(n):
            pipes[k].send("done")
            outs.append(recv(k, "out"))
    finally:
        for p in procs:
            p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    y, _, _, _ = outs[-1]
    assert np.array_equal(y, y_r)
    _, dx, _, _ = outs[0]
    assert np.array_equal(dx, dx_r)
    for y_k, dx_k, dw, lo in outs:
        for j, a in enumerate(dw):
            assert np.array_equal(a, dw_r[lo + j]), ("dW", lo + j)

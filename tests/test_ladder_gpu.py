"""GPU: every rung of the device optimisation ladder (rw_ladder_pass O0-O4: per-gate GEMMs on the
reference-layout weights, grouped, streamed, the fused cell, the pre-transposed step kernel;
runtime.cu run_ladder_forward) computes the same forward pass as the unmodified reference engine,
within the precision's tolerance -- the device form of the reference's equivalent_to_naive gate
(bench.hpp:176-224). Shapes: aligned and ragged (H not a multiple of 64, batch not of 16)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("dims", [(2, 64, 64, 16, 5), (2, 130, 70, 33, 4), (3, 96, 40, 20, 6)])
def test_ladder_rungs_match_reference(prec, dims):
    from oracle import Reference
    from parity import TOL, errors, make_case
    from paper_1604_01946_b200 import Engine, LadderConfig
    try:
        ref = Reference()
    except FileNotFoundError as e:
        pytest.skip(str(e))
    L, H, I, B, T = dims
    cfg = LadderConfig(layers=L, hidden=H, input=I, batch=B, steps=T, seed=11)
    c, params, x, dy, _, _ = make_case(cfg, 11, bias=True)
    want = ref.run(c, [p.w for p in params], [p.r for p in params],
                   [np.ascontiguousarray(p.bias, np.float32) for p in params], x, training=False)["y"]
    e = Engine(c, precision=prec, schedule="stepwise")
    e.set_params(params)
    e.upload_inputs(x, dy)
    tol = TOL[prec]
    for level in range(5):
        e.ladder_pass(level)
        e.sync()
        y = np.zeros((H, B * T), np.float32, order="F")
        e.read_outputs(y=y)
        nw, sm = errors(y, want)
        assert nw <= tol[0] and sm <= tol[1], (level, nw, sm)

"""CPU: the fp64 truth used by the full-size parity tests (tests/fp64_truth.py) agrees with the
reference CPU engine (oracle/_ref, else the C restatement) on small cases -- to fp32 rounding --
including nonzero bias and initial states, so it is the same LSTM the reference computes."""
import pytest

from oracle import Dims
from parity import errors, make_case, run_reference


@pytest.mark.parametrize("dims", [Dims(2, 24, 17, 5, 6), Dims(3, 40, 40, 3, 9)],
                         ids=lambda d: f"L{d.layers}H{d.hidden}I{d.input}B{d.batch}T{d.steps}")
def test_fp64_truth_matches_reference(reference, dims):
    from fp64_truth import lstm_truth
    c, params, x, dy, h0, c0 = make_case(dims, seed=9, bias=True, state=True)
    ref = run_reference(reference, c, params, x, dy, h0, c0)
    tr = lstm_truth(c, params, x, dy, h0, c0, device="cpu")
    bt = c.batch * c.steps
    pairs = [(tr["y"], ref["y"]), (tr["dx0"], ref["dx0"])]
    for l in range(c.layers):
        pairs += [(tr["hT"][l], ref["h_seq"][l][:, bt:]), (tr["cT"][l], ref["c_seq"][l][:, bt:]),
                  (tr["dh0"][l], ref["dh0"][l]), (tr["dc0"][l], ref["dc0"][l]), (tr["dw"][l], ref["dw"][l]),
                  (tr["dr"][l], ref["dr"][l]), (tr["db"][l], ref["db"][l])]
    for a, b in pairs:
        nw, sm = errors(b, a)
        assert nw < 1e-5 and sm < 1e-5, (nw, sm)

"""GPU parity of the GRU (linear before reset) and vanilla-RNN (tanh, relu) cells -- SURVEY §8(f)
row 2 -- against the unmodified reference CPU engine (oracle/_ref, cells.hpp:200-225, 283-333,
365-400, 486-562) on identical SplitMix64 weights and inputs with nonzero bias and h0, through
the reference-shaped API, in both precision modes. Tolerances: tests/parity.py. The device runs
these cells on the cluster schedule (rec_cluster.cuh) and on the persistent / stepwise schedules
(lstm_step.cuh), per-class instantiations."""
import numpy as np
import pytest

from oracle import Dims
from parity import assert_within, compare, make_case, run_device, run_reference

pytestmark = pytest.mark.gpu

KINDS = {0: "rnn-tanh", 1: "rnn-relu", 2: "gru"}
SHAPES = [
    (1, 5, 7, 3, 4),       # everything padded
    (2, 64, 48, 16, 7),
    (3, 96, 40, 20, 10),   # H not a multiple of 64, B not of 16
    (2, 130, 70, 33, 5),   # ragged second tile, 3 batch blocks
    (2, 256, 256, 64, 12), # split critical members (kc > 1)
]


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("kind", list(KINDS), ids=lambda k: KINDS[k])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "L{}H{}I{}B{}T{}".format(*s))
def test_cell_parity(reference, kind, shape, precision):
    from paper_1604_01946_b200 import Engine
    dims = Dims(*shape, kind=kind)
    c, params, x, dy, h0, c0 = make_case(dims, seed=19, bias=True, state=True)
    eng = Engine(c, precision=precision)
    d = eng.describe()
    assert d["fwd_schedule"] == d["bwd_schedule"] == "cluster", d
    dev = run_device(eng, params, x, dy, h0, c0)
    ref = run_reference(reference, c, params, x, dy, h0, c0)
    rows = compare(dev, ref, c)
    if kind == 1 and precision == "bf16":
        # ReLU recurrences do not damp perturbations (tanh's 1 - h^2 and LSTM's gates do): the bf16
        # operand rounding of the backward grows through the steps to 5-10 % normwise on the
        # layer-0 gradients (measured), while fp32-parity mode meets 1e-5. Forward tensors keep
        # the bf16 bound; backward tensors get an explicit, looser one.
        fwd = [r for r in rows if r[0] == "y" or r[0].startswith("hT")]
        assert_within(fwd, precision)
        bad = [r for r in rows if r not in fwd and not (r[1] <= 0.2 and r[2] <= 0.4)]
        assert not bad, bad
        return
    worst = assert_within(rows, precision)
    print(f"{KINDS[kind]} {shape} {precision}: worst {worst}")


def test_gru_tapes_and_errors(reference):
    """GRU tape fields (zrh_seq, dgr_seq, no c_seq) against the reference's, and the reference's
    error for c0 on a cell without cell state (engine.hpp:283-285)."""
    from paper_1604_01946_b200 import Engine
    c, params, x, dy, h0, _ = make_case(Dims(2, 64, 40, 8, 6, kind=2), seed=23, bias=True, state=True)
    eng = Engine(c, precision="fp32")
    fwd = eng.forward(params, x, True, h0)
    bwd = eng.backward_data(params, fwd.tape, dy)
    assert fwd.tape.c_seq == [] and fwd.tape.tanh_c_seq == [] and bwd.dc0 == []
    ref = reference.run(c, [p.w for p in params], [p.r for p in params],
                        [np.ascontiguousarray(p.bias, np.float32) for p in params], x, h0, None, dy)
    for l in range(c.layers):
        g = fwd.tape.gates_seq[l]
        assert g.shape == (3 * c.hidden, c.batch * c.steps)
        err = np.linalg.norm(g - ref["gates_seq"][l]) / np.linalg.norm(ref["gates_seq"][l])
        assert err < 1e-5, err
        assert fwd.tape.zrh_seq[l].shape == (c.hidden, c.batch * c.steps)
        assert bwd.dgr_seq[l].shape == (3 * c.hidden, c.batch * c.steps)
        e2 = np.linalg.norm(bwd.dgw_seq[l] - ref["dgw_seq"][l]) / np.linalg.norm(ref["dgw_seq"][l])
        assert e2 < 1e-5, e2
    with pytest.raises(ValueError, match="c0 supplied for a cell kind without cell state"):
        eng.forward(params, x, True, h0, h0)


# GRU / RNN on the persistent, stepwise and layer-sequential schedules (the large-H path; layerseq
# fp32 = 3xTF32 operands): the kernels sum
# [W|R].[x;h] over K and the GRU candidate's halves stay apart through the forward image's slots
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("kind", list(KINDS), ids=lambda k: KINDS[k])
@pytest.mark.parametrize("schedule", ["persistent", "stepwise", "layerseq"])
@pytest.mark.parametrize("shape", [(2, 64, 48, 16, 7), (2, 130, 70, 33, 5), (3, 96, 40, 20, 6)],
                         ids=lambda s: "L{}H{}I{}B{}T{}".format(*s))
def test_cell_parity_wavefront_schedules(reference, kind, shape, schedule, precision):
    from paper_1604_01946_b200 import Engine
    dims = Dims(*shape, kind=kind)
    c, params, x, dy, h0, c0 = make_case(dims, seed=29, bias=True, state=True)
    eng = Engine(c, precision=precision, schedule=schedule)
    d = eng.describe()
    assert d["fwd_schedule"] == d["bwd_schedule"] == schedule, d
    dev = run_device(eng, params, x, dy, h0, c0)
    ref = run_reference(reference, c, params, x, dy, h0, c0)
    rows = compare(dev, ref, c)
    if kind == 1 and precision == "bf16":  # as test_cell_parity: ReLU backward in bf16
        fwd = [r for r in rows if r[0] == "y" or r[0].startswith("hT")]
        assert_within(fwd, precision)
        assert not [r for r in rows if r not in fwd and not (r[1] <= 0.2 and r[2] <= 0.4)]
        return
    assert_within(rows, precision)


@pytest.mark.parametrize("kind", [2, 0], ids=["gru", "rnn-tanh"])
def test_cell_large_hidden_auto_schedule(reference, kind):
    """H = 1024 does not fit the cluster schedule: AUTO picks the persistent kernels for GRU / RNN."""
    from paper_1604_01946_b200 import Engine
    dims = Dims(1, 1024, 256, 32, 5, kind=kind)
    c, params, x, dy, h0, c0 = make_case(dims, seed=31, bias=True, state=True)
    eng = Engine(c, precision="fp32")
    assert eng.describe()["fwd_schedule"] != "cluster"
    dev = run_device(eng, params, x, dy, h0, c0)
    ref = run_reference(reference, c, params, x, dy, h0, c0)
    assert_within(compare(dev, ref, c), "fp32")

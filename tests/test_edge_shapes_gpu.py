"""GPU edge shapes (the reference's validation allows every positive size, config.hpp:74-96):
single step, single batch column, hidden / input of 1, one layer -- every schedule that takes the
shape, both precisions, every cell kind, against the reference engine."""
import pytest

from oracle import Dims
from parity import assert_within, compare, make_case, run_device, run_reference

pytestmark = pytest.mark.gpu

EDGE = [
    (1, 1, 1, 1, 1),     # everything 1
    (2, 3, 2, 1, 1),     # T = 1, B = 1
    (1, 17, 5, 2, 3),
    (3, 8, 300, 5, 2),   # input wider than hidden, ragged
]


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("kind", [3, 2, 0], ids=["lstm", "gru", "rnn-tanh"])
@pytest.mark.parametrize("schedule", ["auto", "persistent", "stepwise", "layerseq"])
@pytest.mark.parametrize("shape", EDGE, ids=lambda s: "L{}H{}I{}B{}T{}".format(*s))
def test_edge_shapes(reference, shape, schedule, kind, precision):
    from paper_1604_01946_b200 import Engine
    dims = Dims(*shape, kind=kind)
    c, params, x, dy, h0, c0 = make_case(dims, seed=37, bias=True, state=True)
    eng = Engine(c, precision=precision, schedule=schedule)
    dev = run_device(eng, params, x, dy, h0, c0)
    ref = run_reference(reference, c, params, x, dy, h0, c0)
    assert_within(compare(dev, ref, c), precision)

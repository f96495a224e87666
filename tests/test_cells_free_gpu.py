"""GPU: the free pointwise stage (cells.hpp:181 pointwise_forward, 349 pointwise_backward) on
the device (rw_pointwise_*, paper_1604_01946_b200.cells) against the unmodified reference's
functions (oracle/_ref) on the same inputs, every cell kind, fused and kernel-per-op modes,
training and inference. The device follows the reference's rounded operation chain (no FMA
contraction); only expf / tanhf may differ by an ulp or two from the host libm, so the bound is
a few fp32 ulps: |dev - ref| <= 4e-7 + 2e-6 |ref|."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))


def _ref():
    from oracle import Reference
    try:
        return Reference()
    except FileNotFoundError as e:
        pytest.skip(str(e))


def _close(a, b):
    np.testing.assert_allclose(a, b, rtol=2e-6, atol=4e-7)


def _mat(rng, r, c, s=1.0):
    return np.asfortranarray((rng.uniform(-s, s, (r, c))).astype(np.float32))


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", [(9, 5), (130, 33), (512, 64)])
def test_pointwise_forward_backward_vs_reference(kind, shape):
    from paper_1604_01946_b200 import cells
    from paper_1604_01946_b200.engine import gate_count
    ref = _ref()
    H, B = shape
    G = gate_count(kind)
    rng = np.random.default_rng(kind * 100 + H)
    zw, zr = _mat(rng, G * H, B, 3.0), _mat(rng, G * H, B, 3.0)
    bias = rng.uniform(-0.5, 0.5, G * H).astype(np.float32)
    h_prev, c_prev = _mat(rng, H, B), _mat(rng, H, B, 2.0)
    cp = c_prev if kind == 3 else None
    for fused in (True, False):
        r = ref.pointwise_forward(kind, fused, zw, zr, bias, h_prev, cp, training=True)
        h = np.zeros((H, B), np.float32, order="F")
        c = np.zeros((H, B), np.float32, order="F") if kind == 3 else None
        gates = np.zeros((G * H, B), np.float32, order="F") if kind in (2, 3) else None
        tanh_c = np.zeros((H, B), np.float32, order="F") if kind == 3 else None
        zr_h = np.zeros((H, B), np.float32, order="F") if kind == 2 else None
        cells.pointwise_forward(kind, fused, zw, zr, bias, h_prev, cp, h, c, gates, tanh_c, zr_h)
        _close(h, r["h"])
        for k, v in (("c", c), ("gates", gates), ("tanh_c", tanh_c)):
            if v is not None:
                _close(v, r[k])
        if kind == 2:
            np.testing.assert_array_equal(zr_h, r["zr_h"])  # a copy of zr's candidate block
        # inference: nothing saved, same h
        h2 = np.zeros((H, B), np.float32, order="F")
        c2 = np.zeros((H, B), np.float32, order="F") if kind == 3 else None
        cells.pointwise_forward(kind, fused, zw, zr, bias, h_prev, cp, h2, c2)
        np.testing.assert_array_equal(h2, h)

        saved = r["h"] if kind in (0, 1) else r["gates"]
        d_above, dh_carry, dc_carry = _mat(rng, H, B), _mat(rng, H, B), _mat(rng, H, B)
        db0 = rng.uniform(-1, 1, G * H).astype(np.float32)
        db_ref = db0.copy()
        rb = ref.pointwise_backward(kind, fused, saved, r.get("tanh_c"), r.get("zr_h"), h_prev, cp, d_above,
                                    dh_carry, dc_carry if kind == 3 else None, db_ref)
        dgw = np.zeros((G * H, B), np.float32, order="F")
        dgr = np.zeros((G * H, B), np.float32, order="F") if kind == 2 else None
        dhl = np.zeros((H, B), np.float32, order="F")
        dcp = np.zeros((H, B), np.float32, order="F") if kind == 3 else None
        db = db0.copy()
        cells.pointwise_backward(kind, fused, saved, r.get("tanh_c"), r.get("zr_h"), h_prev, cp, d_above, dh_carry,
                                 dc_carry if kind == 3 else None, dgw, dgr, dhl, dcp, db)
        # the backward chain has no transcendental: bitwise equal to the reference
        np.testing.assert_array_equal(dgw, rb["dgw"])
        np.testing.assert_array_equal(dhl, rb["dh_local"])
        if kind == 2:
            np.testing.assert_array_equal(dgr, rb["dgr"])
        if kind == 3:
            np.testing.assert_array_equal(dcp, rb["dc_prev"])
        np.testing.assert_array_equal(db, db_ref)


def test_pointwise_errors_match_reference_messages():
    from paper_1604_01946_b200 import cells
    H, B = 4, 3
    z = np.zeros((4 * H, B), np.float32, order="F")
    m = np.zeros((H, B), np.float32, order="F")
    with pytest.raises(ValueError, match="cells: cell state supplied for a cell kind without one"):
        cells.pointwise_forward(2, True, z[: 3 * H], z[: 3 * H], np.zeros(3 * H, np.float32), m, m, m.copy())
    with pytest.raises(ValueError, match="cells: zw is 8x3, expected 16x3"):
        cells.pointwise_forward(3, True, z[:8], z, np.zeros(4 * H, np.float32), m, m, m.copy(), m.copy())
    g = np.zeros((3 * H, B), np.float32, order="F")
    with pytest.raises(ValueError, match="cells: GRU needs distinct dgw and dgr blocks"):
        cells.pointwise_backward(2, True, g, None, m, m, None, m, m, None, g, g, m.copy())

"""CPU: pin the oracle before trusting it.

* The C restatement (oracle/lstm_oracle.c) must reproduce the reference's golden vectors
  BITWISE (same op chains, same libm, -ffp-contract=off) on every output tensor.
* The reference shim (oracle/_ref), when present, must reproduce them bitwise too (sanity
  of the fixture pipeline).
* Known-answer tests of the reference unit suite (test_cells.cpp, test_engine.cpp) hold.
"""
import math

import numpy as np
import pytest

import golden

CASES = golden.cases()


def _bitwise(out, case):
    for k, ref in case.out.items():
        refs = ref if isinstance(ref, list) else [ref]
        gots = out[k] if isinstance(out[k], list) else [out[k]]
        assert len(refs) == len(gots), k
        for l, (g, r) in enumerate(zip(gots, refs)):
            assert g.shape == r.shape, (k, l)
            assert g.tobytes() == r.tobytes(), f"{k}[{l}] differs (max {np.abs(g - r).max()})"


@pytest.mark.parametrize("case", CASES, ids=repr)
def test_restatement_matches_golden_bitwise(restatement, case):
    out = restatement.run(case.dims, case.w, case.r, case.b, case.x, case.h0, case.c0, case.dy)
    _bitwise(out, case)


@pytest.mark.parametrize("case", CASES, ids=repr)
def test_restatement_init_and_inputs(restatement, case):
    """init_params streams 2l/2l+1 and verify::make_input/make_dy streams 1000/1001."""
    w, r = restatement.init_params(case.dims, case.seed)
    for l in range(case.L):
        assert w[l].tobytes() == case.w[l].tobytes()
        assert r[l].tobytes() == case.r[l].tobytes()
    assert restatement.make_input(case.dims, case.seed).tobytes() == case.x.tobytes()
    assert restatement.make_dy(case.dims, case.seed).tobytes() == case.dy.tobytes()


def test_python_mirror_init_matches_golden():
    from paper_1604_01946_b200 import LadderConfig, init_params, make_dy, make_input
    for case in CASES:
        cfg = LadderConfig(layers=case.L, hidden=case.H, input=case.I, batch=case.B,
                           steps=case.T, seed=case.seed)
        p = init_params(cfg)
        for l in range(case.L):
            assert p[l].w.tobytes() == case.w[l].tobytes()
            assert p[l].r.tobytes() == case.r[l].tobytes()
        assert make_input(cfg).tobytes() == case.x.tobytes()
        assert make_dy(cfg).tobytes() == case.dy.tobytes()


@pytest.mark.parametrize("case", CASES, ids=repr)
def test_reference_shim_matches_golden(case):
    import oracle
    if oracle.reference_path() is None:
        pytest.skip("oracle/_ref not built")
    out = oracle.Reference().run(case.dims, case.w, case.r, case.b, case.x, case.h0, case.c0, case.dy)
    _bitwise(out, case)


def test_reference_vs_restatement_random(restatement):
    """Bitwise agreement on fresh random shapes (not only the fixtures)."""
    import oracle
    if oracle.reference_path() is None:
        pytest.skip("oracle/_ref not built")
    R = oracle.Reference()
    rng = np.random.default_rng(1234)
    for _ in range(6):
        d = oracle.Dims(int(rng.integers(1, 4)), int(rng.integers(1, 40)), int(rng.integers(1, 40)),
                        int(rng.integers(1, 6)), int(rng.integers(1, 9)))
        w, r = R.init_params(d, int(rng.integers(1 << 30)))
        b = [rng.uniform(-0.5, 0.5, 4 * d.hidden).astype(np.float32) for _ in range(d.layers)]
        x = R.make_input(d, 3)
        dy = R.make_dy(d, 3)
        a = R.run(d, w, r, b, x, None, None, dy)
        o = restatement.run(d, w, r, b, x, None, None, dy)
        for k in a:
            va = a[k] if isinstance(a[k], list) else [a[k]]
            vo = o[k] if isinstance(o[k], list) else [o[k]]
            for p, q in zip(va, vo):
                assert p.tobytes() == q.tobytes(), (d, k)


# ---------------------------------------------------------------- known answers
def _zero_net(restatement, H=4, B=3, c0val=0.0):
    import oracle
    d = oracle.Dims(1, H, 2, B, 1)
    w = [np.zeros((4 * H, 2), np.float32, order="F")]
    r = [np.zeros((4 * H, H), np.float32, order="F")]
    b = [np.zeros(4 * H, np.float32)]
    x = np.asfortranarray(np.ones((2, B), np.float32))
    c0 = [np.asfortranarray(np.full((H, B), c0val, np.float32))]
    return restatement.run(d, w, r, b, x, None, c0, None, training=True)


def test_zero_network_fixed_point(restatement):
    """test_cells.cpp:62-82: zero pre-activations -> h = c = 0, gates 0.5/0.5/0.5/0."""
    out = _zero_net(restatement)
    H = 4
    assert np.all(out["y"] == 0.0)
    g = out["gates_seq"][0]
    assert np.all(g[:3 * H] == 0.5) and np.all(g[3 * H:] == 0.0)


def test_unit_cell_state(restatement):
    """test_cells.cpp:84-101: c_prev = 1 -> c = 0.5, h = 0.5 tanh(0.5) = 0.2310585786."""
    out = _zero_net(restatement, H=2, B=2, c0val=1.0)
    assert np.all(out["c_seq"][0][:, 2:] == 0.5)
    assert np.all(np.abs(out["y"] - 0.5 * math.tanh(0.5)) < 1e-6)


def test_saturated_gates_copy_cell(restatement):
    """test_cells.cpp:188-200: b_i = -40, b_f = +40 -> c_t == c_prev bitwise."""
    import oracle
    H, B = 3, 2
    d = oracle.Dims(1, H, 2, B, 1)
    w = [np.zeros((4 * H, 2), np.float32, order="F")]
    r = [np.zeros((4 * H, H), np.float32, order="F")]
    b = np.zeros(4 * H, np.float32)
    b[:H] = -40.0
    b[H:2 * H] = 40.0
    x = np.asfortranarray(np.ones((2, B), np.float32))
    c0 = [np.asfortranarray(np.linspace(-0.9, 0.9, H * B, dtype=np.float32).reshape(H, B))]
    out = restatement.run(d, w, r, [b], x, None, c0, None)
    assert out["c_seq"][0][:, B:].tobytes() == c0[0].tobytes()


def test_flop_count(restatement):
    """test_cells.cpp:333-338."""
    from paper_1604_01946_b200 import flop_count
    assert restatement.flop_count_cell(512, 512, 64) == 268435456
    assert flop_count(3, 512, 512, 64) == 268435456


def test_scalar_hand_recurrence(restatement):
    """test_engine.cpp:58-86: 1x1 LSTM against a hand-written fp64 recurrence."""
    import oracle
    d = oracle.Dims(1, 1, 1, 1, 1)
    w, r = restatement.init_params(d, 11)
    x = np.asfortranarray(np.array([[0.63]], np.float32))
    out = restatement.run(d, w, r, [np.zeros(4, np.float32)], x, None, None, None, training=False)
    sig = lambda v: 1.0 / (1.0 + math.exp(-v))  # noqa: E731
    wv = [float(w[0][g, 0]) for g in range(4)]
    xv = float(np.float32(0.63))
    iv, ov, cb = sig(wv[0] * xv), sig(wv[2] * xv), math.tanh(wv[3] * xv)
    hv = ov * math.tanh(iv * cb)
    assert abs(float(out["y"][0, 0]) - hv) < 1e-6

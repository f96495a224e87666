"""CPU: the bench's roofline inputs (bench.py) -- reference FLOP convention, algorithmic HBM
bytes, the committed-ncu traffic lookup -- against hand-computed values."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_pass_flops_reference_convention():
    # B both = 322.1 GFLOP, E both = 41,232 GFLOP, A fwd = 26.8 GFLOP
    assert abs(bench.pass_flops(bench.CONFIGS["B"]) / 1e9 - 322.1) < 0.1
    assert abs(bench.pass_flops(bench.CONFIGS["E"]) / 1e9 - 41231.7) < 1.0
    assert abs(bench.pass_flops(bench.CONFIGS["A"], 1) / 1e9 - 26.8) < 0.1


def test_recurrent_bytes_weights_resident_vs_streamed():
    b, e = bench.CONFIGS["B"], bench.CONFIGS["E"]
    # config B: 16 MB of bf16 [W|R] read once; tapes dominate (30 B / cell element forward)
    L, H, I, B, T = b["layers"], b["hidden"], b["input"], b["batch"], b["steps"]
    w = sum(4 * H * ((I if l == 0 else H) + H) * 2 for l in range(L))
    assert bench.recurrent_bytes(b, True) == w + L * T * H * B * 30
    # config E: 512 MB of weights cannot stay on chip -> re-read every step
    L, H, I, B, T = e["layers"], e["hidden"], e["input"], e["batch"], e["steps"]
    w = sum(4 * H * ((I if l == 0 else H) + H) * 2 for l in range(L))
    assert bench.recurrent_bytes(e, True) == w * T + L * T * H * B * 30
    assert bench.recurrent_bytes(e, False) > 60e9


def test_ncu_traffic_lookup_uses_committed_capture():
    t = bench.ncu_traffic("k_cl_bwd", "B")
    assert t is None or 5e8 < t < 1e9  # ~0.72 GB per launch in profiles/r01
    assert bench.ncu_traffic("no_such_kernel", "B") is None

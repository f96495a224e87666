"""CPU: profiles/validate_trace.py flags a violated wavefront edge and accepts a consistent
trace (synthetic CSVs in the device trace schema)."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location("vt", os.path.join(ROOT, "profiles", "validate_trace.py"))
vt = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(vt)

HDR = "task_layer,task_block,phase,worker,span,start_ns,end_ns\n"


def _write(tmp_path, rows):
    p = tmp_path / "t.csv"
    p.write_text(HDR + "".join(",".join(map(str, r)) + "\n" for r in rows))
    return str(p)


def test_consistent_trace_passes(tmp_path):
    rows = []
    for t in range(3):
        for w in range(2):
            rows.append((0, t, "fwd", w, "wait", 100 * t, 100 * t + 10))
            rows.append((0, t, "fwd", w, "publish", 100 * t + 50, 100 * t + 60 + w))
    assert vt.validate(_write(tmp_path, rows)) is None


def test_violated_recurrence_edge_is_reported(tmp_path):
    rows = [(0, 0, "fwd", 0, "publish", 50, 200), (0, 1, "fwd", 0, "wait", 100, 150),
            (0, 1, "fwd", 0, "publish", 300, 310)]
    v = vt.validate(_write(tmp_path, rows))
    assert v is not None and "edge violated" in v


def test_violated_layer_edge_is_reported(tmp_path):
    rows = [(0, 0, "fwd", 0, "publish", 50, 200), (1, 0, "fwd", 0, "offload", 150, 160),
            (1, 0, "fwd", 0, "publish", 300, 310)]
    v = vt.validate(_write(tmp_path, rows))
    assert v is not None and "off-critical" in v

"""CPU: profiles/validate_trace.py (the reference's validate_trace, scheduler.hpp:371-404, over
build_graph(L, T, 1)) accepts a consistent trace in the write_trace_csv schema and reports
missing / duplicate tasks and violated forward and backward edges (synthetic CSVs)."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location("vt", os.path.join(ROOT, "profiles", "validate_trace.py"))
vt = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(vt)

HDR = "task_layer,task_block,phase,worker,start_ns,end_ns\n"


def wavefront(L, T, reverse=False):
    """A consistent schedule: task (l, t) at diagonal slot l + t (forward) or the mirror."""
    rows = []
    for l in range(L):
        for t in range(T):
            d = (l + t) if not reverse else ((L - 1 - l) + (T - 1 - t))
            if not reverse:
                rows.append((l, t, "INPUT_GEMM", 0, 100 * d, 100 * d + 10))
                rows.append((l, t, "RECURRENT_STEP(0)", 1, 100 * d + 20, 100 * d + 90))
            else:  # reversed graph: the output GEMM (INPUT_GEMM) runs after the step
                rows.append((l, t, "RECURRENT_STEP(0)", 1, 100 * d, 100 * d + 60))
                rows.append((l, t, "INPUT_GEMM", 0, 100 * d + 70, 100 * d + 90))
    return rows


def _write(tmp_path, rows):
    p = tmp_path / "t.csv"
    p.write_text(HDR + "".join(",".join(map(str, r)) + "\n" for r in rows))
    return str(p)


def test_consistent_traces_pass(tmp_path):
    assert vt.validate(_write(tmp_path, wavefront(3, 4)), 3, 4, "fwd") is None
    assert vt.validate(_write(tmp_path, wavefront(3, 4, True)), 3, 4, "bwd") is None


def test_missing_and_duplicate_tasks_are_reported(tmp_path):
    rows = wavefront(2, 3)
    v = vt.validate(_write(tmp_path, rows[:-1]), 2, 3)
    assert v is not None and "records" in v
    v = vt.validate(_write(tmp_path, rows[:-1] + [rows[0]]), 2, 3)
    assert v is not None and "more than once" in v


def test_violated_recurrence_edge_is_reported(tmp_path):
    rows = wavefront(1, 3)
    rows[1] = (0, 0, "RECURRENT_STEP(0)", 1, 20, 250)  # step 0 ends after step 1 starts
    v = vt.validate(_write(tmp_path, rows), 1, 3)
    assert v is not None and "edge violated" in v


def test_violated_layer_edge_is_reported(tmp_path):
    rows = wavefront(2, 2)
    rows = [r if not (r[0] == 1 and r[1] == 0 and r[2] == "INPUT_GEMM") else (1, 0, "INPUT_GEMM", 0, 50, 60)
            for r in rows]  # layer 1's W.x_0 starts before layer 0's step 0 ends
    v = vt.validate(_write(tmp_path, rows), 2, 2)
    assert v is not None and "edge violated" in v


def test_backward_edges_are_reversed(tmp_path):
    # a forward-consistent trace violates the reversed graph
    v = vt.validate(_write(tmp_path, wavefront(2, 3)), 2, 3, "bwd")
    assert v is not None and "edge violated" in v

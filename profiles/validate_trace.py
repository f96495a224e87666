"""Check a device schedule trace (RW_TRACE CSV / Engine.set_trace_sink records, the reference's
write_trace_csv schema scheduler.hpp:406-417: task_layer,task_block,phase,worker,start_ns,end_ns,
phase INPUT_GEMM | RECURRENT_STEP(k)) the way the reference's validate_trace does
(scheduler.hpp:371-404): the trace covers every task of the graph exactly once, and for every
edge u -> v the dependency's end stamp does not exceed the dependent's start stamp.

The graph is build_graph(L, T, 1) (scheduler.hpp:96-155; the device wavefront's unit of work is
one step), reversed for the backward trace (reverse_graph, scheduler.hpp:160-170):
  forward : RECURRENT_STEP(l-1, t) -> INPUT_GEMM(l, t) -> RECURRENT_STEP(l, t),
            RECURRENT_STEP(l, t-1) -> RECURRENT_STEP(l, t)
  backward: every edge reversed.
Usage: python profiles/validate_trace.py trace.csv L T [fwd|bwd]  -> "ok" or the first violation.
"""
import csv
import re
import sys


def graph_edges(L: int, T: int, reverse: bool):
    """(u, v) edges of build_graph(L, T, 1) as ((phase, layer, step), ...) keys."""
    edges = []
    for l in range(L):
        for t in range(T):
            if l > 0:
                edges.append((("R", l - 1, t), ("I", l, t)))
            edges.append((("I", l, t), ("R", l, t)))
            if t > 0:
                edges.append((("R", l, t - 1), ("R", l, t)))
    return [(v, u) for u, v in edges] if reverse else edges


def parse(rows):
    """-> {(phase, layer, step): (start, end, worker)}, or an error string."""
    tasks = {}
    for r in rows:
        ph = r["phase"]
        l, j = int(r["task_layer"]), int(r["task_block"])
        if ph == "INPUT_GEMM":
            key = ("I", l, j)
        else:
            m = re.fullmatch(r"RECURRENT_STEP\((\d+)\)", ph)
            if not m:
                return f"unknown phase label {ph!r}"
            key = ("R", l, j + int(m.group(1)))  # block width 1: step_k is 0
        if key in tasks:
            return f"task {key} appears more than once"
        s, e = int(r["start_ns"]), int(r["end_ns"])
        if e < s:
            return f"task {key} ends before it starts"
        tasks[key] = (s, e, int(r["worker"]))
    return tasks


def validate_rows(rows, L: int, T: int, direction: str = "fwd", slack_ns: int = 0):
    """slack_ns: allowed end-after-start overlap -- 0 is the reference's rule; device traces
    from %globaltimer (32 ns ticks, sampled per SM) pass a couple of ticks for clock skew."""
    tasks = parse(rows)
    if isinstance(tasks, str):
        return tasks
    want = {(p, l, t) for p in ("I", "R") for l in range(L) for t in range(T)}
    if len(tasks) != len(want):
        return f"trace has {len(tasks)} records, graph has {len(want)} tasks"
    missing = want - set(tasks)
    if missing:
        return f"task {sorted(missing)[0]} is missing"
    for u, v in graph_edges(L, T, direction == "bwd"):
        if tasks[u][1] > tasks[v][0] + slack_ns:
            return (f"edge violated: {u} ends at {tasks[u][1]} ns after {v} starts at {tasks[v][0]} ns")
    return None


def validate(path: str, L: int, T: int, direction: str = "fwd", slack_ns: int = 0):
    with open(path) as f:
        return validate_rows(list(csv.DictReader(f)), L, T, direction, slack_ns)


if __name__ == "__main__":
    v = validate(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] if len(sys.argv) > 4 else "fwd")
    print("ok" if v is None else v)
    sys.exit(0 if v is None else 1)

"""Check a device trace (RW_TRACE CSV, the reference's trace schema scheduler.hpp:411-417 plus a
`span` column) against the wavefront's edges, the way the reference's `validate_trace`
(scheduler.hpp:371-404) checks a CPU schedule: every (direction, layer, step) task is present
for every worker, and a dependency's end stamp never exceeds its dependent's start stamp.

Edges (device %globaltimer, same clock on every SM):
  * recurrence: all critical CTAs of (layer l, step t-1) -- forward; t+1 backward -- release
    ("publish" end) before any critical CTA of (l, t) sees its operand ("wait" end);
  * forward layer input: critical CTAs of (l-1, t) publish before the off-critical CTAs of
    (l, t) see their operand ("offload" start).
Usage: python profiles/validate_trace.py trace.csv  -> prints "ok" or the first violation.
"""
import csv
import sys
from collections import defaultdict


def validate(path: str):
    rows = list(csv.DictReader(open(path)))
    pub = defaultdict(list)      # (phase, layer, step) -> publish ends (critical CTAs)
    seen = defaultdict(list)     # (phase, layer, step) -> wait ends (critical CTAs)
    offseen = defaultdict(list)  # (phase, layer, step) -> offload starts (off-critical CTAs)
    workers = defaultdict(set)
    for r in rows:
        key = (r["phase"], int(r["task_layer"]), int(r["task_block"]))
        s, e = int(r["start_ns"]), int(r["end_ns"])
        if e < s:
            return f"span {r['span']} of {key} worker {r['worker']} ends before it starts"
        if r["span"] == "publish":
            pub[key].append(e)
            workers[key].add(r["worker"])
        elif r["span"] == "wait":
            seen[key].append(e)
        elif r["span"] == "offload":
            offseen[key].append(s)
    if not pub:
        return "trace has no publish records"
    counts = {len(v) for v in workers.values()}
    if len(counts) != 1:
        return f"tasks have different numbers of publishing workers: {sorted(counts)}"
    for (ph, l, t), ends in pub.items():
        nxt = (ph, l, t + 1) if ph == "fwd" else (ph, l, t - 1)
        if nxt in seen and max(ends) > min(seen[nxt]):
            return (f"edge violated: ({ph} layer {l}, step {t}) publishes until {max(ends)} ns after "
                    f"(layer {l}, step {nxt[2]}) starts at {min(seen[nxt])} ns")
        if ph == "fwd" and (ph, l + 1, t) in offseen and max(ends) > min(offseen[(ph, l + 1, t)]):
            return (f"edge violated: (fwd layer {l}, step {t}) publishes until {max(ends)} ns after the "
                    f"off-critical CTAs of (layer {l + 1}, step {t}) start at {min(offseen[(ph, l + 1, t)])} ns")
    return None


if __name__ == "__main__":
    v = validate(sys.argv[1])
    print("ok" if v is None else v)
    sys.exit(0 if v is None else 1)

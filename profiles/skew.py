"""Publish skew per wavefront step from a device trace CSV (RW_TRACE): spread between the first
and the last critical CTA publishing (layer, step). Usage: python profiles/skew.py trace.csv"""
import csv
import statistics
import sys
from collections import defaultdict

rows = list(csv.DictReader(open(sys.argv[1])))
pub = defaultdict(list)
for r in rows:
    if r["span"] == "publish":
        pub[(r["phase"], int(r["task_layer"]), int(r["task_block"]))].append(int(r["end_ns"]))
for ph in ("fwd", "bwd"):
    v = [sorted(x) for k, x in pub.items() if k[0] == ph and len(x) > 1]
    if not v:
        continue
    spread = [x[-1] - x[0] for x in v]
    tail = [x[-1] - x[len(x) // 2] for x in v]
    print(f"{ph}: CTAs per step {statistics.median([len(x) for x in v])}, publish spread median "
          f"{statistics.median(spread)} ns (p90 {sorted(spread)[int(0.9 * len(spread))]}), last - median "
          f"{statistics.median(tail)} ns")

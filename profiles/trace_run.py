"""Run one config-B training pass with the device span trace on (RW_TRACE_SPANS) and summarise where a
recurrent step's time goes. Usage (GPU box): python profiles/trace_run.py [bf16|fp32] [out.csv] [bench config, default B]
"""
import csv
import os
import statistics
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def summarize(path):
    rows = list(csv.DictReader(open(path)))
    spans = defaultdict(list)
    by_step = defaultdict(lambda: [1 << 62, 0])
    for r in rows:
        d = int(r["end_ns"]) - int(r["start_ns"])
        spans[(r["phase"], r["span"])].append(d)
        key = (r["phase"], int(r["task_layer"]), int(r["task_block"]))
        if r["span"] == "publish":
            by_step[key][1] = max(by_step[key][1], int(r["end_ns"]))
        if r["span"] == "wait":
            by_step[key][0] = min(by_step[key][0], int(r["start_ns"]))
    out = {}
    for (ph, sp), v in sorted(spans.items()):
        out[f"{ph}.{sp}.median_ns"] = statistics.median(v)
        out[f"{ph}.{sp}.p90_ns"] = sorted(v)[int(0.9 * (len(v) - 1))]
    for ph in ("fwd", "bwd"):
        ends = sorted(v[1] for k, v in by_step.items() if k[0] == ph and v[1])
        starts = sorted(v[0] for k, v in by_step.items() if k[0] == ph and v[0] < (1 << 62))
        if ends:
            out[f"{ph}.span_total_us"] = (ends[-1] - starts[0]) / 1e3
            # publish-to-publish interval of consecutive steps of one layer (the tick)
            lay = defaultdict(list)
            for k, v in by_step.items():
                if k[0] == ph and v[1]:
                    lay[k[1]].append((k[2], v[1]))
            ticks = []
            for l, lst in lay.items():
                lst.sort()
                ticks += [abs(b[1] - a[1]) for a, b in zip(lst, lst[1:])]
            out[f"{ph}.tick_median_ns"] = statistics.median(ticks)
    # flag propagation: last publish of (layer, t-1) over the layer's critical CTAs -> each
    # CTA's wait end at t (forward; backward steps run t descending)
    pub, seen = defaultdict(int), defaultdict(list)
    for r in rows:
        key = (r["phase"], int(r["task_layer"]), int(r["task_block"]))
        if r["span"] == "publish":
            pub[key] = max(pub[key], int(r["end_ns"]))
        if r["span"] == "wait":
            seen[key].append(int(r["end_ns"]))
    # skew between the critical CTAs of one (layer, step): first to last publish
    pubs = defaultdict(list)
    for r in rows:
        if r["span"] == "publish":
            pubs[(r["phase"], int(r["task_layer"]), int(r["task_block"]))].append(int(r["end_ns"]))
    for ph in ("fwd", "bwd"):
        sp = [max(v) - min(v) for k, v in pubs.items() if k[0] == ph and len(v) > 1]
        if sp:
            out[f"{ph}.publish_spread_median_ns"] = statistics.median(sp)
            out[f"{ph}.publish_spread_p90_ns"] = sorted(sp)[int(0.9 * (len(sp) - 1))]
    for ph, d in (("fwd", -1), ("bwd", 1)):
        props = []
        for (p2, l, t), v in seen.items():
            prev = pub.get((p2, l, t + d))
            if p2 == ph and prev:
                props += [x - prev for x in v]
        if props:
            out[f"{ph}.prop_from_last_publish_median_ns"] = statistics.median(props)
            out[f"{ph}.prop_from_last_publish_min_ns"] = min(props)
    return out


def main():
    prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
    path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"trace_{prec}.csv")
    os.environ["RW_TRACE_SPANS"] = path
    from paper_1604_01946_b200 import Engine, LadderConfig, init_params, make_dy, make_input
    name = sys.argv[3] if len(sys.argv) > 3 else "B"
    import bench
    cfg = LadderConfig(**bench.CONFIGS[name], seed=42)
    eng = Engine(cfg, precision=prec)
    eng.set_params(init_params(cfg))
    eng.upload_inputs(make_input(cfg), make_dy(cfg))
    for _ in range(3):
        eng.run_pass(2)
    eng.sync()  # writes the CSV of the last pass
    print(eng.describe())
    for k, v in summarize(path).items():
        print(f"{k}: {v}")


if __name__ == "__main__":
    main()

"""Summarise ncu captures (gpurun_out/prof_*.ncu-rep) and the launch list (launches.csv) into
the committed evidence under profiles/<round>/. Runs here (no GPU): needs `ncu` for -i.

  python profiles/summarize.py r01 [gpurun_out] [output json name]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor_pipe_active_pct"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_mem_active_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster_x"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("sm__cycles_active.avg", "sm_cycles_active"),
]


KEYS += [
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_cycles_active_pct"),
    ("sm__ops_path_tensor_src_fp16_dst_fp32.avg.pct_of_peak_sustained_elapsed", "tensor_fp16_ops_pct"),
    ("sm__ops_path_tensor_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed", "tensor_bf16_ops_pct"),
]


def ncu_raw(rep):
    """rep: an .ncu-rep (read with ncu -i) or an already exported `--page raw --csv` file."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                d[name] = f"{v[i]} {u[i]}".strip()
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = defaultdict(lambda: [0.0, 0])
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0]
        unit = r[hdr.index("Metric Unit")]
        val = float(r[hdr.index("Metric Value")].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        out[name][0] += val * scale
        out[name][1] += 1
    tot = sum(v[0] for v in out.values()) or 1.0
    return sorted(((k, v[0], v[1], v[0] / tot) for k, v in out.items()), key=lambda x: -x[1])


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    out_name = sys.argv[3] if len(sys.argv) > 3 else "ncu_summary.json"
    root = os.path.dirname(os.path.abspath(__file__))
    dst = os.path.join(root, rnd)
    os.makedirs(dst, exist_ok=True)
    summary = {}
    for f in sorted(os.listdir(src)):
        if f.startswith("prof_") and (f.endswith(".ncu-rep") or f.endswith("_raw.csv")):
            summary[f] = ncu_raw(os.path.join(src, f))
    for f in sorted(os.listdir(src)):
        if f.startswith("launches") and f.endswith(".csv"):
            summary["launch_list_" + f[:-4]] = [
                {"kernel": k, "total_us": round(t, 2), "launches": n, "share": round(s, 4)}
                for k, t, n, s in launches(os.path.join(src, f))]
    with open(os.path.join(dst, out_name), "w") as fh:
        json.dump(summary, fh, indent=1)
    for k, v in summary.items():
        print(k)
        for row in v:
            print("   ", row)


if __name__ == "__main__":
    main()

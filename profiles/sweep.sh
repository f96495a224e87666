#!/bin/bash
# Run ON THE GPU BOX from the repo root: one bench.py line per configured shape (no CPU
# baseline), summarised as a table on stdout.
# Usage: [PRECISION=bf16|fp32] bash profiles/sweep.sh [configs...]
cfgs=${*:-"A B C128 C256 C1024 C2048 D1 D4 E"}
prec=${PRECISION:-bf16}
mkdir -p gpurun_out/sweep
for c in $cfgs; do
  steps=20; [[ $c == E ]] && steps=10
  timeout -s KILL 900 python bench.py --config $c --steps $steps --precision $prec --no-cpu-baseline \
      > gpurun_out/sweep/${c}_$prec.json 2> gpurun_out/sweep/${c}_$prec.err
done
python - $prec $cfgs <<'PY'
import json, sys
prec = sys.argv[1]
print(f"precision {prec}")
print("| config | schedule (fwd / bwd) | ms / pass | TFLOP/s | e2e TFLOP/s | % burst / sustained peak | roofline bound, frac | SM MHz |")
print("|---|---|---|---|---|---|---|---|")
for c in sys.argv[2:]:
    try:
        d = json.loads(open(f"gpurun_out/sweep/{c}_{prec}.json").read().strip().split("\n")[-1])
    except Exception as e:
        print(f"| {c} | failed: {e} |"); continue
    sc = d["config"]["schedule"]; r = d["roofline"]
    print(f"| {c} {d['config']['workload'].split(' LSTM')[0]} | {sc['fwd_schedule']} / {sc['bwd_schedule']} | "
          f"{d['ms_per_step']:.2f} | {d['value']:.0f} | {d['e2e']['value']:.0f} | "
          f"{d['config']['pct_of_bf16_peak']:.1f} / {d['config']['pct_of_bf16_peak_sustained']:.1f} | "
          f"{r['bound']} {r['frac']:.2f} | {d['clocks']['sm_mhz']:.0f} |")
PY

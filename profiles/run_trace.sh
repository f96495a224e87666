#!/bin/bash
# GPU box: span traces (where a recurrent step's time goes) for config B in both precisions.
mkdir -p gpurun_out
for p in fp32 bf16; do
  timeout -s KILL 300 python profiles/trace_run.py $p gpurun_out/spans_$p.csv > gpurun_out/spans_$p.txt 2>&1
  rm -f gpurun_out/spans_$p.csv  # summarised above; the CSV is ~6 MB
done

#!/bin/bash
# GPU box: fp32 forward activation variants (RW_CL_DEBUG bits, rec_cluster.cuh): cell-phase time
# (profiles/trace_run.py) and config-B parity (profiles/parity_probe.py) per variant
mkdir -p gpurun_out
: > gpurun_out/cellx_summary.txt
for bits in ${BITS:-0 1024 2048 4096 5120 7168}; do
  RW_CL_DEBUG=$bits timeout -s KILL 300 python profiles/trace_run.py fp32 gpurun_out/cellx_$bits.csv > gpurun_out/cellx_$bits.txt 2>&1
  RW_CL_DEBUG=$bits timeout -s KILL 300 python profiles/parity_probe.py fp32 > gpurun_out/cellp_$bits.txt 2>&1
  { echo "== bits $bits"; grep "fwd.cell.median\|fwd.tick" gpurun_out/cellx_$bits.txt; sed -n 2,3p gpurun_out/cellp_$bits.txt; } >> gpurun_out/cellx_summary.txt
done

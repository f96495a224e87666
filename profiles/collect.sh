#!/bin/bash
# Run ON THE GPU BOX (via gpurun) from the repo root. Produces, under gpurun_out/:
#   bench.json      one bench.py line (the numbers; never taken under a profiler)
#   launches.csv    ncu per-launch device times of the same command (cold-cache, serialised)
#   prof_*.ncu-rep  one `ncu --set full` capture per hot kernel (read back with ncu -i)
# Usage: [KERNELS="k1 k2"] profiles/collect.sh [bench|launches|full|all] [extra bench args]
# (config E: KERNELS="k_lstm_fwd k_lstm_bwd k_gemm_p2" profiles/collect.sh all --config E)
set -u
what=${1:-all}; shift || true
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline $*"
if [[ $what == bench || $what == all ]]; then
  timeout -s KILL 600 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
fi
if [[ $what == launches || $what == all ]]; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv $B --steps 2 --warmup 1 > gpurun_out/launches.out 2>&1
fi
KERNELS=${KERNELS:-"k_cl_fwd k_cl_bwd k_gemm_tc"}
if [[ $what == full || $what == all ]]; then
  for k in $KERNELS; do
    timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
        -o gpurun_out/prof_$k -f $B --steps 1 --warmup 1 > gpurun_out/prof_$k.out 2>&1
  done
fi

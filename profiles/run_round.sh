#!/bin/bash
# Run ON THE GPU BOX (gpurun) from the repo root: GPU tests, then the default bench line.
# Usage: bash profiles/run_round.sh [tests|bench|sweep ...]   (default: tests bench)
set -u
mkdir -p gpurun_out
what=${*:-"tests bench"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
for w in $what; do
  case $w in
    tests) export RW_PARITY_LOG=gpurun_out/parity.jsonl; timeout -s KILL ${PYTEST_TIMEOUT:-1500} python -m pytest ${PYTEST_FILES:-tests} -m gpu -q -rs ${PYTEST_X--x} ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
           echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log ;;
    bench) timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
           echo "bench rc=$?" >> gpurun_out/bench.err ;;
    sweep) PRECISION=${PRECISION:-fp32} bash profiles/sweep.sh ${CONFIGS:-} > gpurun_out/sweep_${PRECISION:-fp32}.md 2>&1 ;;
  esac
done

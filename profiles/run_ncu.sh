#!/bin/bash
# GPU box: ncu evidence for the headline config: the launch list of a short bench run, and one
# --set full capture (with source) per hot kernel, summarised to CSV right away (the .ncu-rep
# files are large; only the summaries and the smallest report come back).
# Usage: [KERNELS="k_cl_fwd k_cl_bwd"] [PREC=fp32] [KEEP_REP=1] [SOURCE=1] [NO_LAUNCHES=1] bash profiles/run_ncu.sh [extra bench args]
mkdir -p gpurun_out
PREC=${PREC:-fp32}
B="python bench.py --no-cpu-baseline --single-precision --precision $PREC $*"
[ -n "${NO_LAUNCHES:-}" ] || timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$PREC.csv $B --steps 2 --warmup 1 > gpurun_out/launches_$PREC.out 2>&1
for k in ${KERNELS:-k_cl_fwd k_cl_bwd}; do
  rep=gpurun_out/prof_${k}_$PREC
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
      -o $rep -f $B --steps 1 --warmup 3 > $rep.out 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > ${rep}_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > ${rep}_details.csv 2>/dev/null
  if [ -n "${SOURCE:-}" ]; then  # per-line / per-instruction warp-stall samples
    ncu -i $rep.ncu-rep --page source --csv --print-source cuda > ${rep}_src_cuda.csv 2>/dev/null
    ncu -i $rep.ncu-rep --page source --csv --print-source sass > ${rep}_src_sass.csv 2>/dev/null
  fi
  [ -n "${KEEP_REP:-}" ] || rm -f $rep.ncu-rep
done
du -sh gpurun_out

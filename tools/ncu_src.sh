#!/bin/bash
# ncu --set full with source of one launch each of the step's main kernels
# (after the warm-up frames; skip counts for the default four contexts of B = 64):
# tools/ncu_src.sh TAG [bench args]
# Leaves gpurun_out/src_TAG_<kernel>.ncu-rep and the SASS-level source pages as CSV.
TAG=${1:-src}; shift
mkdir -p gpurun_out
for KS in k_sgm_sweep:26 k_sgm_row:26 k_wta_runs:13 k_cost_runs:13; do
  K=${KS%%:*}; S=${KS##*:}; N=${K%%<*}
  timeout 900 ncu --set full --import-source on --clock-control none \
      -k regex:"$K" -s $S -c 1 -f -o gpurun_out/src_${TAG}_${N} \
      python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/src_${TAG}_${N}.log 2>&1
  echo "$K ncu rc=$?"
  ncu -i gpurun_out/src_${TAG}_${N}.ncu-rep --page source --csv --print-source sass \
      > gpurun_out/src_${TAG}_${N}_sass.csv 2>/dev/null
  ncu -i gpurun_out/src_${TAG}_${N}.ncu-rep --page raw --csv > gpurun_out/src_${TAG}_${N}_raw.csv 2>/dev/null
done
ls -la gpurun_out | tail -20

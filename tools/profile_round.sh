#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   tools/profile_round.sh TAG [B]
# 1. bench line (no profiler)             -> gpurun_out/prof_TAG_bench.json
# 2. launch list of the same command       -> gpurun_out/prof_TAG_launches.csv
#    (ncu --metrics gpu__time_duration.sum --clock-control none)
# 3. ncu --set full of one timed step's aggregation + other hot kernels
#    (launches after the warm-up)          -> gpurun_out/prof_TAG_full.ncu-rep
set -e
TAG=$1; B=${2:-64}
CMD="python bench.py --steps 2 --warmup 3 --batch $B --no-cpu --no-e2e"
$CMD > gpurun_out/prof_${TAG}_bench.json 2> gpurun_out/prof_${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof_${TAG}_launches.csv $CMD > /dev/null 2>&1
# warm-up = 3 steps (frame 0 full range + 2); 19 matching launches per step (12 aggregation launches: 6 jobs x 2
# regime variants) of every step: skip 4 steps' worth, capture one step
ncu --set full --import-source on --clock-control none -k regex:"k_sgm_grp4|k_cost_runs|k_wta_runs|k_warp|k_resolve|k_fill_v|k_checks" \
    -s $((3 * 19)) -c 19 -o gpurun_out/prof_${TAG}_full $CMD > gpurun_out/prof_${TAG}_ncu.log 2>&1

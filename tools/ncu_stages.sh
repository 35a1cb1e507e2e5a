#!/bin/bash
# ncu --set full (with source) of one timed step's non-aggregation kernels
# (cost, WTA, prediction, checks): tools/ncu_stages.sh TAG [bench args]
TAG=${1:-stages}; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"k_cost_runs|k_wta_runs|k_warp_zmax|k_checks_fuse|k_resolve_fill_h|k_fill_v" -s 18 -c 6 \
    -o gpurun_out/stages_${TAG} \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/stages_${TAG}.log 2>&1
echo "ncu stages rc=$?"

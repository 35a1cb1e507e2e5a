#!/bin/bash
# ncu --set full (with source) of one timed step's aggregation launches
# (both sweeps + both row jobs, both regime variants) of the default bench: tools/ncu_agg.sh TAG [bench args]
TAG=${1:-agg}; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"k_sgm_sweep|k_sgm_grp4" -s 18 -c 6 -o gpurun_out/full_${TAG} \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/full_${TAG}.log 2>&1
echo "ncu full rc=$?"

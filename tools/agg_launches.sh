#!/bin/bash
# launch list of a short bench (aggregation kernels): tools/agg_launches.sh TAG [bench args]
TAG=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_${TAG}.csv \
    timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/l_${TAG}.out 2>&1
python tools/launch_table.py gpurun_out/l_${TAG}.csv 4

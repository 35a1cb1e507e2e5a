#!/bin/bash
# One GPU-box pass (run from the repo root under gpurun):
#   tools/gpu_check.sh TAG [tests|notests]
# pytest -m gpu, the default bench line, the hash-stamped ncu traffic of one
# bench step (tools/ncu_traffic.py) and the launch list of a short bench.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ "${2:-tests}" = tests ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/gputest_${TAG}.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/gputest_${TAG}.log
fi
# traffic first: the bench line then carries the ncu DRAM bytes of this build
timeout 900 python tools/ncu_traffic.py --tag ${TAG} > gpurun_out/ncu_traffic_${TAG}.log 2>&1
echo "ncu traffic rc=$?"; cat gpurun_out/ncu_traffic_${TAG}.log | tail -12
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_all_${TAG}.json 2>/dev/null
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches_${TAG}.out 2>&1
echo "launch list rc=$?"

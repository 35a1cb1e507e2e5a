timeout 1500 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_full_configs.py tests/test_gpu_c_abi.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu > gpurun_out/bench_g4.json 2> gpurun_out/bench_g4.err; tail -c 400 gpurun_out/bench_g4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_g4.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['ms_per_step'], d['config']['contexts_per_gpu'], d['stage_ms_per_step'], d['gpu_launches'])
PY

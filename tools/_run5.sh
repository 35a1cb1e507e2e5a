timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_bench_path.py -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do for v in 0 1; do echo "ROW=$v $(ES_SGM_ROW=$v tools/quick_bench.sh 64)"; done; done

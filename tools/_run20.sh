for r in 1 2; do for B in 8 16; do for v in 1 2; do echo "B=$B ROW=$v $(ES_SGM_ROW=$v tools/quick_bench.sh $B)"; done; done; done
timeout 1500 python -m pytest tests/test_gpu_sweep.py -m gpu -x -q 2>&1 | tail -3

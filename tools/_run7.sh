timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_bench_path.py -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do for v in 0 1; do echo "ROW=$v $(ES_SGM_ROW=$v tools/quick_bench.sh 64)"; done; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_sgm_row|k_sgm_grp4" -s 13 -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>/dev/null | grep -i "k_sgm" | cut -d, -f5,13- | cut -c1-200

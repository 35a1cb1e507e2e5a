timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sgm_row -s 13 -c 2 -f -o gpurun_out/src_row python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/src_row.log 2>&1
ncu -i gpurun_out/src_row.ncu-rep --page source --csv --print-source sass > gpurun_out/src_row_sass.csv 2>/dev/null
ncu -i gpurun_out/src_row.ncu-rep --page raw --csv > gpurun_out/src_row_raw.csv 2>/dev/null

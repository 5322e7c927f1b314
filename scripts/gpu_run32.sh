python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep2d -c 2 -o gpurun_out/prof_sweep2_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_sweep.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/prof_sweep2_c2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed 2>&1 | tail -3

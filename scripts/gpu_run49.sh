python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smooth_small -c 2 -o gpurun_out/prof_small_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_small.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/prof_small_c2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,smsp__issue_active.avg.pct_of_peak_sustained_active 2>&1 | tail -2

python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep2d -c 8 -o gpurun_out/prof_sweep_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_sweep.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/prof_sweep_c2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,smsp__average_warp_latency_issue_stalled_barrier,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio > gpurun_out/sweep_raw.csv 2>&1
head -20 gpurun_out/sweep_raw.csv

# ncu --set full of the finest-level FD pass (c2)
python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fd_pass_dmma_kernel -c 1 -o gpurun_out/prof_fd_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_fd.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/prof_fd_c2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active 2>&1 | tail -3

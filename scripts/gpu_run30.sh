python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c2_warm.csv python scripts/solve_once.py c2 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_c2_warm.csv > gpurun_out/launches_c2_warm.txt; head -12 gpurun_out/launches_c2_warm.txt

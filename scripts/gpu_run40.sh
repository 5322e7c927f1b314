python scripts/precond_once.py c4 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c4_warm.csv python scripts/precond_once.py c4 > gpurun_out/ncu_c4.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_c4_warm.csv > gpurun_out/launches_c4_warm.txt; head -24 gpurun_out/launches_c4_warm.txt

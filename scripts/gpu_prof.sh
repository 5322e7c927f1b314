CFG=${1:-c2}
python scripts/solve_once.py $CFG 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fd_pass -c 1 -o gpurun_out/prof_fd_$CFG python scripts/solve_once.py $CFG 1 > gpurun_out/ncu_fd.log 2>&1; echo "fd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:spmv -c 1 -o gpurun_out/prof_spmv_$CFG python scripts/solve_once.py $CFG 1 > gpurun_out/ncu_spmv.log 2>&1; echo "spmv rc=$?"

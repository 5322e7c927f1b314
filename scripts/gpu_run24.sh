timeout 900 ncu --set full --import-source on --clock-control none -k regex:fd_pass_dmma -s 0 -c 4 -o gpurun_out/prof_fd3_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_fd3.log 2>&1
echo "ncu rc=$?"

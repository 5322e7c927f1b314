timeout 900 ncu --set full --import-source on --clock-control none -k regex:fd_pass_dmma -s 0 -c 2 -o gpurun_out/prof_fd4_c2 python scripts/precond_once.py c2 > gpurun_out/ncu_fd4.log 2>&1
echo "ncu rc=$?"

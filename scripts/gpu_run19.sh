timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmv_kernel -c 2 -o gpurun_out/prof_spmv_small_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_small.log 2>&1
echo "ncu rc=$?"

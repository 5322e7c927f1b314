timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmv_tma_half -s 0 -c 1 -o gpurun_out/prof_spmv_c4 python scripts/precond_once.py c4 > gpurun_out/ncu_sc4.log 2>&1
echo "ncu rc=$?"

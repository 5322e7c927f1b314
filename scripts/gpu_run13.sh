timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=long -x -k "half_band or L5 or L3" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -30
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmv_tma_half -c 8 -o gpurun_out/prof_spmv_half_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_spmv_half.log 2>&1
echo "ncu rc=$?"

timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=long -x -k "pcg and c2-p4-L5" 2>&1 | grep -E "^E|assert|passed|failed" | head -30
PMG_FULL_BAND=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=line -x -k "pcg and c2-p4-L5" 2>&1 | tail -3
python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmv_tma_half -s 20 -c 1 -o gpurun_out/prof_spmv_half_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_spmv_half.log 2>&1
echo "ncu rc=$?"

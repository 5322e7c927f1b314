python -m pytest tests/test_gpu_parity.py -q --tb=short -k "pcg" 2>&1 | grep -E "max \|dr|passed|failed" > gpurun_out/pytest.log; cat gpurun_out/pytest.log
python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fd_pass -c 1 -o gpurun_out/prof_fd_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_fd.log 2>&1; echo "fd rc=$?"

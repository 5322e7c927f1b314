python -m pytest tests/test_gpu_parity.py -q --tb=short -k "pcg" 2>&1 | grep -E "max \|dr|passed|failed" > gpurun_out/pytest.log; cat gpurun_out/pytest.log
python scripts/breakdown.py c2 3 2>&1 | head -40

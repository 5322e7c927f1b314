timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x --tb=short 2>&1 | tail -25
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --tb=short 2>&1 | tail -3

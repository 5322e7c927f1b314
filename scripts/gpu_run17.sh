for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "L3 or L5" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5; done
timeout 1800 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -20

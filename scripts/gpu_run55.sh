# full-size property tests (c2, c4)
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q --tb=short 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error|assert" | head -20

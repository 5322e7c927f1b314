timeout 900 python -m pytest tests/test_gpu_multirank.py -q --tb=short -k "concurrent" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10

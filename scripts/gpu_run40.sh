timeout 1200 python -m pytest tests/test_gpu_parity.py -q --tb=short -k "line_sweep" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10
echo "== split"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv L[67]|wall"

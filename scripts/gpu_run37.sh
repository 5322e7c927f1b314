timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -k "transfers or cycle or pcg" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10
echo "== new"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "transfer L[4567]|wall|Error"

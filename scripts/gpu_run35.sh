timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "transfers or cycle or pcg" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
echo "== tiles"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "transfer L[4567]|wall"

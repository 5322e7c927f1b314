timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "smooth and (c2 or c3 or c4)" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
echo "== default"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "fd_interior|wall"
echo "== ntc11"; PMG_FD_NTC=11 timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "fd_interior|wall"

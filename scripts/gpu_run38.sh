timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -k "smooth or cycle" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10
echo "== c2"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "fd_interior L[567]|wall"
echo "== c4"; timeout 600 python scripts/breakdown.py c4 2 2>&1 | grep -E "fd_interior L[345]|wall"

timeout 1200 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "smooth or cycle or pcg" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
echo "== small 4608"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "fd_interior|interface_pieces|wall"
echo "== small 2048"; PMG_FD_SMALL_MAX=2048 timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "fd_interior|interface|wall"
echo "== c4"; timeout 600 python scripts/breakdown.py c4 2 2>&1 | grep -E "fd_interior|interface|wall"

timeout 1200 python -m pytest tests/test_gpu_parity.py -q --tb=short -k "apply_op or half_band or cycle or pcg" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10
for v in 1 0; do echo "== deep $v"; PMG_HALF_DEEP=$v timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv L[1-5]|wall"; done
for v in 1 0; do echo "== c4 deep $v"; PMG_HALF_DEEP=$v timeout 600 python scripts/breakdown.py c4 2 2>&1 | grep -E "spmv L[1-5]|wall"; done

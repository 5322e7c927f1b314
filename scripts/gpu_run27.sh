# persistent coarse cycle: parity, timing on/off
timeout 1500 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "cycle or pcg" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in c2 c4; do
echo "== $cfg cc"; timeout 600 python scripts/breakdown.py $cfg 3 2>&1 | grep -E "wall|coarse"
echo "== $cfg no cc"; PMG_NO_COARSE_CYCLE=1 timeout 600 python scripts/breakdown.py $cfg 3 2>&1 | grep -E "wall"
done

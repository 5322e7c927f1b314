# golden-fixture GPU parity + smoke
timeout 900 python -m pytest tests/test_golden.py -m gpu -q --tb=short 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

python -m pytest tests/test_gpu_parity.py -q --tb=short -x 2>&1 | tail -3
python scripts/breakdown.py c2 3 2>&1 | head -24

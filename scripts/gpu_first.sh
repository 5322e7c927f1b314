nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_parity.py -q -x --tb=short -k "lshape or fichera-p2 or c1" 2>&1 | tail -30
python -m pytest tests/test_gpu_parity.py -q --tb=line 2>&1 | tail -40

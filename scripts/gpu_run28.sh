timeout 1200 python -m pytest tests/test_gpu_assembly.py -q --tb=short -x 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10
timeout 900 python scripts/assembly_bench.py c2 c4 2>&1 | tail -3 | tee gpurun_out/assembly_bench.txt

timeout 1500 python -m pytest tests/test_gpu_parity.py -q --tb=short -k "line_sweep or c2 or c1" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
timeout 900 python scripts/determinism.py 5 2>&1 | tail -3
echo "== sweep"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv L[67]|wall"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print('c2', d['ms_per_step'], d['roofline']['avg_ms'], d['roofline']['frac'])"

# line-sweep SpMV v2 (chunk stages): parity, per-level spmv on/off, bench
timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "line_sweep" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
echo "== sweep"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv|wall"
echo "== nosweep"; PMG_SWEEP=0 timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv|wall"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_sweep.json 2> gpurun_out/bench_c2_sweep.err; python -c "import json;d=json.load(open('gpurun_out/bench_c2_sweep.json'));print('sweep ms',d['ms_per_step'], d['roofline']['avg_ms'], d['roofline']['frac'])"

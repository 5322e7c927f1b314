timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "line_sweep or half_band or c2 or c1" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
echo "== sweep"; timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv|wall"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_sweep.json 2> gpurun_out/bench_c2_sweep.err; python -c "import json;d=json.load(open('gpurun_out/bench_c2_sweep.json'));print('sweep ms',d['ms_per_step'], d['roofline']['avg_ms'], d['roofline']['frac'])"
python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep2d -c 1 -o gpurun_out/prof_sweep_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_sweep.log 2>&1; echo "rc=$?"

timeout 1200 python -m pytest tests/test_gpu_parity.py -q --tb=short -k "line_sweep or c2" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10
timeout 900 python scripts/determinism.py 2 2>&1 | tail -1
PMG_SWEEP_MIN_EXT=1 timeout 900 python scripts/determinism.py 2 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print('c2', d['ms_per_step'], round(d['roofline']['frac'],3), round(d['roofline']['avg_ms']*1e3,1))" || tail -3 gpurun_out/b.err

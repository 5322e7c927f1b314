timeout 1200 python -m pytest tests/test_gpu_parity.py -q --tb=short -k "line_sweep" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -10
for cfg in c2 c3p4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$cfg.json'));print('$cfg', d['ms_per_step'], round(d['roofline']['frac'],3), round(d['roofline']['avg_ms']*1e3,1))" || tail -3 gpurun_out/b.err
done

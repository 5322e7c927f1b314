# the other BASELINE configs (parity cases for the bench contract, measured for the record)
for cfg in c1 c3p2 c3p3 c3p4 c3p6 c3p8; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$cfg.json'));print('$cfg', d['ms_per_step'], '%.3g'%d['value'], d['config']['pcg_iterations'], round(d['roofline']['frac'],3), round(d['roofline']['fd_finest']['achieved_tflops'],2))" || tail -3 gpurun_out/bench_$cfg.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=short -k "c3-p3" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20

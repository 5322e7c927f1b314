timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "half_band" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -20
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
python - <<'PY'
import json
for f in ['gpurun_out/bench_c2.json','gpurun_out/bench_c4.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f, d['ms_per_step'], d['value'], r['achieved'], r['avg_ms'], r['spmv_share_of_step'], r['fd_finest']['achieved_tflops'])
PY

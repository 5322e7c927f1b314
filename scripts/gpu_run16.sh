timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "L3 or L5 or lshape or fichera" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -20
for cfg in c2 c4; do
for fsm in 2048 100000; do
PMG_FD_SMALL_MAX=$fsm timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}_$fsm.json 2> gpurun_out/bench_${cfg}_$fsm.err; echo "$cfg $fsm rc=$?"
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_c*_*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f, round(d['ms_per_step'],2), '%.4g'%d['value'], round(r['achieved']), round(r['avg_ms']*1000,1), round(r['spmv_share_of_step'],3), round(r['fd_finest']['achieved_tflops'],2))
PY
python scripts/breakdown.py c2 3 2>&1 | head -30

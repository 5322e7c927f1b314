timeout 1500 python -m pytest tests -m gpu -q --tb=short -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
timeout 600 python scripts/determinism.py 5 2>&1 | tail -1
for cfg in c2 c4; do
for pd in 0 1; do
PMG_NO_PDL=$pd timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}_pdl$pd.json 2> gpurun_out/bench_${cfg}_pdl$pd.err; echo "$cfg $pd rc=$?"
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_c*_pdl*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f, round(d['ms_per_step'],2), '%.4g'%d['value'], round(r['achieved']), round(r['avg_ms']*1000,1), round(r['spmv_share_of_step'],3), round(r['fd_finest']['achieved_tflops'],2))
PY

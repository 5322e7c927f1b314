timeout 1500 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "c2 or c4 or fichera" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for cfg in c2 c4; do
timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}.json 2> gpurun_out/bench_${cfg}.err; echo "$cfg rc=$?"
done
python - <<'PY'
import json,glob
for f in ['gpurun_out/bench_c2.json','gpurun_out/bench_c4.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print(f, round(d['ms_per_step'],2), '%.4g'%d['value'], round(r['achieved']), round(r['avg_ms']*1000,1), round(r['spmv_share_of_step'],3), round(r['fd_finest']['achieved_tflops'],2))
PY
python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c2_warm.csv python scripts/solve_once.py c2 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_c2_warm.csv > gpurun_out/launches_c2_warm.txt; head -6 gpurun_out/launches_c2_warm.txt
python - <<'PY'
import sys
sys.path.insert(0,'scripts')
from ncu_summary import load
rows=load('gpurun_out/launches_c2_warm.csv')
print([ (n[-22:],round(v,1)) for n,v,g in rows if 'fd_pass' in n][:12])
PY

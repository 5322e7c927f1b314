timeout 1500 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "transfers or cycle or pcg" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for v in 0 1; do
PMG_NO_TILED_TRANSFER=$v timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('notiled=$v', round(d['ms_per_step'],2))"
done
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"tile2d|fused" --csv --log-file gpurun_out/tr.csv python scripts/precond_once.py c2 > /dev/null 2>&1
python - <<'PY'
import sys
sys.path.insert(0,'scripts')
from ncu_summary import load
print([(n.split('::')[-1][:12], round(v,1), g.split(',')[0]) for n,v,g in load('gpurun_out/tr.csv')][:16])
PY

for v in 0 1 2; do
PMG_DEBUG_SMOOTH=$v ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:smooth_small -c 8 --csv --log-file gpurun_out/ss_$v.csv python scripts/precond_once.py c2 > /dev/null 2>&1
python - <<PY
import sys
sys.path.insert(0,'scripts')
from ncu_summary import load
print($v, [round(v,1) for n,v,g in load('gpurun_out/ss_$v.csv')])
PY
done

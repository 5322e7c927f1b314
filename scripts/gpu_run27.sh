for cfg in c2 c4; do
for v in "PMG_FD_GROUP=1" "PMG_FD_NTC=9" "PMG_FD_NTC=5"; do
env $v timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$cfg $v', round(d['ms_per_step'],2), round(d['roofline']['fd_finest']['achieved_tflops'],2))"
done; done

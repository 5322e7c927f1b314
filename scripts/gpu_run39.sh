PMG_FD_WM=2 timeout 1500 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "smooth or pcg" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for cfg in c2 c4; do
for v in "PMG_FD_WM=1" "PMG_FD_WM=2" "PMG_FD_WM=2 PMG_FD_NTC=5" "PMG_FD_WM=2 PMG_FD_NTC=11"; do
env $v timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$cfg $v', round(d['ms_per_step'],2), round(d['roofline']['fd_finest']['achieved_tflops'],2))"
done; done

timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q --tb=short -x 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
timeout 600 python scripts/determinism.py 3 2>&1 | tail -1
for cfg in c2 c4; do
for v in "PMG_NO_FUSED_SMOOTH=0" "PMG_NO_FUSED_SMOOTH=1"; do
env $v timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$cfg $v', round(d['ms_per_step'],2), round(d['roofline']['fd_finest']['achieved_tflops'],2))"
done; done

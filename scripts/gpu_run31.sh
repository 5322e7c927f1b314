timeout 1500 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "c2 or c4 or fichera or lshape" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for cfg in c2 c4; do
timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],2), round(d['roofline']['fd_finest']['achieved_tflops'],2))"
done
python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c2_warm.csv python scripts/solve_once.py c2 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_c2_warm.csv > gpurun_out/launches_c2_warm.txt; head -8 gpurun_out/launches_c2_warm.txt

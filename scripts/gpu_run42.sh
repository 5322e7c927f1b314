timeout 1500 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "half_band or c4 or c5 or fichera" 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -5
for cfg in c4 c2; do
timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg', round(d['ms_per_step'],2), round(r['avg_ms']*1000,1), round(r['achieved']))"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmv_tma_half -c 1 python scripts/precond_once.py c4 2>&1 | grep -E "duration|dram__bytes|hit_rate" | head -5

# line-sweep SpMV: parity, bench on/off, warm launch list
timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "line_sweep or half_band" 2>&1 | grep -E "^E  |^FAILED|passed|failed|Error" | head -20
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_sweep.json 2> gpurun_out/bench_c2_sweep.err; tail -c 1500 gpurun_out/bench_c2_sweep.json | head -c 1400; echo
PMG_SWEEP=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_nosweep.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c2_nosweep.json'));print('nosweep ms',d['ms_per_step'])"
python scripts/solve_once.py c2 2 > gpurun_out/solve_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c2_warm.csv python scripts/solve_once.py c2 2 > gpurun_out/ncu_c2.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/launches_c2_warm.csv | head -24

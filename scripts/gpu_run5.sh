python -m pytest tests/test_gpu_parity.py -q -x --tb=short 2>&1 | tail -4 > gpurun_out/pytest.log; cat gpurun_out/pytest.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_c2.err
python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/solve_once.py c2 1 > gpurun_out/ncu_c2.log 2>&1
echo "ncu rc=$?"

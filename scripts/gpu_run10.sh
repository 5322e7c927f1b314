python scripts/solve_once.py c2 1 > gpurun_out/solve_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/solve_once.py c2 1 > gpurun_out/ncu_c2.log 2>&1
echo "ncu rc=$?"
( time python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err ) 2>&1 | tail -3; echo "c4 rc=$?"; tail -2 gpurun_out/bench_c4.err

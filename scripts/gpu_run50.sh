# round-end measurement pass: GPU suite, smoke, c2 bench (+ reference arm), c4, c5, c2 launch list, sweep capture
timeout 1800 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 700 gpurun_out/bench_c2.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; tail -c 300 gpurun_out/bench_ref_c2.json; echo
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --assembly device > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4', d['ms_per_step'], d['value'], d['roofline']['frac'])"
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --assembly device > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print('c5', d['ms_per_step'], d['value'], d['roofline']['frac'])"
python scripts/solve_once.py c2 2 > gpurun_out/solve_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c2_warm.csv python scripts/solve_once.py c2 2 > gpurun_out/ncu_c2.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_c2_warm.csv > gpurun_out/launches_c2_warm.txt; head -8 gpurun_out/launches_c2_warm.txt
ncu --set full --clock-control none --import-source on -k regex:sweep2d -c 1 -o gpurun_out/prof_sweep_c2 python scripts/solve_once.py c2 1 > gpurun_out/ncu_sweep.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/prof_sweep_c2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum 2>&1 | tail -1

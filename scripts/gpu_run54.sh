# final check on the round's last source: full GPU suite, smoke, c2 bench
timeout 1800 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E  |^FAILED|passed|failed" | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print('c2', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])" || tail -3 gpurun_out/bench_c2.err

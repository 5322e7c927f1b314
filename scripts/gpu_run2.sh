python __graft_entry__.py 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py -q --tb=line 2>&1 | tail -8
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json

python -c "from paper_1804_02539_b200 import build; build.build_all()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=short -x -k "half_band or L5 or L3" 2>&1 | tail -5
python scripts/breakdown.py c2 3 2>&1 | head -24
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"; cat gpurun_out/bench_c2.json
PMG_FULL_BAND=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_full.json 2>&1; echo "c2full rc=$?"
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; cat gpurun_out/bench_c4.json

#!/bin/bash
set -u
mkdir -p gpurun_out
python -m pytest -m gpu -q -p no:cacheprovider -x "tests/test_gpu_assembly.py" "tests/test_gpu_kron.py" > gpurun_out/tests_r02f.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/tests_r02f.log
python bench.py --config c5 --steps 3 > gpurun_out/bench_c5_f.json 2> gpurun_out/bench_c5_f.err; echo "c5 rc=$?"; cut -c1-900 gpurun_out/bench_c5_f.json; tail -3 gpurun_out/bench_c5_f.err
ncu --set full --clock-control none --import-source on -k regex:fd_pass_resident -c 6 -o gpurun_out/prof_fdres6_c5_r02f python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fdres6.log 2>&1; echo "ncu fdres rc=$?"

# FD pass occupancy variants (PMG_FD_STAGES=2 with PMG_FD_MINB=5/6): c2 FD parity subset + c2 bench
L=paper_1804_02539_b200/lib
cp $L/libpmg_cuda.so /tmp/base.so
for v in s2_b5 s2_b6; do
  cp $L/$v/libpmg_cuda.so $L/libpmg_cuda.so
  echo "== $v"
  timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=line -k "c2 and (smooth or pcg)" -x 2>&1 | grep -E "FAILED|passed|failed" | head -3
  timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$v.json 2> gpurun_out/bench_c2_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_c2_$v.json'));r=d['roofline'];print('c2 $v', round(d['ms_per_step'],2), r['fd_finest']['achieved_tflops'])" || tail -3 gpurun_out/bench_c2_$v.err
done
cp /tmp/base.so $L/libpmg_cuda.so

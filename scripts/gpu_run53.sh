# FD pass k-tile/stage variants (PMG_FD_BK, PMG_FD_STAGES): FD parity subset + c2/c4 bench each
L=paper_1804_02539_b200/lib
cp $L/libpmg_cuda.so /tmp/base.so
for v in base v32_2 v32_3; do
  if [ $v = base ]; then cp /tmp/base.so $L/libpmg_cuda.so; else cp $L/$v/libpmg_cuda.so $L/libpmg_cuda.so; fi
  echo "== $v"
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=line -k "smooth or cycle or pcg" -x 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -4
  for cfg in c2 c4; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}_$v.json 2> gpurun_out/bench_${cfg}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/bench_${cfg}_$v.json'));r=d['roofline'];print('$cfg $v', round(d['ms_per_step'],2), r['fd_finest']['achieved_tflops'], r['fd_finest']['share_of_step'])" || tail -3 gpurun_out/bench_${cfg}_$v.err
  done
done
cp /tmp/base.so $L/libpmg_cuda.so

for sm in 200000 110000 72000; do
  for cfg in c3p2 c3p4; do
    PMG_SWEEP_SMEM=$sm timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err
    python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$sm $cfg', d['ms_per_step'], round(d['roofline']['frac'],3), round(d['roofline']['avg_ms']*1e3,1))" || tail -3 gpurun_out/b.err
  done
done

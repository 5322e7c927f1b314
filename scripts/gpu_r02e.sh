#!/bin/bash
set -u
mkdir -p gpurun_out
python -m pytest -m gpu -q -p no:cacheprovider -x "tests/test_gpu_parity.py::test_smooth_forced_fd_panels" "tests/test_gpu_parity.py::test_transfers" "tests/test_gpu_fullsize_parity.py" -k "not c3p" > gpurun_out/tests_r02e.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/tests_r02e.log
b() { tag=$1; shift; python bench.py --no-cpu-baseline --steps 3 "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "$tag rc=$?"; python - <<P
import json
try:
    d=json.load(open("gpurun_out/bench_$tag.json")); r=d["roofline"]
    print("  ms/step %.3f its %d spmv %.4f ms frac %.3f fd %.2f TF/s vcycle %.3f" % (d["ms_per_step"], d["config"]["pcg_iterations"], r["avg_ms"], r["frac"], r["fd_finest"]["achieved_tflops"] or 0, d["vcycle"]["ms"]))
    for lv,row in r["per_level"].items():
        print("   L"+lv, {k:(round(v["ms_per_step"],3), round(v.get("hbm_frac",v.get("tflops",0)),3)) for k,v in row.items()})
except Exception as e: print("  fail", e)
P
}
b c5_e --config c5
PMG_FD_RESIDENT=0 b c5_e_nores --config c5
b c4_e --config c4
PMG_FD_CFG=9,0 b c4_e_res --config c4

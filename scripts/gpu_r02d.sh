#!/bin/bash
set -u
mkdir -p gpurun_out
python -m pytest -m gpu -q -p no:cacheprovider -x tests/test_gpu_kron.py "tests/test_gpu_parity.py::test_smooth_forced_fd_panels" "tests/test_gpu_parity.py::test_plane_sweep_matches_tma_half" "tests/test_gpu_parity.py::test_smooth" "tests/test_gpu_parity.py::test_pcg_matches_oracle" "tests/test_gpu_parity.py::test_cycle_parameters_match_oracle" > gpurun_out/tests_r02d.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/tests_r02d.log
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
b c5_d --config c5
PMG_FD_RESIDENT=0 b c5_d_nores --config c5
b c4_d --config c4
PMG_FD_RESIDENT=0 b c4_d_nores --config c4
b c3p8_kron_d --config c3p8 --operator kronecker
b c2_d --config c2
# profiles
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r02d.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c5_r02d.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:spmv_sweep3d -c 1 -o gpurun_out/prof_sweep3d_c5_r02d python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sweep3d.log 2>&1; echo "ncu sweep3d rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fd_pass_resident -c 1 -o gpurun_out/prof_fdres_c5_r02d python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fdres.log 2>&1; echo "ncu fdres rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fd_pass_dmma -c 1 -o gpurun_out/prof_fdwide_c2_r02d python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fdwide.log 2>&1; echo "ncu fdwide rc=$?"

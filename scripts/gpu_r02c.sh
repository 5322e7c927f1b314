#!/bin/bash
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fd_probe scripts/fd_probe.cu && /tmp/fd_probe > gpurun_out/fd_probe_r02.txt 2>&1
cat gpurun_out/fd_probe_r02.txt
python -m pytest -m gpu -q -p no:cacheprovider -x tests/test_gpu_kron.py "tests/test_gpu_parity.py::test_smooth_forced_fd_panels" "tests/test_gpu_parity.py::test_plane_sweep_matches_tma_half" "tests/test_gpu_parity.py::test_smooth" "tests/test_gpu_parity.py::test_pcg_matches_oracle" > gpurun_out/tests_r02c.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tests_r02c.log
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
b c5_res --config c5
PMG_FD_RESIDENT=0 b c5_nores --config c5
PMG_SWEEP3_TILES_C=1 PMG_SWEEP3_ZSEGS_C=4 b c5_c14 --config c5
PMG_SWEEP3_TILES_C=2 PMG_SWEEP3_ZSEGS_C=2 b c5_c22 --config c5
PMG_SWEEP3_TILES_C=4 PMG_SWEEP3_ZSEGS_C=1 b c5_c41 --config c5
PMG_SWEEP3D=48 b c5_nosweepL4 --config c5
b c4_res --config c4
PMG_FD_RESIDENT=0 b c4_nores --config c4
b c3p8_kron --config c3p8 --operator kronecker
b c3p2_kron --config c3p2 --operator kronecker

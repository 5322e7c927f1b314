#!/bin/bash
# r02b: new-kernel parity, then A/B timings
set -u
mkdir -p gpurun_out
python -m pytest -m gpu -q -p no:cacheprovider -x tests/test_gpu_kron.py "tests/test_gpu_parity.py::test_cycle_parameters_match_oracle" "tests/test_gpu_parity.py::test_smooth_forced_fd_panels" "tests/test_gpu_fullsize_parity.py" -k "not c5 and not c4" > gpurun_out/tests_r02b.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/tests_r02b.log
b() { tag=$1; shift; python bench.py --no-cpu-baseline --steps 3 "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "$tag rc=$?"; python - <<P
import json
try:
    d=json.load(open("gpurun_out/bench_$tag.json")); r=d["roofline"]
    print("  ms/step %.3f its %d spmv %.4f ms frac %.3f fd %.2f TF/s vcycle %.3f" % (d["ms_per_step"], d["config"]["pcg_iterations"], r["avg_ms"], r["frac"], r["fd_finest"]["achieved_tflops"] or 0, d["vcycle"]["ms"]))
except Exception as e: print("  fail", e)
P
}
b c2_wide --config c2
PMG_FD_WIDE=0 b c2_nowide --config c2
PMG_FD_CFG=9,11 b c2_9_11 --config c2
PMG_FD_CFG=11,8 b c2_11_8 --config c2
b c3p8_band --config c3p8
b c3p8_kron --config c3p8 --operator kronecker
b c3p2_band --config c3p2
b c3p2_kron --config c3p2 --operator kronecker
b c1_kron --config c1 --operator kronecker
b c4_default --config c4
PMG_SWEEP3_TILES=4 PMG_SWEEP3_ZSEGS=4 b c4_t4z4 --config c4
PMG_SWEEP3_TILES=3 PMG_SWEEP3_ZSEGS=6 b c4_t3z6 --config c4
PMG_SWEEP3_TILES=4 PMG_SWEEP3_ZSEGS=3 b c4_t4z3 --config c4
PMG_SWEEP3_TILES=12 PMG_SWEEP3_ZSEGS=1 b c4_t12z1 --config c4
PMG_SWEEP3_TILES=9 PMG_SWEEP3_ZSEGS=2 b c4_t9z2 --config c4
PMG_FD_CFG=9,8 b c4_fd98 --config c4
PMG_FD_CFG=9,11 b c4_fd911 --config c4

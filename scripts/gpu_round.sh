#!/bin/bash
# Round-end GPU pass (run under gpurun from the repo root): the full -m gpu
# suite, one bench line per BASELINE config (+ the reference arm and the
# matrix-free variants), the ncu launch list of the headline command and one
# ncu --set full capture per hot kernel.  TAG names the outputs.
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'TAG=r02 bash scripts/gpu_round.sh'
set -u
mkdir -p gpurun_out
TAG=${TAG:-round}
nvidia-smi -L; nproc
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  PMG_TEST_FULL=${PMG_TEST_FULL:-1} python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/tests_$TAG.log 2>&1
  echo "tests rc=$?"; tail -3 gpurun_out/tests_$TAG.log
fi
python bench.py > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err; echo "c5 rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c5_$TAG.json 2> gpurun_out/bench_ref_c5_$TAG.err; echo "ref rc=$?"
for c in c4 c2 c1 c3p2 c3p3 c3p4 c3p6 c3p8; do
  python bench.py --config $c > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?"
done
for c in c1 c3p2 c3p4 c3p8; do
  python bench.py --config $c --operator kronecker --no-cpu-baseline > gpurun_out/bench_${c}_kron_$TAG.json 2> gpurun_out/bench_${c}_kron_$TAG.err; echo "$c kron rc=$?"
done
python - <<P
import glob, json
for f in sorted(glob.glob("gpurun_out/bench_*_$TAG.json")):
    try:
        d = json.load(open(f)); r = d.get("roofline") or {}
        print(f.split("/")[-1], "%.3f ms" % d["ms_per_step"], "%.4g %s" % (d["value"], d["unit"]),
              "e2e %.4g" % d["e2e"]["value"], "spmv frac", r.get("frac"), "fd", (r.get("fd_finest") or {}).get("achieved_tflops"),
              "vcycle", (d.get("vcycle") or {}).get("frac"), "clocks", d.get("clocks"))
    except Exception as e:
        print(f, "unreadable:", e)
P
# profiles: each capture only after the plain command above exited 0
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$TAG.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c5_$TAG.log 2>&1; echo "launch list rc=$?"
cap() { # name, kernel regex, count, bench args.  gpurun brings back <= 64 MiB: keep the raw metric page, not the report
  ncu --set full --clock-control none --import-source on -k "regex:$2" -c $3 -o /tmp/prof_$1_$TAG -f \
    python bench.py $4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$1_$TAG.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i /tmp/prof_$1_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$1_$TAG.csv 2>/dev/null
}
cap sweep3d_c5 spmv_sweep3d 1 "--config c5"
cap fdres_c5 fd_pass_resident 6 "--config c5"
cap sweep3d_c4 spmv_sweep3d 1 "--config c4"
cap sweep2d_c2 spmv_sweep2d 1 "--config c2"
cap fdwide_c2 fd_pass_dmma 4 "--config c2"
cap kron_c3p8 kron2d 1 "--config c3p8 --operator kronecker"

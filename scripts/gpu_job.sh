#!/bin/bash
# One parametrized GPU job (run under gpurun from the repo root):
#   bash scripts/gpu_job.sh tests  <pytest args...>     pytest -m gpu subset -> gpurun_out/tests_<tag>.log
#   bash scripts/gpu_job.sh bench  "<bench args>"       bench.py line        -> gpurun_out/bench_<tag>.json
#   bash scripts/gpu_job.sh launches "<bench args>"     ncu launch list      -> gpurun_out/launches_<tag>.csv
#   bash scripts/gpu_job.sh ncu "<kernel regex>" "<bench args>"  ncu --set full of one launch -> gpurun_out/prof_<tag>.ncu-rep
# TAG (env) names the outputs.
set -u
mkdir -p gpurun_out
TAG=${TAG:-run}
job=$1; shift
case "$job" in
  tests)
    python -m pytest -m gpu -q -p no:cacheprovider "$@" > gpurun_out/tests_$TAG.log 2>&1
    echo "tests rc=$?"; tail -5 gpurun_out/tests_$TAG.log ;;
  bench)
    python bench.py $1 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
    echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err ;;
  launches)
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
      python bench.py $1 --no-cpu-baseline > gpurun_out/launches_$TAG.log 2>&1
    echo "launches rc=$?" ;;
  ncu)
    ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${SKIP:-0} -c 1 -o gpurun_out/prof_$TAG \
      python bench.py $2 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
    echo "ncu rc=$?" ;;
  *) echo "unknown job $job"; exit 2 ;;
esac

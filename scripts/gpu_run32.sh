timeout 900 ncu --set full --import-source on --clock-control none -k regex:smooth_small -s 0 -c 1 -o gpurun_out/prof_smooth_small python scripts/solve_once.py c2 1 > gpurun_out/ncu_ss.log 2>&1
echo "ncu rc=$?"

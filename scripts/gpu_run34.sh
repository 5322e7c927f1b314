PMG_DEBUG_SMOOTH=1 timeout 900 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:smooth_small -s 0 -c 1 -o gpurun_out/prof_ss_fd python scripts/precond_once.py c2 > gpurun_out/ncu_ss.log 2>&1
echo "ncu rc=$?"

PMG_COARSE_TRACE=1 timeout 300 python scripts/solve_once.py c2 2 2>&1 | tail -3
PMG_COARSE_TRACE=1 timeout 300 python scripts/solve_once.py c4 1 2>&1 | tail -2

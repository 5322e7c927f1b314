for me in 128 60 30; do echo "== min_ext $me"; PMG_SWEEP_MIN_EXT=$me timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv L[3-7]|wall"; done

for sm in 0 225000; do echo "== smem $sm"; PMG_SWEEP_SMEM=$sm timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv L[67]|wall"; done

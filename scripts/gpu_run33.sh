for sm in 200000 110000 96000; do
echo "== smem $sm"; PMG_SWEEP_SMEM=$sm timeout 600 python scripts/breakdown.py c2 3 2>&1 | grep -E "spmv L[67]|wall"
done

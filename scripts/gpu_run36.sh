for i in 1 2 3 4 5 6; do timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no -x -k "c2-p4-L5 and (cycle or transfers)" 2>&1 | grep -E "passed|failed" | head -1; done
echo "== old"
cp paper_1804_02539_b200/lib/libpmg_cuda_old.so paper_1804_02539_b200/lib/libpmg_cuda.so
for i in 1 2 3 4 5 6; do timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no -x -k "c2-p4-L5 and (cycle or transfers)" 2>&1 | grep -E "passed|failed" | head -1; done

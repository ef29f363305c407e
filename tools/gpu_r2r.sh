#!/bin/bash
# row passes with their twiddle rows staged in shared memory (product) vs from global (rowtws0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2r
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
HKS_LIB_PATH=tools/exp/rowtws0/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_rowtws0.json 2>/dev/null
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > ${O}_batched.json 2>/dev/null

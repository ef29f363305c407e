#!/bin/bash
# tensor-core base conversion: contiguous target runs per epilogue warp (two 32-column TMEM loads per tile)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
HKS_LIB_PATH=tools/exp/bctrace/libhks.so timeout 200 python tools/bc_trace.py > ${O}_bctrace.txt 2>&1

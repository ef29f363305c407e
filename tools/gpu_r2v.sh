#!/bin/bash
# fused row pass + key product: input rows staged by cp.async with the twiddles (product) vs loaded in round 0
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2v
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "keyswitch or hmult or rotate or kip or linear or moddown" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
HKS_LIB_PATH=tools/exp/exts0/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_exts0.json 2>/dev/null
HKS_LIB_PATH=tools/exp/kiptrace/libhks.so timeout 200 python tools/kip_trace.py > ${O}_kiptrace.txt 2>&1

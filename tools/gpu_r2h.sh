#!/bin/bash
# Round-2 session-2 baseline: GPU tests at HEAD, C2 bench (batched and one at a time), TC column-pass variant A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > ${O}_c2.json 2> ${O}_c2.err
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_c2s1.json 2> ${O}_c2s1.err
HKS_LIB_PATH=tools/exp/tc1/libhks.so timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_c2s1_tc1.json 2> ${O}_c2s1_tc1.err

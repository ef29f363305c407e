#!/bin/bash
# fused key product with a fourth warp (xwarp) vs product; HEAD launch list of the default bench step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r3e
HKS_LIB_PATH=tools/exp/xwarp/libhks.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "keyswitch or hmult or rotate or kip or linear" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
HKS_LIB_PATH=tools/exp/xwarp/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_xwarp.json 2>/dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 600 --csv --log-file ${O}_launches.csv \
  python bench.py --steps 5 --warmup 3 --quick > ${O}_launches.log 2>&1

#!/bin/bash
# cluster INTT with L2-prefetched row twiddles and explicit DSMEM loads vs two-pass (nocl); ncu of the cluster kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ntt or keyswitch or moddown or modup" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base1.json 2>/dev/null
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_base1.json 2>/dev/null
HKS_LIB_PATH=tools/exp/nocl/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_nocl1.json 2>/dev/null
HKS_LIB_PATH=tools/exp/nocl/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_nocl1.json 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_intt_cl" --launch-skip 3 --launch-count 1 \
  -o ${O}_prof -f python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_ncu.log 2>&1
echo "ncu rc=$?" >> ${O}_ncu.log

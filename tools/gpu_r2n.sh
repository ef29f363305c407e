#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2n
HKS_LIB_PATH=tools/exp/tctrace/libhks.so timeout 120 python tools/nc_trace.py 90 > ${O}_trace_fwd90.txt 2>&1
export HKS_LIB_PATH=tools/exp/tc3/libhks.so
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ntt_parity or keyswitch_parity_c2" > ${O}_ntt.txt 2>&1
echo "pytest rc=$?" >> ${O}_ntt.txt
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --streams 1 --quick > ${O}_c2s1.json 2> ${O}_c2s1.err

#!/bin/bash
# launch list of the default bench command (libhks kernels only) + detailed KIP phase trace
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r3c
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 600 --csv --log-file ${O}_launches.csv \
  python bench.py --steps 5 --warmup 3 --quick > ${O}_launches.log 2>&1
echo "ncu rc=$?" >> ${O}_launches.log
HKS_LIB_PATH=tools/exp/kiptrace/libhks.so timeout 200 python tools/kip_trace.py > ${O}_kiptrace.txt 2>&1

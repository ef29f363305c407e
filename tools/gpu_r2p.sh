#!/bin/bash
# ncu --set full (with source) of one C2 KeySwitch (9 kernels) at HEAD
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2p
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"^k_" --launch-skip 27 --launch-count 9 \
  -o ${O}_prof -f python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_ncu.log 2>&1
echo "ncu rc=$?" >> ${O}_ncu.log

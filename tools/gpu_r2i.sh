#!/bin/bash
# ncu --set full of the tensor-core column pass v2 (tools/exp/tc1) inside a C2 KeySwitch
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2i
HKS_LIB_PATH=tools/exp/tc1/libhks.so timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"k_ntt_cols_tc" --launch-skip 6 --launch-count 2 -o ${O}_tc -f \
  python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_tc.log 2>&1
echo "ncu rc=$?" >> ${O}_tc.log

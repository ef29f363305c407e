#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
HKS_LIB_PATH=tools/exp/bctrace/libhks.so timeout 200 python tools/bc_trace.py > gpurun_out/r2w_bctrace.txt 2>&1

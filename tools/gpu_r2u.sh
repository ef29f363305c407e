#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
HKS_LIB_PATH=tools/exp/kiptrace/libhks.so timeout 200 python tools/kip_trace.py > gpurun_out/r2u_kiptrace.txt 2>&1

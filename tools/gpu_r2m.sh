#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
HKS_LIB_PATH=tools/exp/tctrace/libhks.so timeout 120 python tools/nc_trace.py 90 > gpurun_out/r2m_trace_fwd90.txt 2>&1
HKS_LIB_PATH=tools/exp/tctrace/libhks.so timeout 120 python tools/nc_trace.py 30 inv > gpurun_out/r2m_trace_inv30.txt 2>&1

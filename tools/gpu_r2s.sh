#!/bin/bash
# register budget of the 128-thread (column) passes: 4 (product) vs 5 / 6 / 8 resident CTAs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2s
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
for v in mb5 mb6 mb8; do
  HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_$v.json 2>/dev/null
done

#!/bin/bash
# A/B of tensor-core column-pass variants (stage width) against the butterfly product build, one KeySwitch per step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2o
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
for v in tc3a tc3b tc3c; do
  HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_$v.json 2>/dev/null
done

#!/bin/bash
# concurrent KeySwitches per step (2 / 3 / 4) with the 4-row fused kernel: three interleaved repeats
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r5c
for rep in 1 2 3; do
  for k in 2 3 4; do
    timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline --streams $k > ${O}_s${k}_r$rep.json 2>/dev/null
  done
done

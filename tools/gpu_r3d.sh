#!/bin/bash
# concurrent KeySwitches per step at HEAD: 2 / 3 / 4 / 5 streams
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r3d
for n in 3 2 4 5 3; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --quick --streams $n > ${O}_s$n.json 2>/dev/null
done

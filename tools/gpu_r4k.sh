#!/bin/bash
# level and NTT limb-batch sweeps at HEAD (NEXT-4 evidence)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --out gpurun_out/sweep_r4.json > gpurun_out/sweep_r4.log 2>&1
echo "rc=$?" >> gpurun_out/sweep_r4.log

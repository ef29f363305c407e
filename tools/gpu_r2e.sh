#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 bash tools/ab.sh r2e tw ks twks ic6
timeout 600 bash tools/ab.sh r2e2 twks

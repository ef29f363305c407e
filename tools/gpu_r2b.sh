#!/bin/bash
# GPU tests + one ncu --set full capture of a C2 KeySwitch (the 4th KeySwitch of the run, 9 kernels).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2b
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"^k_" --launch-skip 27 --launch-count 9 \
  -o ${O}_prof -f python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_ncu.log 2>&1
echo "ncu rc=$?" >> ${O}_ncu.log

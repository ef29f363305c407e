#!/bin/bash
# HEAD evidence: ncu --set full of one C2 KeySwitch (9 kernels) + the launch list of the default bench command
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r3b
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"^k_" --launch-skip 27 --launch-count 9 \
  -o ${O}_prof -f python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_ncu.log 2>&1
echo "ncu rc=$?" >> ${O}_ncu.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file ${O}_launches.csv \
  python bench.py --steps 2 --warmup 1 > ${O}_launches.log 2>&1
echo "ncu rc=$?" >> ${O}_launches.log

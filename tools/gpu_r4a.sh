#!/bin/bash
# warp-synchronised row passes (product) vs CTA barriers (nows); inverse-table L2 persistence (pinv, pinvks);
# ncu --set full with source of one C2 KeySwitch at the product build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4a
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in nows pinv pinvks; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_$v$rep.json 2>/dev/null
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_" --launch-skip 27 --launch-count 9 \
  -o ${O}_prof -f python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_ncu.log 2>&1
echo "ncu rc=$?" >> ${O}_ncu.log

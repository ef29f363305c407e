#!/bin/bash
# fused kernel (4 rows per CTA) at a 64-register budget: 5 resident CTAs per SM instead of 4 (r64)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r5b
HKS_LIB_PATH=tools/exp/r64/libhks.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "keyswitch_parity_c2 or hmult_parity_c2 or kip" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in r64; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  HKS_LIB_PATH=tools/exp/r64/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_r64$rep.json 2>/dev/null
done
done
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  HKS_LIB_PATH=tools/exp/r64/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_r64$rep.json 2>/dev/null
done

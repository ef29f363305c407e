#!/bin/bash
# fused row pass + key product with 4 rows per CTA (nb2) after the per-warp barriers
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4x
HKS_LIB_PATH=tools/exp/nb2/libhks.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ntt or keyswitch or hmult or rotate or rescale or bconv or modup or moddown" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in nb2; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_$v$rep.json 2>/dev/null
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
done

#!/bin/bash
# tensor-core base conversion with 12 / 8 epilogue warps (fewer registers per SM: room for other streams' CTAs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4u
HKS_LIB_PATH=tools/exp/epw8/libhks.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ntt or keyswitch or hmult or rotate or rescale" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in epw12 epw8; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_$v$rep.json 2>/dev/null
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
done

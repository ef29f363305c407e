#!/bin/bash
# tensor-core base conversion with 8 / 12 epilogue warps (runs reduced in 8-target chunks), at a 96-register cap (room for other CTAs) or uncapped
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4v
HKS_LIB_PATH=tools/exp/epw8r96/libhks.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ntt or keyswitch or hmult or rotate or rescale or bconv or modup or moddown" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
HKS_LIB_PATH=tools/exp/epw12r96/libhks.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "keyswitch_parity or bconv or moddown or hmult_parity_c2" > ${O}_pytest12.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest12.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in epw8r96 epw12r96 epw8; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_$v$rep.json 2>/dev/null
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
done

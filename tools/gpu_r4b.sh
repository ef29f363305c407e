#!/bin/bash
# butterfly carry-adds on the ALU pipe (opaque zero, product) vs plain adds (noopq) vs predicated low word (opq2)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4b
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in noopq opq2; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_$v$rep.json 2>/dev/null
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
done

#!/bin/bash
# fused row pass + key product with 4 rows per CTA (nb2) vs 2 (product): three interleaved repeats, C2 and C4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4y
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  HKS_LIB_PATH=tools/exp/nb2/libhks.so timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline > ${O}_s3_nb2$rep.json 2>/dev/null
done
for rep in 1 2; do
  timeout 300 python bench.py --config C4 --steps 60 --warmup 5 --no-cpu-baseline > ${O}_c4_base$rep.json 2>/dev/null
  HKS_LIB_PATH=tools/exp/nb2/libhks.so timeout 300 python bench.py --config C4 --steps 60 --warmup 5 --no-cpu-baseline > ${O}_c4_nb2$rep.json 2>/dev/null
done
HKS_LIB_PATH=tools/exp/nb2/libhks.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c4 or kip or linear or rotate" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt

#!/bin/bash
# batched-step shapes: fused kernel with 8 rows per CTA (nb3); small-batch passes with 16 sub-transforms per CTA (sel6)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r5a
HKS_LIB_PATH=tools/exp/nb3/libhks.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "keyswitch_parity_c2 or hmult_parity_c2 or kip" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in nb3 sel6; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
done

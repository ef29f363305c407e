#!/bin/bash
# fused row pass + key product: twiddles staged in shared memory (product build) / key L2 prefetch variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2q
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "keyswitch or hmult or rotate or kip or moddown or linear" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
for v in kipa kipb kipc; do
  HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_$v.json 2>/dev/null
done

#!/bin/bash
# key-load pipelining in the fused row pass + key product
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2t
HKS_LIB_PATH=tools/exp/pipe2/libhks.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "keyswitch or hmult or rotate or kip or linear" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_base.json 2>/dev/null
for v in pipe1 pipe2 pipe2r96; do
  HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_$v.json 2>/dev/null
done

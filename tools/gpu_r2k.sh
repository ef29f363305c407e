#!/bin/bash
# tensor-core column pass v3 (tools/exp/tc3): NTT parity first (short timeout: a protocol bug hangs), then KeySwitch parity and timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2k
export HKS_LIB_PATH=tools/exp/tc3/libhks.so
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ntt_parity" > ${O}_ntt.txt 2>&1
rc=$?
echo "pytest rc=$rc" >> ${O}_ntt.txt
if [ $rc -ne 0 ]; then exit 0; fi
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ntt or keyswitch or hmult or rescale or moddown or rotate or linear" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_c2s1.json 2> ${O}_c2s1.err
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > ${O}_c2.json 2> ${O}_c2.err

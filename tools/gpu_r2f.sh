#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2f
timeout 1500 python -m pytest tests/test_shard.py tests/test_multirank.py -q -p no:cacheprovider -m gpu > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 1500 bash tools/ab.sh r2f tc1 tc90 tc90s tcf

#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2g
timeout 1500 python -m pytest tests/test_shard.py tests/test_multirank.py -q -p no:cacheprovider -m gpu -x > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for m in nccl pipe a2a; do
  timeout 300 python bench.py --config C4 --shard $m --steps 50 --warmup 5 --quick > ${O}_c4_$m.json 2> ${O}_c4_$m.err
done

#!/bin/bash
# byte-sum reduction on the ALU pipe: base-conversion parity + C2 bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2j
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bconv or modup or keyswitch_parity_c2 or hmult" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_c2s1.json 2> ${O}_c2s1.err
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > ${O}_c2.json 2> ${O}_c2.err

#!/bin/bash
# prepared keys (hks_evk_prepare): parity tests, bench with prepared (default) vs plain keys
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4l
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "prepared or keyswitch or hmult or rotate or error or evk" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2; do
  for k in prepared plain; do
    timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 --key $k > ${O}_s1_$k$rep.json 2>/dev/null
    timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --key $k > ${O}_s3_$k$rep.json 2>/dev/null
  done
done
timeout 300 python bench.py --config C1 --steps 2000 --warmup 10 --no-cpu-baseline --key prepared > ${O}_c1_prepared.json 2>/dev/null
timeout 300 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu-baseline --key prepared > ${O}_c4_prepared.json 2>/dev/null
timeout 300 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu-baseline --key plain > ${O}_c4_plain.json 2>/dev/null

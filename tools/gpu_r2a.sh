#!/bin/bash
# Round-2 evidence run: GPU tests, smoke, C2 bench, compute-sanitizer on the small configs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > ${O}_smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.txt 2>&1
timeout 900 python bench.py > ${O}_bench_c2.json 2> ${O}_bench_c2.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py C1 T16s > ${O}_san_${tool}.txt 2>&1
  echo "rc=$?" >> ${O}_san_${tool}.txt
done

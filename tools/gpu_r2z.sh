#!/bin/bash
# Evidence at HEAD: full GPU test suite, smoke, compute-sanitizer (C1, T16s), C1-C5 bench lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2z
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${O}_smoke.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py C1 T16s > ${O}_san_${tool}.txt 2>&1
  echo "rc=$?" >> ${O}_san_${tool}.txt
done
for c in C2 C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c > ${O}_bench_$(echo $c | tr A-Z a-z).json 2> ${O}_bench_$(echo $c | tr A-Z a-z).err
done

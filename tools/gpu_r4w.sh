#!/bin/bash
# final check at HEAD: GPU test suite, smoke, default bench line (C2) and C1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4w
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${O}_smoke.txt 2>&1
timeout 900 python bench.py > ${O}_bench_c2.json 2> ${O}_bench_c2.err
timeout 900 python bench.py --config C1 > ${O}_bench_c1.json 2> ${O}_bench_c1.err

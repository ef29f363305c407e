#!/bin/bash
# final evidence at HEAD (fused kernel with 4 rows per CTA at N = 2^16): GPU test suite, smoke, C1-C5 bench lines,
# ncu launch list and ncu --set full of one C2 KeySwitch
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4z
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${O}_smoke.txt 2>&1
timeout 900 python bench.py > ${O}_bench_c2.json 2> ${O}_bench_c2.err
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c > ${O}_bench_$(echo $c | tr A-Z a-z).json 2> ${O}_bench_$(echo $c | tr A-Z a-z).err
done
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_c2_streams1.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 600 --csv --log-file ${O}_launches.csv \
  python bench.py --steps 5 --warmup 3 --quick > ${O}_launches.log 2>&1
echo "ncu rc=$?" >> ${O}_launches.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"^k_" --launch-skip 28 --launch-count 9 \
  -o ${O}_prof -f python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_ncu.log 2>&1
echo "ncu rc=$?" >> ${O}_ncu.log

#!/bin/bash
# single-pass cluster INTT (product) vs two-pass INTT (nocl); racecheck / memcheck of T16s; ncu of the cluster kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r4d
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_base$rep.json 2>/dev/null
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_base$rep.json 2>/dev/null
  for v in nocl; do
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --streams 1 > ${O}_s1_$v$rep.json 2>/dev/null
    HKS_LIB_PATH=tools/exp/$v/libhks.so timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > ${O}_s3_$v$rep.json 2>/dev/null
  done
done
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py T16s > ${O}_racecheck.txt 2>&1; echo "rc=$?" >> ${O}_racecheck.txt
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py T16s > ${O}_memcheck.txt 2>&1; echo "rc=$?" >> ${O}_memcheck.txt
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_run.py T16s > ${O}_synccheck.txt 2>&1; echo "rc=$?" >> ${O}_synccheck.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_intt_cl" --launch-skip 3 --launch-count 1 \
  -o ${O}_prof -f python bench.py --steps 1 --warmup 3 --quick --no-graph --streams 1 --sets 1 > ${O}_ncu.log 2>&1
echo "ncu rc=$?" >> ${O}_ncu.log

#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root): bench lines for every config,
# the ncu launch list and one `ncu --set full` capture of a C2 KeySwitch.   tools/full_run.sh TAG
tag=${1:-r1}
out=gpurun_out
python bench.py > $out/bench_${tag}_c2.json 2> $out/bench_${tag}_c2.err
for c in C1 C3 C4 C5; do
  python bench.py --config $c --steps $([ $c = C1 ] && echo 2000 || echo 30) --warmup 5 --no-cpu-baseline \
    > $out/bench_${tag}_$(echo $c | tr A-Z a-z).json 2>> $out/bench_${tag}_c2.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file $out/launches_${tag}.csv \
  python bench.py --quick --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_" --launch-skip 90 --launch-count 9 \
  -o $out/prof_${tag} -f python bench.py --quick --streams 1 --steps 12 --warmup 3 --sets 2 --no-cpu-baseline > /dev/null 2>&1
ls -la $out | grep $tag

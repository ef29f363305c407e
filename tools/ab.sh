#!/bin/bash
# A/B timing of experimental libhks variants (tools/exp/<name>/libhks.so) against the product build.
# Usage (on the GPU box): tools/ab.sh OUTPREFIX name1 name2 ...   -> gpurun_out/OUTPREFIX_<name>.json
pre=$1; shift
python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/${pre}_base.json 2>/dev/null
for v in "$@"; do
  HKS_LIB_PATH=tools/exp/$v/libhks.so python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/${pre}_$v.json 2>/dev/null
done

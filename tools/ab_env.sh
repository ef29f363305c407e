#!/bin/bash
# A/B timing of experimental libhks variants with extra environment (e.g. HKS_NTT_TC=1):
#   tools/ab_env.sh OUTPREFIX "ENV=..." name1 name2 ...   -> gpurun_out/OUTPREFIX_<name>.json
pre=$1; shift
envs=$1; shift
env $envs python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/${pre}_base.json 2>/dev/null
python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/${pre}_default.json 2>/dev/null
for v in "$@"; do
  env $envs HKS_LIB_PATH=tools/exp/$v/libhks.so python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/${pre}_$v.json 2>/dev/null
done

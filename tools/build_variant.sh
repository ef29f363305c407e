#!/bin/bash
# Build an experimental libhks variant with extra nvcc flags into tools/exp/<name>/libhks.so
# (A/B timing via HKS_LIB_PATH; never the product library).  Usage: tools/build_variant.sh NAME FLAGS...
set -e
name=$1; shift
out=/root/repo/tools/exp/$name
mkdir -p $out
cd /root/repo/paper_2507_04775_b200/csrc
for f in ctx ntt ntt_tc kernels capi prof shard; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c $f.cu -o $out/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/libhks.so $out/*.o
rm -f $out/*.o
echo $out/libhks.so

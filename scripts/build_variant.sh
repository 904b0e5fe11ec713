#!/bin/bash
# Builds the engine with extra nvcc defines into paper_0912_2555_b200/_lib/variants/<name>.so
#   scripts/build_variant.sh t1024 -DCYC_RL_THREADS=1024
set -e
cd "$(dirname "$0")/../paper_0912_2555_b200/csrc"
name=$1; shift
out=../_lib/variants/$name; mkdir -p $out
for f in $(sed -n "s/^SRCS := //p" Makefile | sed "s/\.cu//g"); do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr "$@" -c $f.cu -o $out/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o ../_lib/variants/$name.so $out/*.o
rm -rf $out
echo built ../_lib/variants/$name.so

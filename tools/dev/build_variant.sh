#!/bin/bash
# Variant build of liblc for compile-time A/B: tools/dev/build_variant.sh NAME [nvcc flags...] -> build_var/NAME/liblc.so
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
mkdir -p build_var/$name
objs=()
for f in paper_2001_01158_b200/csrc/*.cu; do
  o=build_var/$name/$(basename $f).o
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -fmad=false "$@" -gencode arch=compute_100a,code=sm_100a \
    -Xcompiler -fPIC -Iinclude -Xptxas -v -c $f -o $o 2> build_var/$name/$(basename $f).ptxas &
  objs+=($o)
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build_var/$name/liblc.so "${objs[@]}"
echo built build_var/$name/liblc.so

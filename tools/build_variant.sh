#!/bin/bash
# Build liblc with extra nvcc defines for an A/B (not the product build): tools/build_variant.sh NAME -DX=Y ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_var/$name
objs=()
for f in paper_2001_01158_b200/csrc/*.cu; do
  o=build_var/$name/$(basename $f).o
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -fmad=false "$@" -gencode arch=compute_100a,code=sm_100a \
    -Xcompiler -fPIC -Iinclude -c $f -o $o &
  objs+=($o)
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build_var/$name/liblc.so "${objs[@]}"

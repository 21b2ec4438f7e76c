#!/bin/bash
# A/B build that recompiles ONE source with extra defines and links it with the product build's other objects
# (python -m paper_2001_01158_b200.build first): tools/dev/build_one_variant.sh NAME FILE.cu -DX=Y ...
set -e
cd "$(dirname "$0")/../.."
name=$1; src=$2; shift 2
mkdir -p build_var/$name
o=build_var/$name/$(basename $src).o
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -fmad=false "$@" -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC -Iinclude -c paper_2001_01158_b200/csrc/$src -o $o
objs=($o)
for f in build/*.cu.o; do [ "$(basename $f)" = "$src.o" ] || objs+=($f); done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build_var/$name/liblc.so "${objs[@]}"

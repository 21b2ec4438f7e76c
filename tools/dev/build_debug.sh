#!/bin/bash
# Debug build of liblc with the device timelines (-DLC_DEBUG_TIMELINE): build_dbg/liblc_dbg.so
set -e
cd "$(dirname "$0")/../.."
mkdir -p build_dbg
objs=()
for f in paper_2001_01158_b200/csrc/*.cu; do
  o=build_dbg/$(basename $f).o
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -fmad=false -DLC_DEBUG_TIMELINE -gencode arch=compute_100a,code=sm_100a \
    -Xcompiler -fPIC -Iinclude -c $f -o $o &
  objs+=($o)
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build_dbg/liblc_dbg.so "${objs[@]}"

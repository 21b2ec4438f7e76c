#!/bin/bash
O=gpurun_out/r4n; mkdir -p $O
for v in main d_r2 d_r1 d_r8 main; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 3 >> $O/ab.txt 2>&1
done

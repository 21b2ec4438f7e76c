#!/bin/bash
O=gpurun_out/r4b; mkdir -p $O
for v in g_base g_none g_sp g_red g_coal g_sp_red2 g_base g_sp; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 4 >> $O/ab.txt 2>&1
done

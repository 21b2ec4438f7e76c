#!/bin/bash
O=gpurun_out/r4d; mkdir -p $O
for v in g_base g_v0 g_v1 g_v1h1 g_v1h2 g_v0h1 g_v1; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 4 >> $O/ab.txt 2>&1
done

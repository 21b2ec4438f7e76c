#!/bin/bash
O=gpurun_out/r4c; mkdir -p $O
for v in g_base g_sp_red2 g_pf0 g_pf1 g_pf2 g_pf4 g_pf6 g_pf7 g_pf6c1 g_pf6c3 g_base; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 4 >> $O/ab.txt 2>&1
done

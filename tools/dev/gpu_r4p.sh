#!/bin/bash
O=gpurun_out/r4p; mkdir -p $O
for v in main g_ib2 g_ib3 g_ib4 g_cc1 main; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 4 >> $O/ab.txt 2>&1
done

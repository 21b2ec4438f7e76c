#!/bin/bash
O=gpurun_out/r2z2; mkdir -p $O
for L in paper_2001_01158_b200/liblc.so build_var/gib3/liblc.so build_var/gib4/liblc.so build_var/gib6/liblc.so build_var/gib3cc1/liblc.so build_var/gib3cc3/liblc.so; do
  timeout 300 python tools/dev/ab_solves.py $L 4 >> $O/ab.txt 2>&1
done

#!/bin/bash
O=gpurun_out/r4r; mkdir -p $O
for v in g_u1 g_u2 g_u4 g_u1; do
  timeout 300 python tools/dev/ab_solves.py build_var/$v/liblc.so 4 >> $O/ab.txt 2>&1
done

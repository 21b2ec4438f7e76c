#!/bin/bash
O=gpurun_out/r4h; mkdir -p $O
for v in l2h0 l2h1 l2h3 l2h0; do
  timeout 900 python tools/dev/ab_solves.py build_var/$v/liblc.so 2 3 5 1 >> $O/ab.txt 2>&1
done

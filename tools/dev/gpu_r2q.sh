#!/bin/bash
O=gpurun_out/r2q; mkdir -p $O
timeout 300 python tools/dev/tl_dyn.py build_dbg/liblc_dbg.so 3 > $O/tl_dyn.txt 2>&1
for v in dynr2 dynr8; do timeout 300 python tools/dev/ab_solves.py build_var/$v/liblc.so 3 >> $O/ab.txt 2>&1; done
timeout 300 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 3 >> $O/ab.txt 2>&1

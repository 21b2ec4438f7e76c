#!/bin/bash
O=gpurun_out/r3a; mkdir -p $O
L=paper_2001_01158_b200/liblc.so
for c in 148 296 444 592; do timeout 300 python tools/dev/ab_solves.py $L 2 5 --tune pcg_max_ctas=$c >> $O/ab.txt 2>&1; done

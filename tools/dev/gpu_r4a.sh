#!/bin/bash
# round 2 session 4 (a): GMRES A/B -- branch-free five-point SpMV row, one-round-trip reduce, coalesced basis access
O=gpurun_out/r4a; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gmres or config4 or 3t or block" > $O/pytest_gmres.log 2>&1; echo "EXIT $?" >> $O/pytest_gmres.log
for v in g_base main g_nocoal g_nored g_nosp g_minb1 g_minb1cc1 g_ib4; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 4 >> $O/ab.txt 2>&1
done

#!/bin/bash
O=gpurun_out/r4f; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gmres or config4 or 3t or block" > $O/pytest_gmres.log 2>&1; echo "EXIT $?" >> $O/pytest_gmres.log
for v in g_base main g_ib1 g_ib2 g_ib4 g_cc1 g_h0 main; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 4 >> $O/ab.txt 2>&1
done
timeout 300 python tools/tl_gmres.py build_var/g_tl/liblc.so > $O/tl_gmres.txt 2>&1

#!/bin/bash
O=gpurun_out/r4e; mkdir -p $O
for v in g_base main g_h1 g_h2 main; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 4 >> $O/ab.txt 2>&1
done
timeout 300 python tools/tl_gmres.py build_var/g_tl/liblc.so > $O/tl_gmres.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gmres -s 1 -c 1 -o $O/gmres_c4 -f \
  python tools/one_solve.py 4 > $O/ncu_gmres_c4.log 2>&1

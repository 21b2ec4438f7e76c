#!/bin/bash
O=gpurun_out/r4l; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg -s 2 -c 1 -o $O/pcg_c5_local -f \
  python tools/dev/local_one.py > $O/ncu_c5_local.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg -s 1 -c 1 -o $O/pcg_c2 -f \
  python tools/one_solve.py 2 > $O/ncu_c2.log 2>&1

#!/bin/bash
O=gpurun_out/r2t; mkdir -p $O
for i in 1 2 3; do
  timeout 120 python -m pytest tests/test_gpu_parity.py -k "dynamic_teams or config3" -x -q > $O/pytest_$i.log 2>&1
  echo "EXIT $?" >> $O/pytest_$i.log
  grep -q "EXIT 0" $O/pytest_$i.log || exit 0
done
L=paper_2001_01158_b200/liblc.so
timeout 300 python tools/dev/ab_solves.py $L 3 4 >> $O/ab.txt 2>&1
timeout 300 python tools/dev/ab_solves.py build_var/grev0/liblc.so 4 >> $O/ab.txt 2>&1
timeout 300 python tools/tl_gmres.py build_dbg/liblc_dbg.so > $O/tl_gmres.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -k "config4 or gmres" -x -q > $O/pytest_c4.log 2>&1

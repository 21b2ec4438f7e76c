#!/bin/bash
O=gpurun_out/r4o; mkdir -p $O
for v in main d_nob main d_nob; do
  lib=build_var/$v/liblc.so; [ $v = main ] && lib=paper_2001_01158_b200/liblc.so
  timeout 300 python tools/dev/ab_solves.py $lib 3 >> $O/ab.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_method.py -q -x -k "config3 or batched or dyn or team or 3" > $O/pytest_c3.log 2>&1; echo "EXIT $?" >> $O/pytest_c3.log

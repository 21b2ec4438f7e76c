#!/bin/bash
O=gpurun_out/r3d; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_ninepoint.py -q > $O/pytest_9.log 2>&1; echo "EXIT $?" >> $O/pytest_9.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_ds -s 1 -c 1 -o $O/pcgds_c1 -f \
  python tools/one_solve.py 1 > $O/ncu_pcgds.log 2>&1

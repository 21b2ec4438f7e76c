#!/bin/bash
O=gpurun_out/r2s; mkdir -p $O
timeout 200 python -m pytest tests/test_gpu_parity.py -k "dynamic_teams or config3" -x -q > $O/pytest.log 2>&1
echo "EXIT $?" >> $O/pytest.log
timeout 300 python tools/dev/tl_dyn.py build_dbg/liblc_dbg.so 3 > $O/tl_dyn.txt 2>&1
L=paper_2001_01158_b200/liblc.so
timeout 300 python tools/dev/ab_solves.py $L 3 >> $O/ab.txt 2>&1
timeout 300 python tools/dev/ab_solves.py build_var/dynr2/liblc.so 3 >> $O/ab.txt 2>&1
timeout 300 python tools/c3_ideal.py 3 > $O/c3.txt 2>&1
timeout 300 python tools/c3_ideal.py 10 >> $O/c3.txt 2>&1

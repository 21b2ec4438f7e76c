#!/bin/bash
O=gpurun_out/r2r; mkdir -p $O
timeout 200 python -m pytest tests/test_gpu_parity.py -k "dynamic_teams or config3" -x -q > $O/pytest.log 2>&1
echo "EXIT $?" >> $O/pytest.log
timeout 300 python tools/dev/tl_dyn.py build_dbg/liblc_dbg.so 3 > $O/tl_dyn.txt 2>&1
L=paper_2001_01158_b200/liblc.so
for t in 1 2; do timeout 300 python tools/dev/ab_solves.py $L 3 --tune batched_schedule=$t >> $O/ab.txt 2>&1; done
timeout 300 python tools/c3_ideal.py 3 > $O/c3.txt 2>&1

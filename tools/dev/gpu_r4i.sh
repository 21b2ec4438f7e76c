#!/bin/bash
O=gpurun_out/r4i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "l2_stream or lazy_x or subsystem_repr or determin" > $O/pytest_sel.log 2>&1; echo "EXIT $?" >> $O/pytest_sel.log
timeout 900 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 2 3 5 1 >> $O/ab.txt 2>&1
timeout 900 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 2 3 5 --tune l2_stream_hint=0 >> $O/ab.txt 2>&1
timeout 900 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 2 3 5 --tune l2_stream_hint=1 >> $O/ab.txt 2>&1

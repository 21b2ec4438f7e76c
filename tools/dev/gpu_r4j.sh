#!/bin/bash
O=gpurun_out/r4j; mkdir -p $O
timeout 900 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 2 3 5 1 >> $O/ab.txt 2>&1
timeout 900 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 2 3 5 --tune l2_stream_hint=0 >> $O/ab.txt 2>&1
timeout 900 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 2 3 5 --tune l2_stream_hint=1 >> $O/ab.txt 2>&1
timeout 900 python tools/dev/ab_solves.py build_var/l2h0/liblc.so 2 3 5 1 >> $O/ab.txt 2>&1

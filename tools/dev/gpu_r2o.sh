#!/bin/bash
O=gpurun_out/r2o; mkdir -p $O
for t in batched_cluster=0 batched_cluster=8; do timeout 300 python tools/dev/tl_c3.py build_dbg/liblc_dbg.so $t >> $O/tl.txt 2>&1; done

#!/bin/bash
O=gpurun_out/r2w; mkdir -p $O
timeout 600 python tools/heat_table2.py norm=vec grids=512:3 methods=0 > $O/t2_vec.jsonl 2>&1
timeout 1800 python tools/heat_table2.py norm=h grids=512:5,1024:3,2048:2,4096:1 > $O/t2_h.jsonl 2>&1
timeout 600 python tools/step_phases.py 1 > $O/phases_c1.txt 2>&1

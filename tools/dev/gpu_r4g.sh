#!/bin/bash
O=gpurun_out/r4g; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 300 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 4 >> $O/ab.txt 2>&1
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 > $O/bench_c4.jsonl 2> $O/bench_c4.err

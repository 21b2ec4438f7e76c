#!/bin/bash
O=gpurun_out/r4s; mkdir -p $O
timeout 300 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 1 >> $O/ab.txt 2>&1
timeout 300 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 1 --tune pcg_cluster_resident=1 >> $O/ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 600 python bench.py --config 1 --no-cpu-baseline > $O/bench_c1.jsonl 2>$O/bench_c1.err

#!/bin/bash
O=gpurun_out/r4u; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_method.py -q -x -k "gmres or config4 or 3t or block" > $O/pytest_gmres.log 2>&1; echo "EXIT $?" >> $O/pytest_gmres.log
timeout 300 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 4 >> $O/ab.txt 2>&1
timeout 600 python tools/ncu_traffic.py > $O/ncu_traffic.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5.jsonl 2>$O/bench_c5.err

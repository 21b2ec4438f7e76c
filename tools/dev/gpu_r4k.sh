#!/bin/bash
O=gpurun_out/r4k; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c5.jsonl 2>$O/bench_c5.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.jsonl 2>$O/bench_c$c.err; done

#!/bin/bash
O=gpurun_out/r2v; mkdir -p $O
for i in 1 2; do timeout 600 python bench.py --config 3 --no-cpu-baseline > $O/bench_c3_$i.jsonl 2>$O/bench_c3_$i.err; done
timeout 600 python bench.py --config 3 --no-cpu-baseline --tune batched_schedule=0 > $O/bench_c3_lock.jsonl 2>$O/bench_c3_lock.err

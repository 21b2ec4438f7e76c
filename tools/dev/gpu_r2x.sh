#!/bin/bash
O=gpurun_out/r2x; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -k "config1 or resident or dsmem or heat" -x -q > $O/pytest.log 2>&1; echo "EXIT $?" >> $O/pytest.log
for L in paper_2001_01158_b200/liblc.so build_var/dsmincl0/liblc.so build_var/dst1024/liblc.so; do
  timeout 300 python tools/dev/ab_solves.py $L 1 >> $O/ab.txt 2>&1
done
timeout 600 python bench.py --config 1 --no-cpu-baseline > $O/bench_c1.jsonl 2>$O/bench_c1.err
timeout 600 python tools/heat_experiment.py n=99 steps=100 > $O/heat99.json 2>&1

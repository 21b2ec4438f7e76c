#!/bin/bash
O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -k "config3 or spmv" -x -q > $O/pytest_c3.log 2>&1
L=paper_2001_01158_b200/liblc.so
timeout 300 python tools/c3_ideal.py 3 > $O/c3.txt 2>&1
for cl in 0 4 16; do timeout 300 python tools/dev/ab_solves.py $L 3 --tune batched_cluster=$cl >> $O/ab.txt 2>&1; done
timeout 300 python tools/dev/ab_solves.py $L 3 >> $O/ab.txt 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > $O/bench_c3.jsonl 2>$O/bench_c3.err

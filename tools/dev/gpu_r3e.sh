#!/bin/bash
O=gpurun_out/r3e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "EXIT $?" >> $O/pytest.log
L=paper_2001_01158_b200/liblc.so
timeout 300 python tools/dev/ab_solves.py $L 1 >> $O/ab.txt 2>&1
timeout 600 python bench.py --config 1 --no-cpu-baseline > $O/bench_c1.jsonl 2>$O/bench_c1.err
timeout 600 python tools/heat_experiment.py n=99 steps=100 > $O/heat99.json 2>&1

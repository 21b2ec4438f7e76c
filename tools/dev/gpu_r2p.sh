#!/bin/bash
O=gpurun_out/r2p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 120 python -m pytest tests/test_gpu_parity.py -k "dynamic_teams" -x -q > $O/pytest_dyn.log 2>&1
echo "EXIT $?" >> $O/pytest_dyn.log
grep -q "EXIT 0" $O/pytest_dyn.log || exit 0
timeout 300 python -m pytest tests/test_gpu_parity.py -k "config3" -x -q > $O/pytest_c3.log 2>&1
L=paper_2001_01158_b200/liblc.so
timeout 300 python tools/c3_ideal.py 3 > $O/c3.txt 2>&1
timeout 300 python tools/c3_ideal.py 10 >> $O/c3.txt 2>&1
timeout 300 python tools/dev/ab_solves.py $L 3 --tune batched_schedule=0 >> $O/ab.txt 2>&1
timeout 300 python tools/dev/ab_solves.py $L 3 >> $O/ab.txt 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > $O/bench_c3.jsonl 2>$O/bench_c3.err

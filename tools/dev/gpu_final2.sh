#!/bin/bash
O=gpurun_out/fin; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python tools/ncu_traffic.py > $O/ncu_traffic.log 2>&1
cp gpurun_out/ncu_traffic/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py > $O/bench_c5.jsonl 2>$O/bench_c5.err
for c in 1 3; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.jsonl 2>$O/bench_c$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launches.log 2>&1

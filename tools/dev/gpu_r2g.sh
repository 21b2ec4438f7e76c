#!/bin/bash
# round-2 session 2 check-in: GPU tests on the current head, bench config 5 + 3 + 4, k_pcg traffic stamp
O=gpurun_out/r2g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c5.jsonl 2>$O/bench_c5.err
for c in 1 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.jsonl 2>$O/bench_c$c.err; done
timeout 600 python tools/ncu_traffic.py > $O/ncu_traffic.log 2>&1
ls -la $O gpurun_out/ncu_traffic > $O/ls.txt

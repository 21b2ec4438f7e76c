#!/bin/bash
# full GPU suite + bench lines of every config on the current head
O=gpurun_out/r2u; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "EXIT $?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.jsonl 2>$O/bench_c$c.err; done
timeout 900 python bench.py > $O/bench_c5.jsonl 2>$O/bench_c5.err

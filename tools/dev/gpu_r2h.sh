#!/bin/bash
# one-call Alg. 1 (lc_local_method): GPU tests + bench configs 1, 5
O=gpurun_out/r2h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_method.py -x -q > $O/pytest_method.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in 1 4 3; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.jsonl 2>$O/bench_c$c.err; done
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c5.jsonl 2>$O/bench_c5.err

#!/bin/bash
O=gpurun_out/r2y; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -k "config4 or gmres or 3t or bsr" -x -q > $O/pytest.log 2>&1; echo "EXIT $?" >> $O/pytest.log
L=paper_2001_01158_b200/liblc.so
timeout 300 python tools/dev/ab_solves.py $L 4 >> $O/ab.txt 2>&1
timeout 300 python tools/dev/ab_solves.py $L 4 --tune block_dcoup=0 >> $O/ab.txt 2>&1
timeout 600 python bench.py --config 4 --no-cpu-baseline > $O/bench_c4.jsonl 2>$O/bench_c4.err

#!/bin/bash
O=gpurun_out/r2l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -k "spmv" -x -q > $O/pytest_spmv.log 2>&1
L=paper_2001_01158_b200/liblc.so
timeout 600 python tools/dev/ab_solves.py $L 1 2 3 5 > $O/ab.txt 2>&1
timeout 600 python tools/dev/ab_solves.py build_var/pt1024/liblc.so 1 2 3 5 >> $O/ab.txt 2>&1

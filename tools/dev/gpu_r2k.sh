#!/bin/bash
O=gpurun_out/r2k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -k "spmv" -x -q > $O/pytest_spmv.log 2>&1
timeout 300 python tools/spmv_ab.py 2 5 > $O/spmv.txt 2>&1
timeout 300 python tools/spmv_ab.py 5 >> $O/spmv.txt 2>&1

#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_method.py -x -q > $O/pytest_method.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
timeout 300 python tools/spmv_ab.py 2 5 > $O/spmv.txt 2>&1

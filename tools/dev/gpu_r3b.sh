#!/bin/bash
O=gpurun_out/r3b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_ninepoint.py -x -q > $O/pytest_9.log 2>&1; echo "EXIT $?" >> $O/pytest_9.log
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "EXIT $?" >> $O/pytest.log
L=paper_2001_01158_b200/liblc.so
timeout 300 python tools/dev/ab_solves.py $L 2 4 5 >> $O/ab.txt 2>&1

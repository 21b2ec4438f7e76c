#!/bin/bash
O=gpurun_out/r3c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_ninepoint.py -q > $O/pytest_9.log 2>&1; echo "EXIT $?" >> $O/pytest_9.log
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "EXIT $?" >> $O/pytest.log

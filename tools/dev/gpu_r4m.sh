#!/bin/bash
O=gpurun_out/r4m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > $O/pytest_dist.log 2>&1; echo "EXIT $?" >> $O/pytest_dist.log

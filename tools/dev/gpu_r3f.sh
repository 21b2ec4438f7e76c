#!/bin/bash
O=gpurun_out/r3f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -k "full_size_local_method or full_size_method0" -q --durations=10 > $O/pytest_full.log 2>&1; echo "EXIT $?" >> $O/pytest_full.log

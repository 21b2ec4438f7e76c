#!/bin/bash
O=gpurun_out/r4t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_resident or dsmem" > $O/pytest_sel.log 2>&1; echo "EXIT $?" >> $O/pytest_sel.log
timeout 900 python tools/heat_experiment.py > $O/heat_experiment.log 2>&1

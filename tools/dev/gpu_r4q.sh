#!/bin/bash
O=gpurun_out/r4q; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_method.py -q -x -k "gmres or config4 or 3t or block" > $O/pytest_gmres.log 2>&1; echo "EXIT $?" >> $O/pytest_gmres.log
timeout 300 python tools/dev/ab_solves.py paper_2001_01158_b200/liblc.so 4 >> $O/ab.txt 2>&1
timeout 300 python tools/dev/tl_gmres_local.py build_var/g_tl/liblc.so > $O/tl_local.txt 2>&1

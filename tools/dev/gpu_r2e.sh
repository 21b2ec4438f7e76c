#!/bin/bash
# round-2 A/B: TMA-staged explicit subsystems, CSR SpMV copy unrolled, config 1 step phases
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
L=paper_2001_01158_b200/liblc.so
timeout 200 python tools/time_local.py $L 5 2 3 > $O/local.txt 2>&1
timeout 200 python tools/time_local.py $L 5 2 3 pcg_tma=0 >> $O/local.txt 2>&1
timeout 200 python tools/spmv_ab.py 2 5 > $O/spmv.txt 2>&1
timeout 200 python tools/step_phases.py 1 > $O/phases_c1.txt 2>&1
timeout 200 python tools/step_phases.py 4 >> $O/phases_c1.txt 2>&1

timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
python tools/tl_cta.py build_dbg/liblc_dbg.so 3 1600 > gpurun_out/tl_c3_tail.jsonl 2>&1
python tools/tl_cta.py build_dbg/liblc_dbg.so 3 10 > gpurun_out/tl_c3_head.jsonl 2>&1
python tools/c3_ideal.py 3 > gpurun_out/t_c3_3.json 2>&1
python tools/c3_ideal.py 10 > gpurun_out/t_c3_10.json 2>&1

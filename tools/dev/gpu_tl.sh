timeout 600 python -m pytest tests -m gpu -x -q -k "determinism" > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
python tools/tl_cta.py build_dbg/liblc_dbg.so 3 1600 > gpurun_out/tl_c3_tail.jsonl 2>&1
python tools/tl_cta.py build_dbg/liblc_dbg.so 3 10 > gpurun_out/tl_c3_head.jsonl 2>&1
python tools/tl_cta.py build_dbg/liblc_dbg.so 3 800 > gpurun_out/tl_c3_mid.jsonl 2>&1

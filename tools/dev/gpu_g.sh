timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
python tools/time_lib.py paper_2001_01158_b200/liblc.so 4 > gpurun_out/t_ib.txt 2>&1
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/t_bench_c4.log 2>&1

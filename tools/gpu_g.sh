timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
python tools/tl_gmres.py build_dbg/liblc_dbg.so > gpurun_out/tl_gmres.txt 2>&1
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/t_bench_c4.log 2>&1

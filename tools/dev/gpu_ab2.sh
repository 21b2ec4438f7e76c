timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t_bench_c5.log 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/t_bench_c3.log 2>&1
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/t_bench_c4.log 2>&1
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/t_bench_c2.log 2>&1

# quick A/B: GPU tests, config 3 global solve device time, config 5 and 3 bench lines
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
python tools/c3_ideal.py 3 > gpurun_out/t_c3_3.json 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t_bench_c5.log 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/t_bench_c3.log 2>&1

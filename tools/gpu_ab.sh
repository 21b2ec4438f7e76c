# quick A/B: GPU tests, global solve device times (lazy x on / off), config 3 and 5 bench lines
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
timeout 300 python tools/time_pcg.py 5 2 3 > gpurun_out/t_pcg.txt 2>&1
LC_NO_LAZY_X=1 timeout 300 python tools/time_pcg.py 5 2 3 > gpurun_out/t_pcg_nolazy.txt 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/t_bench_c3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t_bench_c5.log 2>&1

# quick A/B: GPU tests, global solve device times (lazy x depth 3 / 2 / off), config 5 bench line
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
timeout 300 python tools/time_pcg.py 5 2 > gpurun_out/t_pcg.txt 2>&1
LC_LAZY_X_DEPTH=2 timeout 300 python tools/time_pcg.py 5 2 > gpurun_out/t_pcg_d2.txt 2>&1
LC_NO_LAZY_X=1 timeout 300 python tools/time_pcg.py 5 2 > gpurun_out/t_pcg_nolazy.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t_bench_c5.log 2>&1

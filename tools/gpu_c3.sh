# config 3 schedules: GPU tests, device time of the global solve, bench (auto / lock step forced)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
timeout 300 python tools/c3_ideal.py 3 > gpurun_out/t_c3_auto_3.json 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/t_bench_c3.log 2>&1
LC_TEAMS=0 timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/t_bench_c3_lockstep.log 2>&1

# batched lock step: parity tests, config 3 global solve device time, bench config 3
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
for s in 3 10; do echo "lock $s $(timeout 300 python tools/c3_ideal.py $s 2>&1 | tail -1)" >> gpurun_out/t_c3_sched.txt; done
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/t_bench_c3.log 2>&1

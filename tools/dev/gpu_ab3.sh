timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
for c in 5 3 2; do timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > gpurun_out/t_bench_c$c.log 2>&1; done

# batched lock step: config 3 global solve device time vs the TMA chunk threshold
timeout 600 python -m pytest tests -m gpu -x -q -k "batched or determinism" > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
for th in 4 8 16 32; do echo "th$th 3 $(LC_TMA_BATCH_CHUNKS=$th timeout 300 python tools/c3_ideal.py 3 2>&1 | tail -1)" >> gpurun_out/t_c3_sched.txt; done
echo "plain 3 $(LC_NO_TMA_BATCH=1 timeout 300 python tools/c3_ideal.py 3 2>&1 | tail -1)" >> gpurun_out/t_c3_sched.txt

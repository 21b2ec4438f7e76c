# batched schedules: parity tests, then config 3 global solve device time per schedule
timeout 600 python -m pytest tests -m gpu -x -q -k "batched" > gpurun_out/t_pytest.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/t_pytest.log
for sch in lock flow; do
 for s in 3 10; do
  echo "$sch $s $(LC_TEAMS=0 LC_BATCH=$sch timeout 300 python tools/c3_ideal.py $s 2>&1 | tail -1)" >> gpurun_out/t_c3_sched.txt
 done
done

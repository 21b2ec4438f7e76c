#!/bin/bash
# Round evidence on one box: GPU tests, smoke, bench lines of every config + the reference arm, the ncu launch
# list of the default bench, full ncu captures of the top kernels and the k_pcg DRAM traffic stamp.
O=gpurun_out/ev2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_c5.jsonl 2>$O/bench_c5.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.jsonl 2>$O/bench_c$c.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.jsonl 2>$O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg -s 3 -c 1 -o $O/pcg_c5 -f \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/ncu_pcg_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gmres -c 1 -o $O/gmres_c4 -f \
  python tools/one_solve.py 4 > $O/ncu_gmres_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_dyn -c 1 -o $O/pcgdyn_c3 -f \
  python tools/one_solve.py 3 > $O/ncu_pcgdyn_c3.log 2>&1
timeout 600 python tools/ncu_traffic.py > $O/ncu_traffic.log 2>&1
ls -la $O gpurun_out/ncu_traffic > $O/ls.txt
timeout 600 python tools/parity_sweep.py --configs 1,4 --out $O/parity_sweep_c1_c4.json > $O/parity_sweep_c1_c4.log 2>&1
timeout 1500 python tools/parity_sweep.py --configs 2,3,5 --out $O/parity_sweep_c2_c3_c5.json > $O/parity_sweep_c2_c3_c5.log 2>&1

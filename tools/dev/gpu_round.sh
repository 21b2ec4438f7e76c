# End-of-round evidence: bench lines for all configs, the reference arm, the ncu launch list of the default
# bench, full captures of the top kernels (k_pcg config 5 / config 3, k_gmres config 4) and the k_pcg DRAM traffic.
O=gpurun_out/round; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $O/smi.txt
timeout 600 python bench.py > $O/bench_c5.jsonl 2>&1
for c in 1 2 3 4; do timeout 600 python bench.py --config $c > $O/bench_c$c.jsonl 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg -s 3 -c 1 -o $O/pcg_c5 -f \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/ncu_pcg_c5.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_pcg python tools/one_solve.py 5 > $O/ncu_pcg_traffic.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gmres -c 1 -o $O/gmres_c4 -f \
  python tools/one_solve.py 4 > $O/ncu_gmres_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o $O/pcg_c3 -f \
  python tools/one_solve.py 3 > $O/ncu_pcg_c3.log 2>&1
ls -la $O > $O/ls.txt

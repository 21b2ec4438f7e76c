O=gpurun_out/tr; mkdir -p $O
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:k_pcg python tools/one_solve.py 5 > $O/ncu_pcg_traffic.log 2>&1
timeout 600 python bench.py > $O/bench_c5.jsonl 2>&1

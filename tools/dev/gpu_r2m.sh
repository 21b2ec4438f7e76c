#!/bin/bash
O=gpurun_out/r2m; mkdir -p $O
cd tools/micro && timeout 120 ./reduce_bench > ../../$O/reduce_bench.txt 2>&1; cd ../..

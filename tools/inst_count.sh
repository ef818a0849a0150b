#!/bin/bash
# Per-kernel executed warp instructions of one serial bench frame.
timeout 120 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/b0.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --cache-control none -c 400 --csv \
  --log-file gpurun_out/inst.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 \
  > gpurun_out/ncu.log 2>&1
echo "inst rc=$?"

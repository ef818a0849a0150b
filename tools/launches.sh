#!/bin/bash
# Serial launch list of one bench frame (ncu gpu__time_duration, cold cache).
timeout 120 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/b0.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 \
  > gpurun_out/ncu.log 2>&1
echo "launches rc=$?"

#!/bin/bash
# Per-kernel SM-cycles consumed by one serial bench frame (what bounds the
# concurrent throughput when the latency-bound stages overlap).
timeout 400 ncu --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__grid_size \
  --clock-control none -c 400 --csv --log-file gpurun_out/smtime.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/ncu_sm.log 2>&1
echo "smtime rc=$?"

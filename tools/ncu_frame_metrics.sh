#!/bin/bash
# Per-kernel evidence table of ONE cfg frame (tools/one_frame.py): duration,
# DRAM bytes, pipe utilisation, issue activity, occupancy -> gpurun_out/frame_metrics.csv
cfgid=${1:-5}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
M=$M,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
timeout 900 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/frame_metrics.csv python tools/one_frame.py "$cfgid" 3 > gpurun_out/ncu_fm.log 2>&1
echo "frame metrics rc=$?"
python tools/frame_metrics_summary.py gpurun_out/frame_metrics.csv

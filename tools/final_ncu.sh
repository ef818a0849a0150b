#!/bin/bash
# Round-end ncu evidence for the current build:
#  1. launch list of the bench command (B200_PROFILING.md recipe)
#  2. per-kernel metrics table of one config-5 frame
#  3. --set full capture of both aggregation launches of one frame
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras \
  > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
bash tools/ncu_frame_metrics.sh 5 > gpurun_out/frame_metrics.txt 2>&1
echo "frame metrics rc=$?"
bash tools/ncu_frame.sh aggfinal "k_aggregate_tma" 2 5
python tools/ncu_keys.py gpurun_out/aggfinal.ncu-rep > gpurun_out/aggfinal_keys.txt 2>&1
python tools/ncu_lines.py gpurun_out/aggfinal.ncu-rep 20 > gpurun_out/aggfinal_lines.txt 2>&1
echo done

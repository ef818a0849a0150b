#!/bin/bash
# DRAM bytes of both aggregation launches of one frame per BASELINE config
# (ncu, one frame via tools/one_frame.py) -> gpurun_out/agg_traffic_cfgN.csv
for c in 1 2 3 4 5; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --profile-from-start off -k regex:k_aggregate_tma -c 2 --csv \
    --log-file gpurun_out/agg_traffic_cfg$c.csv python tools/one_frame.py $c 3 > /dev/null 2>&1
  echo "cfg$c rc=$?"
done

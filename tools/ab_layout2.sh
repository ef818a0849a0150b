#!/bin/bash
# A/B of bootstrap SGM layouts on the checked build: args "G,WPL" for RPD_SGM_LAYOUT_BIG
for rep in 1 2; do
for v in "$@"; do
  RPD_SGM_LAYOUT_BIG=$v timeout 150 python bench.py --lib paper_2012_10802_b200/_lib_dbg/librpd_b200.so \
    --steps 20 --warmup 5 --no-cpu-baseline --no-extras > "gpurun_out/ly2_${v}_$rep.log" 2>&1
  python - "gpurun_out/ly2_${v}_$rep.log" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    s = d["stage_ms"]
    print(sys.argv[2], d["value"], d["e2e"]["value"], d["value_serial"], s["sgm_bootstrap"], s["sgm_pt"], d["roofline"]["agg_ms_per_frame"])
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
done

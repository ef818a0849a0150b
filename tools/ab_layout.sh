#!/bin/bash
# A/B of SGM layouts: args are "SMALL|BIG" pairs like 1,5/4,5
for v in "$@"; do
  sm=${v%/*}; bg=${v#*/}
  RPD_SGM_LAYOUT_SMALL=$sm RPD_SGM_LAYOUT_BIG=$bg timeout 100 python bench.py --steps 10 --warmup 3 \
    --no-cpu-baseline > "gpurun_out/ly_${sm}_${bg}.log" 2>&1
  python - "gpurun_out/ly_${sm}_${bg}.log" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    s = d["stage_ms"]
    print(sys.argv[2], d["value"], d["value_serial"], s["sgm_bootstrap"], s["sgm_pt"], d["roofline"]["agg_ms_per_frame"])
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done

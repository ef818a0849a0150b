#!/bin/bash
# A/B timing of the aggregation variants built by tools/build_agg_variants.sh
for v in "$@"; do
  RPD_B200_LIB=paper_2012_10802_b200/_lib/var_$v/librpd_b200.so timeout 100 \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
done
for v in "$@"; do
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.log").read().strip().splitlines()[-1])
    s = d["stage_ms"]
    print(v, d["value"], d["value_serial"], s["sgm_bootstrap"], s["sgm_pt"], d["roofline"]["agg_ms_per_frame"])
except Exception as e:
    print(v, "failed", e)
PY
done

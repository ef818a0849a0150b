#!/bin/bash
# A/B of the SLIC incremental modes on the checked build (RPD_SLIC_INCREMENTAL = 0 / 1 / 2)
for rep in 1 2 3; do
for v in "$@"; do
  RPD_SLIC_INCREMENTAL=$v timeout 150 python bench.py --lib paper_2012_10802_b200/_lib_dbg/librpd_b200.so \
    --steps 20 --warmup 5 --no-cpu-baseline --no-extras > "gpurun_out/si_${v}_$rep.log" 2>&1
  python - "gpurun_out/si_${v}_$rep.log" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    s = d["stage_ms"]
    print(sys.argv[2], d["value"], d["e2e"]["value"], d["value_serial"], s["slic"])
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
done

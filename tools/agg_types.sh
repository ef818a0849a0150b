#!/bin/bash
# Aggregation time (serial bench frame) with only some job types launched (RPD_TMA_TYPES bitmask:
# 1 = horizontal, 2 = vertical, 4 = diagonal); results are garbage, timing only.
for m in 7 1 2 4 3 6; do
  RPD_TMA_TYPES=$m timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/at_$m.log 2>&1
  python - $m <<'PY'
import json, sys
m = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/at_{m}.log").read().strip().splitlines()[-1])
    print(f"types {m}: agg {d['roofline']['agg_ms_per_frame']:.4f} ms/frame, sgm_bo {d['stage_ms']['sgm_bootstrap']:.3f} sgm_pt {d['stage_ms']['sgm_pt']:.3f}")
except Exception as e:
    print(m, "failed", open(f"gpurun_out/at_{m}.log").read()[-300:])
PY
done

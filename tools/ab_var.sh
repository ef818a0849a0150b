#!/bin/bash
# ab_var.sh V1 V2 ... : bench each paper_2012_10802_b200/_lib/var_V (2 runs each, interleaved)
for rep in 1 2; do
  for v in "$@"; do
    timeout 120 python bench.py --lib paper_2012_10802_b200/_lib/var_$v/librpd_b200.so \
      --steps 20 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab_${v}_$rep.log 2>&1
  done
done
for v in "$@"; do
  for rep in 1 2; do
    python - "$v" "$rep" <<'PY'
import json, sys
v, rep = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}_{rep}.log").read().strip().splitlines()[-1])
    s = d["stage_ms"]
    print(f"{v:10s} {d["value"]:8.1f} agg {d["roofline"]["agg_ms_per_frame"]:.4f} serial {d['value_serial']:7.1f} e2e {d['e2e']['value']:7.1f} " +
          " ".join(f"{k[:6]}={x:.3f}" for k, x in s.items()))
except Exception as e:
    print(v, "failed", e)
PY
  done
done

#!/bin/bash
# ab_var3.sh V1 V2 ... : like ab_var.sh with 3 interleaved runs each
for rep in 1 2 3; do
  for v in "$@"; do
    timeout 120 python bench.py --lib paper_2012_10802_b200/_lib/var_$v/librpd_b200.so \
      --steps 20 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab_${v}_$rep.log 2>&1
  done
done
for v in "$@"; do
  python - "$v" <<'PY'
import json, sys, statistics
v = sys.argv[1]
vals = []
for rep in (1, 2, 3):
    try:
        d = json.loads(open(f"gpurun_out/ab_{v}_{rep}.log").read().strip().splitlines()[-1])
        vals.append((d["value"], d["e2e"]["value"], d["value_serial"]))
    except Exception as e:
        pass
if vals:
    print(f"{v:8s} n={len(vals)} value {statistics.mean(x[0] for x in vals):7.1f} "
          f"(min {min(x[0] for x in vals):.1f}) e2e {statistics.mean(x[1] for x in vals):7.1f} "
          f"serial {statistics.mean(x[2] for x in vals):6.1f}")
PY
done

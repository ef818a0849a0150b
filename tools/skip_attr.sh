#!/bin/bash
# Cost attribution in the concurrent regime: bench with RPD_SKIP_STAGES masks.
for m in "$@"; do
  RPD_SKIP_STAGES=$m timeout 120 python bench.py --lib paper_2012_10802_b200/_lib_dbg/librpd_b200.so --no-extras --steps 20 --warmup 5 --no-cpu-baseline \
    > gpurun_out/sk_$m.log 2>&1
done
for m in "$@"; do
  python - "$m" <<'PY'
import json, sys
m = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sk_{m}.log").read().strip().splitlines()[-1])
    print(f"skip {m:>3s}: value {d['value']:8.1f}  serial {d['value_serial']:7.1f}  ms/frame {1000/d['value']:.3f}")
except Exception as e:
    lines = open(f"gpurun_out/sk_{m}.log").read().strip().splitlines()
    print(f"skip {m}: failed: {lines[-1][:150] if lines else e}")
PY
done

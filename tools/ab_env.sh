#!/bin/bash
# ab_env.sh "ENV=1" "ENV2=x" ... : interleaved bench runs (2 each) under env settings ("-" = none)
for rep in 1 2; do
  for e in "$@"; do
    tag=$(echo "$e" | tr -c 'A-Za-z0-9_\n' '_')
    if [ "$e" = "-" ]; then envs=X_NONE=1; else envs=$e; fi
    env $envs timeout 150 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/abe_${tag}_$rep.log 2>&1
  done
done
for e in "$@"; do
  tag=$(echo "$e" | tr -c 'A-Za-z0-9_\n' '_')
  for rep in 1 2; do
    python - "$tag" "$rep" "$e" <<'PY'
import json, sys
t, rep, e = sys.argv[1:4]
try:
    d = json.loads(open(f"gpurun_out/abe_{t}_{rep}.log").read().strip().splitlines()[-1])
    s = d["stage_ms"]
    print(f"{e[:28]:28s} {d['value']:8.1f} serial {d['value_serial']:7.1f} e2e {d['e2e']['value']:7.1f} " +
          " ".join(f"{k[:6]}={x:.3f}" for k, x in s.items()))
except Exception as ex:
    print(e, "failed", open(f"gpurun_out/abe_{t}_{rep}.log").read()[-400:])
PY
  done
done

#!/bin/bash
# ab_cfg.sh CONFIG V1 V2 ...: 2 interleaved bench runs per variant library on one BASELINE config
c=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    timeout 200 python bench.py --config $c --lib paper_2012_10802_b200/_lib/var_$v/librpd_b200.so \
      --steps 20 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/abc_${c}_${v}_$rep.log 2>&1
    python - "gpurun_out/abc_${c}_${v}_$rep.log" "cfg$c $v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], d["value"], d["e2e"]["value"], d["value_serial"], d["stage_ms"]["slic"])
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
  done
done

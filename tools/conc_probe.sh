#!/bin/bash
# Concurrency probes: value under different stream counts / hardware queue limits / config overrides.
run() {  # tag, env..., -- bench args
  local tag=$1; shift
  env "$@" timeout 150 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BARGS} > gpurun_out/cp_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/cp_{t}.log").read().strip().splitlines()[-1])
    print(f"{t:24s} value {d['value']:8.1f} serial {d['value_serial']:7.1f} e2e {d['e2e']['value']:7.1f}")
except Exception as e:
    print(t, "failed", open(f"gpurun_out/cp_{t}.log").read()[-300:])
PY
}
BARGS="--streams 8" run s8 X=1
BARGS="--streams 8" run s8_c32 CUDA_DEVICE_MAX_CONNECTIONS=32
BARGS="--streams 16" run s16_c32 CUDA_DEVICE_MAX_CONNECTIONS=32
BARGS="--streams 24" run s24_c32 CUDA_DEVICE_MAX_CONNECTIONS=32
BARGS="--streams 8" run s8_it1 RPD_BENCH_CFG=slic_iterations=1
BARGS="--streams 8" run s8_p4 RPD_BENCH_CFG=sgm_paths=4

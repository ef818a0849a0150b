#!/bin/bash
# e2e frames/s vs host threads (fewer threads than contexts: async streaming C-ABI)
for et in 16 4 2; do
  timeout 150 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras --e2e-threads $et > gpurun_out/e2e_$et.log 2>&1
  tail -1 gpurun_out/e2e_$et.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads $et', d['value'], d['e2e'])" || tail -3 gpurun_out/e2e_$et.log
done

#!/bin/bash
# concurrent frames/s vs number of pipeline contexts (streams)
for s in 4 8 16 24 32 48; do
  timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --streams $s --frames $((2*s)) > gpurun_out/ss_$s.log 2>&1
  tail -1 gpurun_out/ss_$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams $s', d['value'], d['e2e']['value'])" || tail -3 gpurun_out/ss_$s.log
done

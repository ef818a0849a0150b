#!/bin/bash
# Round-end evidence: full GPU suite (writes the parity sweep JSON), then one
# bench line per BASELINE config -> gpurun_out/bench_cfgN.json
RPD_SWEEP_JSON=gpurun_out/parity_sweep.json timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1
tail -3 gpurun_out/t.log
for c in 5 1 2 3 4; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_cfg$c.log 2>&1
  tail -1 gpurun_out/bench_cfg$c.log > gpurun_out/bench_cfg$c.json
  python -c "import json; d=json.load(open('gpurun_out/bench_cfg$c.json')); print('cfg$c', d['value'], d['value_serial'], d['e2e']['value'], d['roofline']['agg_ms_per_frame'], d.get('cpu_baseline',{}).get('value'))" || tail -3 gpurun_out/bench_cfg$c.log
done

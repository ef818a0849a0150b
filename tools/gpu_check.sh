#!/bin/bash
# GPU tests + a short bench; prints the test summary and the key bench numbers.
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/b.log 2>&1
tail -2 gpurun_out/t.log
tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'serial', d['value_serial'], 'e2e', d['e2e']['value'], d['stage_ms'], 'agg', d['roofline']['agg_ms_per_frame'])" || tail -5 gpurun_out/b.log

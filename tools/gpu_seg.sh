timeout 300 python -m pytest tests/test_parity_sgm_segments.py tests/test_parity_sgm_production.py tests/test_known_sgm.py -m gpu -q -x > gpurun_out/t2.log 2>&1
tail -15 gpurun_out/t2.log
timeout 500 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1
tail -3 gpurun_out/t.log
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b.log 2>&1
tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'serial', d['value_serial'], 'e2e', d['e2e']['value'], d['stage_ms'], 'agg', d['roofline']['agg_ms_per_frame'])" || tail -5 gpurun_out/b.log

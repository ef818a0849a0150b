#!/bin/bash
# quick parity (SGM layouts + segments + one config) then A/B of the given variants
timeout 600 python -m pytest tests/test_parity_sgm_segments.py tests/test_parity_sgm_production.py tests/test_known_sgm.py tests/test_parity_sgm.py tests/test_parity_configs.py -m gpu -q -x > gpurun_out/tq.log 2>&1
tail -3 gpurun_out/tq.log
bash tools/ab_var.sh "$@"

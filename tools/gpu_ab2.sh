#!/bin/bash
# pipeline parity (SLIC, configs, guards) then A/B of the given variants
timeout 600 python -m pytest tests/test_parity_pipeline.py tests/test_parity_configs.py tests/test_guards.py tests/test_known_segmentation.py -m gpu -q -x > gpurun_out/tq.log 2>&1
tail -3 gpurun_out/tq.log
bash tools/ab_var.sh "$@"

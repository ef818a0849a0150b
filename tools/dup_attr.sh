#!/bin/bash
# Marginal stage costs in the concurrent regime with the debug-knob build
# (make -C paper_2012_10802_b200/csrc DEBUG_KNOBS=1): RPD_DUP_STAGES runs a
# stage twice.  1 = refit, 2 = SLIC, 4 = detection, 8 = bootstrap SGM, 16 = PT SGM.
LIB=paper_2012_10802_b200/_lib_dbg/librpd_b200.so
for d in 0 1 2 4 8 16; do
  v=$(RPD_DUP_STAGES=$d timeout 150 python bench.py --lib $LIB --steps 20 --warmup 5 \
      --no-cpu-baseline --no-extras | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])")
  echo "dup=$d value=$v"
done

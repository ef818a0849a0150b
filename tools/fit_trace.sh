#!/bin/bash
# clock64 trace of the road fits of one cfg frame (checked build, RPD_FIT_TRACE=1)
RPD_FIT_TRACE=1 timeout 120 python - <<'PY' > gpurun_out/fit_trace.log 2>&1
import sys
sys.path.insert(0, ".")
from paper_2012_10802_b200.api import Library
from paper_2012_10802_b200.synth import make_scene, pipeline_config
lib = Library("paper_2012_10802_b200/_lib_dbg/librpd_b200.so")
ctx = lib.context(0)
sc = make_scene(5, 0)
cfg = pipeline_config(lib, 5)
for _ in range(2):
    ctx.detect(sc.left, sc.right, cfg)
PY
python tools/fit_trace.py gpurun_out/fit_trace.log

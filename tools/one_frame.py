"""Runs warm-up frames, then ONE cfg frame inside cudaProfilerStart/Stop, for
ncu --profile-from-start off (per-kernel pipe / instruction breakdowns):
python tools/one_frame.py [config] [warmup]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2012_10802_b200 as pkg  # noqa: E402
from paper_2012_10802_b200.synth import SHAPES, make_scene, pipeline_config  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = pkg.load_library()
ctx = lib.context(0)
h, w = SHAPES[c]
cfg = pipeline_config(lib, c)
sc = make_scene(c, 0)
ld = torch.from_numpy(sc.left).cuda()
rd = torch.from_numpy(sc.right).cuda()
for _ in range(warm):
    ctx.detect_async_u8(ld.data_ptr(), rd.data_ptr(), h, w, cfg)
    ctx.fetch()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ctx.detect_async_u8(ld.data_ptr(), rd.data_ptr(), h, w, cfg)
ctx.fetch()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", ctx.stats().kernels_last_frame)

"""Times the device scene generator on the acceptance batch (profiling helper)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_10802_b200 as pkg  # noqa: E402
from paper_2012_10802_b200.scenes import BatchRanges, batch_spec  # noqa: E402

sigma = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = pkg.load_library().context(0)
specs = [batch_spec(ctx.lib, 7100, i, BatchRanges(noise_sigma=sigma)) for i in range(20)]
h, w = specs[0].height, specs[0].width
dv = torch.device("cuda", 0)
bl = torch.empty((20, h, w), dtype=torch.float32, device=dv)
br, bg = torch.empty_like(bl), torch.empty_like(bl)
bm = torch.empty((20, h, w), dtype=torch.int32, device=dv)
torch.cuda.synchronize()
for i in range(reps + 1):
    if i == 1:
        t0 = time.perf_counter()
    ctx.generate_scenes_device(specs, bl.data_ptr(), br.data_ptr(), bg.data_ptr(), bm.data_ptr())
dt = (time.perf_counter() - t0) / reps
print(f"sigma {sigma}: {dt * 1e3:.3f} ms per batch of 20, {20 / dt:.1f} scenes/s")

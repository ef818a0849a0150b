"""The native C++ frame server (examples/rpd_stream.cpp) on the C-ABI: K
contexts driven by fewer host threads through rpd_detect_async_host_u8 /
rpd_detect_fetch, pinned buffers, no Python or torch in the loop.  Every pass
through a scene must give the same pothole count, and the counts must equal
the Python API's detect on the same u8 frames."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2012_10802_b200" / "_lib"


@pytest.mark.gpu
def test_cpp_frame_server(tmp_path, gpu):
    exe = tmp_path / "rpd_stream"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "rpd_stream.cpp"), "-o", str(exe),
                    "-L", str(LIBDIR), "-lrpd_b200", f"-Wl,-rpath,{LIBDIR}", "-lpthread"],
                   check=True)
    out = subprocess.run([str(exe), "96", "8", "3", "6"], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    rep = json.loads(out.stdout.strip().splitlines()[-1])
    assert rep["frames"] == 96 and rep["contexts"] == 8 and rep["threads"] == 3
    assert rep["inconsistent"] == 0 and rep["frames_per_s"] > 0
    # the same frames through the Python mirror of the ABI
    from paper_2012_10802_b200.scenes import BatchRanges, batch_spec
    lib = gpu.lib
    cfg = lib.default_config(delta_pd=0.48, superpixels=2400)
    for i, n_pot in enumerate(rep["potholes"]):
        spec = batch_spec(lib, 7100, i, BatchRanges())
        sc = gpu.generate_scene(spec)
        left = sc[0].astype(np.uint8)
        right = sc[1].astype(np.uint8)
        res = gpu.detect(left, right, cfg, want=("labels",))
        assert res.n_potholes == n_pot, (i, res.n_potholes, n_pot)

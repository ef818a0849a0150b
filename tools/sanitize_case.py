"""A small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): full detect on a reduced scene and BASELINE config 1,
the production SGM dump, aggregate_costs through k_aggregate_tma, SLIC and
the road fit through the C-ABI, each checked against the CPU oracle."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402

import paper_2012_10802_b200 as pkg  # noqa: E402
from paper_2012_10802_b200.api import Library, model  # noqa: E402
from paper_2012_10802_b200.synth import make_scene, pipeline_config, small_scene  # noqa: E402

lib = pkg.load_library()
g = lib.context(0)
orc = Library(str(ROOT / "oracle" / "_build" / "librpd_oracle.so"))
o = orc.context()


def same(cfg):
    return orc.default_config(**{k: getattr(cfg, k) for k, _ in cfg._fields_})


s = small_scene(96, 160, seed=4242, potholes=2)
cfg = lib.default_config(d_max=47, lambda1=10.0, lambda2=120.0, superpixels=120)
a, b = g.detect(s.left, s.right, cfg), o.detect(s.left, s.right, same(cfg))
assert np.array_equal(a.d1.view(np.uint32), b.d1.view(np.uint32)) and np.array_equal(a.labels, b.labels)
a = g.detect(s.left, s.right, cfg)  # graph replay
sc = make_scene(1, 0)
a = g.detect(sc.left, sc.right, pipeline_config(lib, 1))
b = o.detect(sc.left, sc.right, pipeline_config(orc, 1))
assert np.array_equal(a.labels, b.labels)
left, right = s.left.astype(np.float32), s.right.astype(np.float32)
da = g.match_pair_dump_ex(left[:40], right[:40], model(4.0, 0.05, 0.02), cfg, 16)
db = o.match_pair_dump_ex(left[:40], right[:40], model(4.0, 0.05, 0.02), same(cfg), 16)
assert all(np.array_equal(da[k], db[k]) for k in da)
vol = np.random.default_rng(1).integers(0, 61, (9, 13, 6)).astype(np.float32)
assert np.array_equal(g.aggregate_costs(vol, 7.0, 21.0), o.aggregate_costs(vol, 7.0, 21.0))
print("sanitize case ok")

import sys; sys.path.insert(0,'/root/repo')
import numpy as np, paper_2012_10802_b200 as pkg
from paper_2012_10802_b200.synth import small_scene
lib = pkg.load_library(); g = lib.context(0)
s = small_scene(128,192,seed=1001, potholes=2)
cfg = lib.default_config(d_max=47, lambda1=10.0, lambda2=120.0, superpixels=150)
for i in range(3):
    try:
        r = g.detect(s.left, s.right, cfg); print(i, 'ok', r.n_potholes, r.total_ms, r.stage_ms)
    except Exception as e: print(i, 'ERR', e)

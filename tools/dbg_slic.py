import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2012_10802_b200 as pkg
from paper_2012_10802_b200 import synth
from paper_2012_10802_b200.api import Library
lib = Library("paper_2012_10802_b200/_lib_dbg/librpd_b200.so"); ctx = lib.context(0)
sc = synth.make_scene(5, 0); cfg = synth.pipeline_config(lib, 5)
out = ctx.detect(sc.left, sc.right, cfg)
st = ctx.stats(); print('after detect', st.slic_tiles_assigned, st.slic_tiles_skipped)
for it in (1, 2, 3, 5, 10):
    b = ctx.stats()
    r = ctx.slic(out.d2, 2000, cfg.compactness, it)
    a = ctx.stats()
    print(it, a.slic_tiles_assigned - b.slic_tiles_assigned, a.slic_tiles_skipped - b.slic_tiles_skipped, (a.slic_centres_moved - b.slic_centres_moved) & 0xFFFFFFFF, (a.slic_centres_moved - b.slic_centres_moved) >> 32)

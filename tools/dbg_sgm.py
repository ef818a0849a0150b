"""Quick GPU-vs-oracle SGM check used while iterating on kernels."""
import sys, time
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2012_10802_b200 as pkg
from paper_2012_10802_b200.api import Library, model
from test_parity_sgm import stereo_pair
g = pkg.load_library().context(0)
o = Library('/root/repo/oracle/_build/librpd_oracle.so').context()
for (h, w, dm, paths, m) in [(41, 140, 0, 4, model()), (41, 140, 16, 8, model()), (64, 120, 16, 8, model(11, 0.08, 0.03)),
                             (41, 140, 64, 8, model()), (41, 300, 128, 8, model()), (24, 300, 256, 8, model())]:
    l, r = stereo_pair(h, w, 3, a0=dm * 0.4 + 1, a1=0.0, phi=0.0)
    cfg = g.lib.default_config(lambda1=10.0, lambda2=120.0, sgm_paths=paths)
    try:
        a = g.match_pair(l, r, m, cfg, dm)
    except Exception as e:
        print(h, w, dm, 'ERR', e); break
    b = o.match_pair(l, r, m, cfg, dm)
    ok = all(np.array_equal(x.view(np.uint32) if x.dtype == np.float32 else x, y.view(np.uint32) if y.dtype == np.float32 else y) for x, y in zip(a, b))
    print(h, w, dm, paths, 'ok' if ok else 'MISMATCH', (a[0] != b[0]).sum())

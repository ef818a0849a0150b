import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2012_10802_b200 as pkg
from test_sincos import _ref
g = pkg.load_library().context(0)
rng = np.random.default_rng(20121080)
for name, x in [("small", rng.uniform(-0.27, 0.27, 3000)), ("mid", rng.uniform(-0.75, 0.75, 1000)), ("big", rng.uniform(-3, 3, 500))]:
    s, c = g.debug_sincos(x)
    ref = np.array([_ref(v) for v in x])
    bs = np.nonzero(s != ref[:, 0])[0]; bc = np.nonzero(c != ref[:, 1])[0]
    print(name, "sin bad", len(bs), "cos bad", len(bc))
    for i in list(bs[:3]) + list(bc[:3]):
        print("  x=%r s=%r/%r c=%r/%r ulps s %d c %d" % (x[i], s[i], ref[i,0], c[i], ref[i,1],
              int(np.float64(s[i]).view(np.int64) - np.float64(ref[i,0]).view(np.int64)),
              int(np.float64(c[i]).view(np.int64) - np.float64(ref[i,1]).view(np.int64))))
x = np.array([0.0, 1e-300, -1e-12, 0.75, -0.75])
s, c = g.debug_sincos(x)
for i in range(len(x)):
    print(x[i], s[i], _ref(x[i])[0], c[i], _ref(x[i])[1])

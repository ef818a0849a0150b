"""Per-CTA timeline of the aggregation launches of one frame (checked build,
RPD_TMA_DBG=100 device printf): python tools/agg_timeline.py [config]
Prints, per pass and job type, CTA count, start spread, duration stats and
the makespan; and which CTAs end last."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if os.environ.get("AGGTL_CHILD") != "1":
    env = dict(os.environ, AGGTL_CHILD="1", RPD_TMA_DBG="100")
    out = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True,
                         text=True).stdout
    rows = [l.split()[1:] for l in out.splitlines() if l.startswith("AGGTR")]
    rows = [list(map(int, r)) for r in rows]
    # WPL G blk jidx type seg nseg smid t0 t1
    import collections
    launches = collections.defaultdict(list)
    for r in rows:
        launches[(r[0], r[1])].append(r)
    names = {0: "H", 1: "V", 2: "D"}
    for key, rs in launches.items():
        t0 = min(r[8] for r in rs)
        tend = max(r[9] for r in rs)
        print(f"== WPL={key[0]} G={key[1]}: {len(rs)} CTAs, makespan {(tend - t0) / 1e3:.1f} us")
        for ty in range(3):
            sel = [r for r in rs if r[4] == ty]
            if not sel:
                continue
            d = sorted((r[9] - r[8]) / 1e3 for r in sel)
            st = sorted((r[8] - t0) / 1e3 for r in sel)
            en = sorted((r[9] - t0) / 1e3 for r in sel)
            print(f"  {names[ty]}: n={len(sel)} start [{st[0]:.1f}, {st[-1]:.1f}] dur min/med/max "
                  f"{d[0]:.1f}/{d[len(d)//2]:.1f}/{d[-1]:.1f} end med/max {en[len(en)//2]:.1f}/{en[-1]:.1f}")
        last = sorted(rs, key=lambda r: -r[9])[:5]
        for r in last:
            print(f"  last: blk {r[2]} type {names[r[4]]} seg {r[5]}/{r[6]} sm {r[7]} "
                  f"start {(r[8]-t0)/1e3:.1f} end {(r[9]-t0)/1e3:.1f}")
        per_sm = collections.Counter(r[7] for r in rs)
        print(f"  CTAs per SM: min {min(per_sm.values())} max {max(per_sm.values())}")
    sys.exit(0)

sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2012_10802_b200.api import Library  # noqa: E402
from paper_2012_10802_b200.synth import make_scene, pipeline_config  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lib = Library(str(ROOT / "paper_2012_10802_b200" / "_lib_dbg" / "librpd_b200.so"))
ctx = lib.context(0)
sc = make_scene(c, 0)
cfg = pipeline_config(lib, c)
ctx.detect(sc.left, sc.right, cfg)

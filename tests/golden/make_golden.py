"""Generates tests/golden/ref_golden.npz from the LITERAL reference build
(oracle/_ref/librpd_ref.so = the untouched /root/reference/proj/src sources,
see oracle/Makefile).  Run in the build container, where /root/reference
exists:

    python tests/golden/make_golden.py

The fixture holds the INPUTS as well (uint8 pairs, rasters, observations), so
the checks in tests/test_golden.py depend on nothing but this file: they pin
the restated oracle (CPU) and the CUDA product (GPU) to outputs of the
reference's own code even where oracle/_ref cannot be rebuilt.

Cases (reference entry points in brackets):
  pipe_*   detect_potholes_pipeline on a 96x160 scene, 8 paths  [pipeline.cpp:47-109]
  pipe4_*  the same stages with the first 4 directions on 72x104 (BASELINE config 1's P=4)
  sgm_*    match_pair with a road model on a 40x64 pair         [sgm.cpp:172-226]
  slic_*   slic on a 60x80 raster with invalid pixels           [segmentation.cpp:170-229]
  fit_*    fit_road on 20 000 noisy observations with outliers  [road_geometry.cpp:70-101]
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2012_10802_b200.api import Library, model  # noqa: E402
from paper_2012_10802_b200.synth import small_scene  # noqa: E402

REF = ROOT / "oracle" / "_ref" / "librpd_ref.so"


def cases():
    """Inputs and the configuration overrides of every case (shared with the test)."""
    out = {}
    s = small_scene(96, 160, seed=1234, potholes=2)
    out["pipe"] = dict(left=s.left, right=s.right,
                       cfg=dict(d_max=47, lambda1=10.0, lambda2=120.0, superpixels=120))
    s4 = small_scene(72, 104, seed=99, potholes=1, axes=(7.0, 11.0), d_max=24.0)
    out["pipe4"] = dict(left=s4.left, right=s4.right,
                        cfg=dict(d_max=31, lambda1=10.0, lambda2=120.0, superpixels=60, sgm_paths=4))
    rng = np.random.default_rng(2012)
    left = rng.integers(0, 256, (40, 64)).astype(np.float32)
    right = np.rint(np.clip(np.roll(left, 5, axis=1) + rng.normal(0, 4, (40, 64)), 0, 255))
    out["sgm"] = dict(left=left, right=right.astype(np.float32), mdl=(5.0, 0.07, 0.02), d_max=16,
                      cfg=dict(lambda1=10.0, lambda2=120.0, sgm_paths=8))
    v, u = np.mgrid[0:60, 0:80]
    d2 = (0.05 * v + 0.02 * u + rng.normal(0, 0.5, (60, 80))).astype(np.float32)
    d2[rng.random((60, 80)) < 0.03] = -1.0
    out["slic"] = dict(d2=d2, p=30, comp=8.0, it=10)
    k = 20000
    fu = rng.integers(0, 640, k).astype(np.float64)
    fv = rng.integers(0, 480, k).astype(np.float64)
    phi = -0.04
    fd = 12.0 + 0.09 * (fv * np.cos(phi) - fu * np.sin(phi)) + rng.normal(0, 0.2, k)
    fd[:900] -= 5.0
    out["fit"] = dict(d=fd.astype(np.float32).astype(np.float64), u=fu, v=fv,
                      bracket=0.261799, tol=1e-4)
    return out


def run(ctx, c):
    """Every case through one library context -> flat dict of arrays."""
    lib = ctx.lib
    r = {}
    for name in ("pipe", "pipe4"):
        cfg = lib.default_config(**c[name]["cfg"])
        o = ctx.detect(c[name]["left"], c[name]["right"], cfg)
        for f in ("d0", "d1", "d2", "d3", "sp_labels", "labels"):
            r[f"{name}_{f}"] = np.asarray(getattr(o, f))
        r[f"{name}_n_potholes"] = np.array([o.n_potholes])
        # (the reference's DetectResult keeps the final fit only)
        r[f"{name}_model"] = np.array([o.fit.model.a0, o.fit.model.a1, o.fit.model.phi])
        r[f"{name}_used"] = np.array([o.fit.used, o.sp_count])
    cfg = lib.default_config(**c["sgm"]["cfg"])
    d0, d1 = ctx.match_pair(c["sgm"]["left"], c["sgm"]["right"], model(*c["sgm"]["mdl"]), cfg,
                            c["sgm"]["d_max"])[:2]
    r["sgm_d0"], r["sgm_d1"] = np.asarray(d0), np.asarray(d1)
    lab, cen, n, sp = ctx.slic(c["slic"]["d2"], c["slic"]["p"], c["slic"]["comp"], c["slic"]["it"])
    r["slic_labels"], r["slic_centers"] = np.asarray(lab), np.asarray(cen)
    r["slic_count_spacing"] = np.array([float(n), float(sp)])
    f = ctx.fit_road(c["fit"]["d"], c["fit"]["u"], c["fit"]["v"], c["fit"]["bracket"], c["fit"]["tol"])
    r["fit_model"] = np.array([f.model.a0, f.model.a1, f.model.phi])
    r["fit_used"] = np.array([f.used])
    return r


def main():
    if not REF.exists():
        raise SystemExit(f"{REF} missing: make -C oracle (needs /root/reference)")
    c = cases()
    r = run(Library(str(REF)).context(), c)
    ins = {}
    for name, d in c.items():
        for k, v in d.items():
            if isinstance(v, np.ndarray):
                ins[f"in_{name}_{k}"] = v
    out = Path(__file__).with_name("ref_golden.npz")
    np.savez_compressed(out, **ins, **r)
    print(out, out.stat().st_size, "bytes;", len(r), "outputs")


if __name__ == "__main__":
    main()

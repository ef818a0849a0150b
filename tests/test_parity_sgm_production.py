"""Bit-exact parity of the PRODUCTION SGM buffers (north_star: "cost volume,
aggregated costs and integer WTA disparities must be bit-exact").

`rpd_match_pair_dump_ex` runs the pipeline's own match_pair kernels — the
pixel-major u8 cost kernel (k_cost_px) that also generates the right-reference
volume swap_reference(C) (sgm.cpp:112-121) from the census words,
k_aggregate_tma for all 2P paths, the exact u16 path sums — and materialises
them in the reference float layout (v*W+u)*(d_max+1)+d.  They are compared
with the literal reference build (oracle/_ref: census_cost_volume,
swap_reference, aggregate_costs, select_disparity of the untouched
sgm.cpp:38-153) and the restated oracle, at the BASELINE configurations'
pass geometries: the half-resolution bootstrap pass (flat model,
L = (D+1)/2 + 1 = 33 / 65 / 129) and the full-resolution perspective-transformed
pass (the scene's road model, L = d_max_pt + 1 = 17), on row bands of the
configs' own scenes at their full widths.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2012_10802_b200.api import AGG_KERNELS, model
from paper_2012_10802_b200.synth import PIPELINE, make_scene, pipeline_config

pytestmark = pytest.mark.gpu

KEYS = ("cost", "cost_right", "agg_left", "agg_right", "disp_left", "disp_right")


def half(img):
    h, w = img.shape[0] // 2, img.shape[1] // 2
    x = img[:2 * h, :2 * w].astype(np.float32)
    # pipeline.cpp:30-31 order: ((a + b) + c) + d, times 0.25f
    return np.float32(0.25) * (((x[0::2, 0::2] + x[0::2, 1::2]) + x[1::2, 0::2]) + x[1::2, 1::2])


def band(img, rows, v0):
    return np.ascontiguousarray(img[v0:v0 + rows])


def road_model_of(cfg_id):
    """A perspective model in the config's disparity range: the PT pass of
    the pipeline uses the coarse fit; any model exercises the same kernels."""
    sc = make_scene(cfg_id, 0)
    p = sc.params
    return sc, model(p["d_min"] + 2.0, (p["d_max"] - p["d_min"]) / sc.left.shape[0],
                     p["phi"])


def assert_dump_equal(a, b, what):
    for k in KEYS:
        x, y = a[k], b[k]
        mism = x.view(np.uint32) != y.view(np.uint32)
        assert not mism.any(), f"{what}: {k}: {int(mism.sum())} cells differ, first at " \
                               f"{np.argwhere(mism)[0].tolist()}"


def checker(request):
    """The literal reference where built (it travels with the snapshot), else
    the restated oracle (which the CPU suite pins to the literal build)."""
    try:
        return request.getfixturevalue("ref")
    except pytest.skip.Exception:
        return request.getfixturevalue("oracle")


CASES = [
    # (config, pass, rows)
    (1, "boot", 60), (1, "pt", 64),
    (2, "boot", 24), (2, "pt", 40),
    (3, "boot", 20), (3, "pt", 32),
    (4, "boot", 12), (4, "pt", 24),
]


@pytest.mark.parametrize("case", CASES, ids=[f"cfg{c}-{p}" for c, p, _ in CASES])
def test_production_sgm_buffers_bit_exact(gpu, request, case):
    cfg_id, pas, rows = case
    chk = checker(request)
    sc, m = road_model_of(cfg_id)
    cfg_g = pipeline_config(gpu.lib, cfg_id)
    cfg_c = pipeline_config(chk.lib, cfg_id)
    if cfg_id == 1 and chk.lib.path.endswith("librpd_ref.so"):
        pass  # the literal wrapper composes the reference stages for 4 paths
    left, right = sc.left.astype(np.float32), sc.right.astype(np.float32)
    if pas == "boot":
        left, right = half(left), half(right)
        d_max = (PIPELINE[cfg_id]["d_max"] + 1) // 2
        m = model()
    else:
        d_max = cfg_g.d_max_pt
    v0 = (left.shape[0] - rows) // 2
    left, right = band(left, rows, v0), band(right, rows, v0)
    a = gpu.match_pair_dump_ex(left, right, m, cfg_g, d_max)
    assert AGG_KERNELS[gpu.stats().last_agg_kernel] == "u8_tma"
    b = chk.match_pair_dump_ex(left, right, m, cfg_c, d_max)
    assert_dump_equal(a, b, f"cfg{cfg_id} {pas}")
    # the production match_pair (bulk WTA, not the dump WTA) agrees as well
    d0g, d1g, _ = gpu.match_pair(left, right, m, cfg_g, d_max)
    d0c, d1c, _ = chk.match_pair(left, right, m, cfg_c, d_max)
    assert np.array_equal(d0g.view(np.uint32), d0c.view(np.uint32))
    assert np.array_equal(d1g.view(np.uint32), d1c.view(np.uint32))


@pytest.mark.parametrize("paths", [4, 8])
@pytest.mark.parametrize("levels", [1, 5, 17, 33, 40, 65, 100, 129, 144, 200, 257])
def test_production_buffers_all_level_layouts(gpu, oracle, lib, paths, levels):
    """Every u8 layout the fast path picks (G = 1, 2, 4, 8 lanes per chain,
    padded level words) on a ragged raster, with a perspective model so
    out-of-view samples and the right-reference overrides are exercised."""
    h, w = 21, max(levels + 9, 37)
    rng = np.random.default_rng(levels * 10 + paths)
    left = rng.integers(0, 256, (h, w)).astype(np.float32)
    right = np.roll(left, 3, axis=1) + rng.normal(0, 2, (h, w)).astype(np.float32)
    right = np.clip(np.rint(right), 0, 255).astype(np.float32)
    m = model(4.0, 0.05, 0.02)
    cfg = lib.default_config(lambda1=10.0, lambda2=120.0, sgm_paths=paths)
    a = gpu.match_pair_dump_ex(left, right, m, cfg, levels - 1)
    kernel = AGG_KERNELS[gpu.stats().last_agg_kernel]
    assert kernel in ("u8_tma", "u8")
    b = oracle.match_pair_dump_ex(left, right, m, oracle.lib.default_config(
        lambda1=10.0, lambda2=120.0, sgm_paths=paths), levels - 1)
    assert_dump_equal(a, b, f"L={levels} P={paths} ({kernel})")

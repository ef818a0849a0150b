"""GPU vs oracle parity for the SGM stage (bit-exact).

Covers every level layout of the fast path (G = 1, 2, 4, 8 lanes per chain),
both path counts, all census windows, the generic float path (non-integral
penalties), perspective-transformed passes with out-of-view samples, and
ragged / tiny images.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2012_10802_b200.api import model

pytestmark = pytest.mark.gpu


def stereo_pair(h, w, seed, a0=6.0, a1=0.03, phi=0.01, noise=2.0):
    """Left: uniform texture.  Right: left sampled at u + d(u, v) (planar road)."""
    rng = np.random.default_rng(seed)
    left = rng.integers(0, 256, size=(h, w)).astype(np.float64)
    vv, uu = np.meshgrid(np.arange(h), np.arange(w), indexing="ij")
    d = a0 + a1 * (vv * math.cos(phi) - uu * math.sin(phi))
    x = np.clip(uu + d, 0, w - 1)
    x0 = np.floor(x).astype(int)
    x1 = np.minimum(x0 + 1, w - 1)
    t = x - x0
    right = (1 - t) * left[vv, x0] + t * left[vv, x1]
    right = right + rng.normal(0, noise, size=right.shape)
    return (np.clip(np.rint(left), 0, 255).astype(np.float32),
            np.clip(np.rint(right), 0, 255).astype(np.float32))


def assert_bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    mism = a.view(np.uint32 if a.dtype == np.float32 else np.uint64) != \
        b.view(np.uint32 if b.dtype == np.float32 else np.uint64)
    if mism.any():
        idx = np.argwhere(mism)[:5]
        raise AssertionError(f"{int(mism.sum())} mismatches, first at {idx.tolist()}: "
                             f"{a[tuple(idx[0])]} vs {b[tuple(idx[0])]}")


@pytest.mark.parametrize("window", [3, 5, 7])
def test_census_cost_volume_bit_exact(gpu, oracle, window):
    left, right = stereo_pair(37, 83, 1)
    iv = (np.random.default_rng(2).random((37, 83)) < 0.9).astype(np.uint8)
    for in_view in (None, iv):
        a = gpu.census_cost_volume(left, right, 20, window, in_view)
        b = oracle.census_cost_volume(left, right, 20, window, in_view)
        assert_bits_equal(a, b)


@pytest.mark.parametrize("d_max", [0, 5, 16, 35, 40, 64, 100, 128])
@pytest.mark.parametrize("paths", [4, 8])
def test_match_pair_flat_model_levels(gpu, oracle, lib, d_max, paths):
    h, w = 41, 140
    left, right = stereo_pair(h, w, 10 + d_max, a0=d_max * 0.4 + 1, a1=0.0, phi=0.0)
    cfg = lib.default_config(lambda1=10.0, lambda2=120.0, sgm_paths=paths)
    a = gpu.match_pair(left, right, model(), cfg, d_max)
    b = oracle.match_pair(left, right, model(), cfg, d_max)
    for x, y in zip(a, b):
        assert_bits_equal(x, y)
    assert (a[0] != -1).mean() > 0.3 or d_max == 0


def test_match_pair_d_max_256(gpu, oracle, lib):
    left, right = stereo_pair(24, 300, 7, a0=40.0, a1=0.0, phi=0.0)
    cfg = lib.default_config(lambda1=10.0, lambda2=120.0)
    for x, y in zip(gpu.match_pair(left, right, model(), cfg, 256),
                    oracle.match_pair(left, right, model(), cfg, 256)):
        assert_bits_equal(x, y)


@pytest.mark.parametrize("window", [3, 5, 7])
def test_match_pair_perspective_model(gpu, oracle, lib, window):
    h, w = 64, 120
    left, right = stereo_pair(h, w, 3, a0=12.0, a1=0.08, phi=0.03)
    m = model(11.0, 0.08, 0.03)
    cfg = lib.default_config(census_window=window)
    a = gpu.match_pair(left, right, m, cfg, 16)
    b = oracle.match_pair(left, right, m, cfg, 16)
    for x, y in zip(a, b):
        assert_bits_equal(x, y)


def test_match_pair_generic_float_penalties(gpu, oracle, lib):
    left, right = stereo_pair(30, 70, 5)
    for l1, l2 in ((8.5, 32.25), (7.0, 400.0), (1e-3, 2e-3)):
        cfg = lib.default_config(lambda1=l1, lambda2=l2)
        a = gpu.match_pair(left, right, model(5.0, 0.02, 0.0), cfg, 12)
        b = oracle.match_pair(left, right, model(5.0, 0.02, 0.0), cfg, 12)
        for x, y in zip(a, b):
            assert_bits_equal(x, y)


@pytest.mark.parametrize("shape", [(1, 2), (2, 3), (5, 9), (64, 2), (3, 200)])
def test_match_pair_ragged_shapes(gpu, oracle, lib, shape):
    h, w = shape
    rng = np.random.default_rng(h * 1000 + w)
    left = rng.integers(0, 256, size=shape).astype(np.float32)
    right = rng.integers(0, 256, size=shape).astype(np.float32)
    cfg = lib.default_config()
    d_max = min(w - 1, 8)
    for x, y in zip(gpu.match_pair(left, right, model(1.0, 0.0, 0.0), cfg, d_max),
                    oracle.match_pair(left, right, model(1.0, 0.0, 0.0), cfg, d_max)):
        assert_bits_equal(x, y)


def test_aggregate_generic_random(gpu, oracle):
    rng = np.random.default_rng(8)
    vol = rng.uniform(0, 50, size=(13, 17, 9)).astype(np.float32)
    dirs = [(1, 0), (0, 1), (2, 1), (-1, -3)]
    assert_bits_equal(gpu.aggregate_costs(vol, 3.5, 11.25, dirs),
                      oracle.aggregate_costs(vol, 3.5, 11.25, dirs))
    assert_bits_equal(gpu.swap_reference(vol), oracle.swap_reference(vol))
    agg = oracle.aggregate_costs(vol, 3.5, 11.25)
    assert_bits_equal(gpu.select_disparity(agg), oracle.select_disparity(agg))


def test_consistency_filter(gpu, oracle):
    rng = np.random.default_rng(9)
    l = rng.uniform(0, 10, (20, 30)).astype(np.float32)
    r = rng.uniform(0, 10, (20, 30)).astype(np.float32)
    l[rng.random(l.shape) < 0.2] = -1
    r[rng.random(r.shape) < 0.2] = -1
    assert_bits_equal(gpu.consistency_filter(l, r, 1.0), oracle.consistency_filter(l, r, 1.0))


def test_match_pair_large_frame(gpu, oracle, lib):
    """A BASELINE-shaped PT pass (800x1312, L=17, P=8) on a 200-row band."""
    left, right = stereo_pair(200, 1312, 99, a0=30.0, a1=0.05, phi=0.05)
    m = model(28.0, 0.05, 0.05)
    cfg = lib.default_config(lambda1=10.0, lambda2=120.0)
    for x, y in zip(gpu.match_pair(left, right, m, cfg, 16),
                    oracle.match_pair(left, right, m, cfg, 16)):
        assert_bits_equal(x, y)

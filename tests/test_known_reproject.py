"""Known answers of the reference 3-D reprojection tests (SURVEY.md §8(f)
row 2), both implementations: test_road_geometry.cpp:209-266 restated."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2012_10802_b200.api import InvalidArgument, StereoRig
from paper_2012_10802_b200.ply import load_ply, save_ply

INV = -1.0


def rig():
    return StereoRig(700.0, 0.12, 320.0, 240.0)


def test_reproject(ctx):
    d = np.full((2, 2), INV, np.float32)
    d[0, 0] = 7.0
    cloud = ctx.reproject(d, rig())
    assert cloud.shape == (1, 3)
    assert cloud[0, 2] == pytest.approx(12.0)
    centre = np.full((481, 641), INV, np.float32)
    centre[240, 320] = 7.0
    on_axis = ctx.reproject(centre, rig())
    assert on_axis.shape == (1, 3)
    assert on_axis[0, 0] == pytest.approx(0.0) and on_axis[0, 1] == pytest.approx(0.0)
    assert ctx.reproject(np.zeros((2, 2), np.float32), rig()).shape == (0, 3)
    with pytest.raises(InvalidArgument):
        ctx.reproject(d, StereoRig(0.0, 0.12, 0.0, 0.0))


def test_reproject_masked_and_instances(ctx):
    rng = np.random.default_rng(5)
    d = rng.uniform(-1.0, 60.0, (40, 50)).astype(np.float32)
    d[rng.random((40, 50)) < 0.2] = INV
    lab = rng.integers(0, 4, (40, 50)).astype(np.int32)
    r = rig()
    parts = ctx.reproject_instances(d, lab, 3, r)
    for k in (1, 2, 3):
        m = ctx.reproject(d, r, labels=lab, label=k)
        assert np.array_equal(m, parts[k - 1])
        dm = np.where(lab == k, d, INV).astype(np.float32)
        assert np.array_equal(m, ctx.reproject(dm, r))


def test_closest_distance_error(ctx):
    a = np.array([[0, 0, 1]], np.float32)
    assert ctx.closest_distance_error(a, a) == pytest.approx(0.0)
    b = np.array([[0, 0, 1.002]], np.float32)
    assert ctx.closest_distance_error(b, a) == pytest.approx(0.002, rel=1e-4)
    rng = np.random.default_rng(31)
    truth = rng.uniform(-1.0, 1.0, (100, 3)).astype(np.float32)
    truth[:, 2] += 2.0
    test = truth.copy()
    test[:, 0] += np.float32(0.003)
    e = ctx.closest_distance_error(test, truth)
    assert e <= 0.003 + 1e-6
    t64, g64 = test.astype(np.float64), truth.astype(np.float64)
    best = ((t64[:, None, :] - g64[None, :, :]) ** 2).sum(-1).min(1)
    assert e == pytest.approx(math.sqrt(best.sum() / len(test)), rel=1e-12)
    with pytest.raises(InvalidArgument):
        ctx.closest_distance_error(np.zeros((0, 3), np.float32), a)


def test_ply_round_trip(tmp_path):
    cloud = np.array([[1.5, -2.25, 3.0], [0.0, 0.5, 9.75]], np.float32)
    path = tmp_path / "rpd_test_cloud.ply"
    save_ply(cloud, path)
    back = load_ply(path)
    assert back.shape == (2, 3)
    assert back[1, 2] == pytest.approx(9.75)
    assert path.read_text().startswith("ply\nformat ascii 1.0\nelement vertex 2\n")

"""Known answers of the reference perspective and road-geometry suites.

Ports /root/reference/proj/tests/test_perspective.cpp and
test_road_geometry.cpp (the Eigen colPivHouseholderQr oracle of :35-44 is
restated as a long-double-free numpy lstsq; acceptance.cpp:123-175 roll checks).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2012_10802_b200.api import DegenerateError, InvalidArgument, RectRoi, model

DEG = math.pi / 180.0


def road_at(m, u, v):
    return m.a0 + m.a1 * (v * math.cos(m.phi) - u * math.sin(m.phi))


# ------------------------------------------------------------- perspective --
def test_row_shifts_zero_roll_x_independent(ctx):
    t = ctx.compute_row_shifts(model(10.0, 0.5, 0.0), 320, 6, 0.0)
    assert t == pytest.approx([10.0 + 0.5 * v for v in range(6)])


def test_row_shifts_endpoint_minimum_under_roll(ctx):
    t = ctx.compute_row_shifts(model(10.0, 0.5, math.asin(0.1)), 100, 1, 0.0)
    assert t[0] == pytest.approx(10.0 - 0.5 * 100.0 * 0.1)


def test_row_shifts_clamp_at_zero(ctx):
    t = ctx.compute_row_shifts(model(2.0, 0.01, 0.0), 100, 1, 5.0)
    assert t[0] == 0.0


def test_row_shifts_width_error(ctx):
    with pytest.raises(InvalidArgument):
        ctx.compute_row_shifts(model(), 1, 4, 0.0)


def test_warp_zero_shift_identity(ctx):
    img = np.array([[1, 2, 3, 4], [5, 6, 7, 8]], np.float32)
    out, iv = ctx.warp_right_image(img, [0.0, 0.0])
    assert np.array_equal(out, img)
    assert np.all(iv == 1)


def test_warp_integer_and_fractional(ctx):
    img = np.array([[10, 20, 30, 40]], np.float32)
    w1, iv1 = ctx.warp_right_image(img, [1.0])
    assert w1[0, 0] == 0.0 and iv1[0, 0] == 0
    assert list(w1[0, 1:]) == [10.0, 20.0, 30.0]
    w2, iv2 = ctx.warp_right_image(img, [0.5])
    assert iv2[0, 0] == 0
    assert list(w2[0, 1:]) == pytest.approx([15.0, 25.0, 35.0])


def test_restore_adds_shift_keeps_invalid(ctx):
    d0 = np.full((2, 3), 3.0, np.float32)
    d0[1, 2] = -1.0
    d1 = ctx.restore_disparity(d0, [7.0, 7.0])
    assert d1[0, 0] == 10.0 and d1[1, 0] == 10.0 and d1[1, 2] == -1.0


def test_dimension_mismatch_rejected(ctx):
    img = np.zeros((3, 4), np.float32)
    with pytest.raises(InvalidArgument):
        ctx.warp_right_image(img, [0.0, 0.0])
    with pytest.raises(InvalidArgument):
        ctx.restore_disparity(img, [0.0])


def test_planar_scene_property(ctx):
    m = model(12.0, 0.2, 0.01)
    w, h, dpt = 64, 32, 5.0
    t = ctx.compute_row_shifts(m, w, h, dpt)
    uu, vv = np.meshgrid(np.arange(w), np.arange(h))
    truth = m.a0 + m.a1 * (vv * math.cos(m.phi) - uu * math.sin(m.phi))
    resid = truth - t[:, None]
    assert np.all(resid >= dpt - 1e-9)
    assert np.all(resid <= dpt + abs(m.a1 * math.sin(m.phi)) * w + 1e-9)
    d0 = (truth - t[:, None]).astype(np.float32)
    d1 = ctx.restore_disparity(d0, t)
    assert d1 == pytest.approx(truth, rel=1e-5)


# ------------------------------------------------------------ road geometry --
def synth_obs(m, k, sigma, seed, width=640, height=480):
    rng = np.random.default_rng(seed)
    u = rng.uniform(0.0, width - 1.0, k)
    v = rng.uniform(0.0, height - 1.0, k)
    d = m.a0 + m.a1 * (v * math.cos(m.phi) - u * math.sin(m.phi))
    if sigma > 0:
        d = d + rng.normal(0.0, sigma, k)
    return d, u, v


def dense_oracle(d, u, v, phi):
    T = np.stack([np.ones_like(u), math.cos(phi) * v - math.sin(phi) * u], axis=1)
    a, *_ = np.linalg.lstsq(T, d, rcond=None)
    return a[0], a[1], float(np.sum((d - T @ a) ** 2))


def test_fit_line_exact_lines(ctx):
    u = 10.0 * np.arange(5)
    v = 40.0 * np.arange(5)
    f = ctx.fit_line(5.0 + 0.1 * v, u, v, 0.0)
    assert f.model.a0 == pytest.approx(5.0)
    assert f.model.a1 == pytest.approx(0.1)
    assert abs(f.e0min) <= 1e-12
    flat = ctx.fit_line(np.full(5, 7.0), u, v, 0.0)
    assert flat.model.a0 == pytest.approx(7.0)
    assert abs(flat.model.a1) <= 1e-12


def test_fit_line_matches_dense_oracle(ctx):
    d, u, v = synth_obs(model(20.0, 0.15, 0.03), 50, 0.3, 5)
    f = ctx.fit_line(d, u, v, 0.03)
    a0, a1, e = dense_oracle(d, u, v, 0.03)
    assert f.model.a0 == pytest.approx(a0, rel=1e-9)
    assert f.model.a1 == pytest.approx(a1, rel=1e-9)
    assert f.e0min == pytest.approx(e, rel=1e-9)


def test_fit_line_residual_direct(ctx):
    d, u, v = synth_obs(model(8.0, 0.09, -0.02), 300, 0.25, 9)
    f = ctx.fit_line(d, u, v, -0.015)
    r = d - (f.model.a0 + f.model.a1 * (v * math.cos(f.model.phi) - u * math.sin(f.model.phi)))
    assert f.e0min == pytest.approx(float(np.sum(r * r)), rel=1e-9)


def test_e0min_offset_invariance(ctx):
    d, u, v = synth_obs(model(8.0, 0.09, 0.01), 200, 0.2, 13)
    base = ctx.fit_line(d, u, v, 0.01)
    sh = ctx.fit_line(d + 3.5, u, v, 0.01)
    assert sh.model.a0 == pytest.approx(base.model.a0 + 3.5, rel=1e-9)
    assert sh.model.a1 == pytest.approx(base.model.a1, rel=1e-9)
    assert sh.e0min == pytest.approx(base.e0min, rel=1e-6)


def test_fit_line_degenerate(ctx):
    with pytest.raises(DegenerateError):
        ctx.fit_line(np.full(4, 3.0), np.full(4, 10.0), np.full(4, 20.0), 0.0)
    with pytest.raises(InvalidArgument):
        ctx.fit_line(np.zeros(2), np.zeros(2), np.zeros(2), 0.0)


def grid_phi(ctx, d, u, v, lo, hi, step):
    best_phi, best_e = lo, math.inf
    phi = lo
    while phi <= hi:
        e = ctx.fit_line(d, u, v, phi).e0min
        if e < best_e:
            best_e, best_phi = e, phi
        phi += step
    return best_phi


def test_estimate_roll_zero_noiseless(ctx):
    d, u, v = synth_obs(model(20.0, 0.3, 0.0), 2000, 0.0, 17)
    m = ctx.estimate_roll(d, u, v, -15 * DEG, 15 * DEG, 1e-4)
    assert abs(m.phi) <= 1e-4


def test_estimate_roll_two_degrees(ctx):
    d, u, v = synth_obs(model(20.0, 0.3, 2.0 * DEG), 2000, 0.0, 19)
    m = ctx.estimate_roll(d, u, v, -15 * DEG, 15 * DEG, 1e-4)
    assert abs(m.phi - 2.0 * DEG) <= 0.01 * DEG
    assert abs(m.phi - grid_phi(ctx, d, u, v, 1.9 * DEG, 2.1 * DEG, 0.001 * DEG)) <= 0.01 * DEG


def test_estimate_roll_minus_three_noisy(ctx):
    d, u, v = synth_obs(model(20.0, 0.3, -3.0 * DEG), 10000, 0.1, 23)
    m = ctx.estimate_roll(d, u, v, -15 * DEG, 15 * DEG, 1e-4)
    assert abs(m.phi - (-3.0 * DEG)) <= 0.1 * DEG


@pytest.mark.parametrize("deg", [-5.0, -2.0, 0.0, 2.0, 5.0])
def test_acceptance_roll_recovery(ctx, deg):
    """acceptance.cpp:162-175: roll within 0.01 deg noiseless."""
    d, u, v = synth_obs(model(6.0, 0.08, deg * DEG), 5000, 0.0, 400 + int(deg * 10))
    m = ctx.estimate_roll(d, u, v, -15 * DEG, 15 * DEG, 1e-4)
    assert abs(m.phi - deg * DEG) <= 0.01 * DEG


def test_estimate_roll_tol_error(ctx):
    d, u, v = synth_obs(model(20.0, 0.3, 0.0), 100, 0.0, 3)
    with pytest.raises(InvalidArgument):
        ctx.estimate_roll(d, u, v, -0.1, 0.1, 0.0)


def test_fit_road_trims_outliers(ctx):
    truth = model(18.0, 0.12, 0.01)
    d, u, v = synth_obs(truth, 4000, 0.05, 29)
    d[:300] -= 3.0
    f = ctx.fit_road(d, u, v, 15 * DEG, 1e-4)
    assert f.used < 4000
    assert f.model.a0 == pytest.approx(truth.a0, rel=0.02)
    assert f.model.a1 == pytest.approx(truth.a1, rel=0.02)


def test_sample_observations_counts_and_caps(ctx):
    full = np.full((10, 10), 4.0, np.float32)
    assert ctx.sample_observations(full)[0].shape[0] == 100
    sparse = np.full((10, 10), -1.0, np.float32)
    sparse[0, 0] = 1.0
    sparse[5, 5] = 2.0
    with pytest.raises(DegenerateError):
        ctx.sample_observations(sparse)
    big = np.full((1000, 1000), 4.0, np.float32)
    assert ctx.sample_observations(big)[0].shape[0] == 100000


def test_sample_observations_stride_and_roi(ctx):
    rng = np.random.default_rng(5)
    d1 = rng.uniform(1, 40, (50, 70)).astype(np.float32)
    d1[rng.random((50, 70)) < 0.3] = -1.0
    d, u, v = ctx.sample_observations(d1, cap=777)
    vv, uu = np.nonzero(d1 != -1.0)
    n = vv.shape[0]
    idx = (np.arange(777, dtype=np.int64) * n) // 777
    assert np.array_equal(u, uu[idx]) and np.array_equal(v, vv[idx])
    assert np.array_equal(d, d1[vv[idx], uu[idx]].astype(np.float64))
    d, u, v = ctx.sample_observations(d1, roi=RectRoi(10, 5, 20, 100))
    assert np.all((u >= 10) & (u < 30) & (v >= 5))


def test_transform_disparity(ctx):
    m = model(10.0, 0.1, 0.02)
    uu, vv = np.meshgrid(np.arange(30), np.arange(20))
    d1 = (m.a0 + m.a1 * (vv * math.cos(m.phi) - uu * math.sin(m.phi))).astype(np.float32)
    d2, clamped = ctx.transform_disparity(d1, m, 30.0)
    assert d2 == pytest.approx(np.full_like(d2, 30.0), rel=1e-5)
    assert clamped == 0
    p = d1.copy()
    p[5, 5] -= 2.0
    d2p, _ = ctx.transform_disparity(p, m, 30.0)
    assert d2p[5, 5] == pytest.approx(28.0, rel=1e-5)
    q = d1.copy()
    q[0, 0] = -1.0
    q[1, 1] = 0.0
    d2q, cq = ctx.transform_disparity(q, m, 5.0)
    assert d2q[0, 0] == -1.0 and d2q[1, 1] == 0.0 and cq >= 1
    back = d2.astype(np.float64) + (m.a0 + m.a1 * (vv * math.cos(m.phi) - uu * math.sin(m.phi))) - 30.0
    assert back == pytest.approx(d1.astype(np.float64), rel=1e-5)

"""Known answers of the reference scene-generator suite,
both implementations.

Restates the cases of /root/reference/proj/tests/test_synth.cpp (plane truth,
paraboloid dip, determinism, right-view shift, road fit on the truth, invalid
specs, scene_batch ranges, scene-directory round trip), plus the CPU check of
the device random streams against libstdc++ (tests/cpp/synth_rng_check.cpp).
"""
from __future__ import annotations

import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2012_10802_b200.api import DegenerateError, InvalidArgument, RoadModel
from paper_2012_10802_b200.scenes import (BatchRanges, PotholeSpec, SceneSpec, generate_scene,
                                          load_scene, scene_batch, write_scene)

ROOT = Path(__file__).resolve().parents[1]


def small_spec(**kw) -> SceneSpec:
    s = SceneSpec(width=160, height=120, a0=5.0, a1=0.08, phi_true=0.0, texture_seed=42)
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def plane(a0, a1, phi, u, v):
    return a0 + a1 * (v * math.cos(phi) - u * math.sin(phi))


def test_device_random_streams_match_libstdcxx(tmp_path):
    """mt19937 rounds, uniform_real_distribution<float>, normal_distribution<double>
    and the double-double log of synth_rng.cuh against <random> / glibc."""
    exe = tmp_path / "synth_rng_check"
    subprocess.run(["g++", "-O2", "-std=c++17", str(ROOT / "tests" / "cpp" / "synth_rng_check.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")


def test_plane_truth_without_potholes(ctx):
    """test_synth.cpp:28-44."""
    spec = small_spec(phi_true=0.02)
    sc = generate_scene(ctx, spec)
    assert sc.left.shape == (120, 160) and sc.right.shape == (120, 160)
    assert not sc.gt_mask.any()
    for v in range(0, 120, 7):
        for u in range(0, 160, 11):
            want = plane(5.0, 0.08, 0.02, u, v)
            assert sc.gt_disparity[v, u] == pytest.approx(want, rel=1e-6)
    assert sc.left.max() - sc.left.min() > 50.0
    assert sc.left.min() >= 0.0 and sc.left.max() <= 255.0


def test_pothole_dip_is_a_paraboloid(ctx):
    """test_synth.cpp:46-61."""
    spec = small_spec(potholes=[PotholeSpec(80.0, 60.0, 18.0, 12.0, 3.0)])
    sc = generate_scene(ctx, spec)
    assert sc.gt_disparity[60, 80] == pytest.approx(plane(5.0, 0.08, 0.0, 80, 60) - 3.0, rel=1e-6)
    assert sc.gt_mask[60, 80] == 1
    assert sc.gt_mask[60, 100] == 0
    assert sc.gt_mask[73, 80] == 0
    assert sc.gt_disparity[60, 89] == pytest.approx(plane(5.0, 0.08, 0.0, 89, 60) - 3.0 * 0.75,
                                                    rel=1e-6)


def test_same_spec_same_scene(ctx):
    """test_synth.cpp:63-77."""
    spec = small_spec(potholes=[PotholeSpec(60.0, 70.0, 15.0, 15.0, 2.5)])
    a, b = generate_scene(ctx, spec), generate_scene(ctx, spec)
    for x, y in ((a.left, b.left), (a.right, b.right), (a.gt_disparity, b.gt_disparity),
                 (a.gt_mask, b.gt_mask)):
        assert np.array_equal(x, y)
    other = small_spec(potholes=spec.potholes, texture_seed=43)
    assert not np.array_equal(generate_scene(ctx, other).left, a.left)


def test_right_view_is_left_shifted(ctx):
    """test_synth.cpp:79-88: constant integer disparity 6."""
    sc = generate_scene(ctx, small_spec(a0=6.0, a1=0.0))
    for v in range(0, 120, 5):
        for u in range(0, 160 - 6, 3):
            assert sc.right[v, u] == pytest.approx(sc.left[v, u + 6], rel=1e-6)


def test_road_fit_on_truth_recovers_the_line(ctx):
    """test_synth.cpp:90-115."""
    spec = small_spec(phi_true=-0.03, potholes=[PotholeSpec(80.0, 60.0, 20.0, 14.0, 3.0)])
    sc = generate_scene(ctx, spec)
    road = sc.gt_disparity.copy()
    road[sc.gt_mask != 0] = -1.0
    d, u, v = ctx.sample_observations(road)
    m = ctx.estimate_roll(d, u, v, -0.26, 0.26, 1e-5)
    assert m.phi == pytest.approx(-0.03, rel=1e-3)
    assert m.a0 == pytest.approx(5.0, rel=1e-3)
    assert m.a1 == pytest.approx(0.08, rel=1e-3)
    d2, _ = ctx.transform_disparity(sc.gt_disparity, RoadModel(5.0, 0.08, -0.03), 30.0)
    for vv in range(0, 120, 4):
        for uu in range(0, 160, 4):
            if sc.gt_mask[vv, uu]:
                assert d2[vv, uu] < 30.0
            else:
                assert d2[vv, uu] == pytest.approx(30.0, rel=1e-5)


def test_invalid_specs_are_rejected(ctx):
    """test_synth.cpp:117-129."""
    with pytest.raises(DegenerateError):
        generate_scene(ctx, small_spec(a0=-80.0))
    with pytest.raises(InvalidArgument):
        generate_scene(ctx, small_spec(potholes=[PotholeSpec(80.0, 60.0, -5.0, 10.0, 2.0)]))
    with pytest.raises(DegenerateError):
        generate_scene(ctx, small_spec(potholes=[PotholeSpec(80.0, 10.0, 15.0, 15.0, 50.0)]))
    with pytest.raises(InvalidArgument):
        generate_scene(ctx, small_spec(width=0))


def test_scene_batch_ranges_and_determinism(ctx):
    """test_synth.cpp:131-156 (640 x 480 scenes)."""
    r = BatchRanges()
    batch = scene_batch(ctx, 4, 900, r)
    assert len(batch) == 4
    for sc in batch:
        assert 1 <= len(sc.spec.potholes) <= 3
        for p in sc.spec.potholes:
            assert p.cu - p.ru >= r.margin and p.cu + p.ru <= sc.spec.width - r.margin
            assert p.cv - p.rv >= r.margin and p.cv + p.rv <= sc.spec.height - r.margin
            assert r.depth_min <= p.depth <= r.depth_max
        assert abs(sc.spec.phi_true) <= r.phi_abs_max + 1e-12
        assert sc.spec.rig.cu == 320.0 and sc.spec.rig.cv == 240.0
    again = scene_batch(ctx, 4, 900, r)
    for a, b in zip(batch, again):
        assert np.array_equal(a.left, b.left)
        assert np.array_equal(a.gt_disparity, b.gt_disparity)
    other = scene_batch(ctx, 1, 901, r)
    assert not np.array_equal(other[0].gt_disparity, batch[0].gt_disparity)


def test_write_load_scene_round_trip(ctx, tmp_path):
    """test_synth.cpp:158-189."""
    spec = small_spec(phi_true=0.015, potholes=[PotholeSpec(70.0, 64.0, 16.0, 11.0, 2.25)])
    sc = generate_scene(ctx, spec)
    d = tmp_path / "scene_000"
    write_scene(sc, d, ctx)
    for name in ("left.png", "right.png", "disp_gt.png", "mask_gt.png", "spec.txt"):
        assert (d / name).exists()
    back = load_scene(d, ctx)
    # 8-bit storage rounds half away from zero (std::round)
    assert np.array_equal(back.left, np.floor(sc.left + 0.5).astype(np.float32))
    assert np.array_equal(back.gt_mask, sc.gt_mask)
    assert back.spec.a0 == pytest.approx(spec.a0)
    assert back.spec.a1 == pytest.approx(spec.a1)
    assert back.spec.phi_true == pytest.approx(0.015)
    assert len(back.spec.potholes) == 1
    assert back.spec.potholes[0].depth == pytest.approx(2.25)
    assert np.abs(back.gt_disparity[::9, ::9] - sc.gt_disparity[::9, ::9]).max() <= 1.0 / 256.0

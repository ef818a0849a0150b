"""3-D reprojection: device vs oracle.  Points are
bit-identical (same double expression order, same scan order); the cloud
error differs only by the oracle's sequential double summation of the
per-point minima (the device's double-double sum is the more accurate one;
up to ~n ulp apart: 1e-10 relative)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2012_10802_b200.synth import make_scene, pipeline_config

pytestmark = pytest.mark.gpu


def test_pipeline_pothole_clouds_match_oracle(gpu, oracle, cuda_lib):
    """rpd_cli detect's per-pothole clouds (rpd_cli.cpp:96-104) on a frame."""
    sc = make_scene(2, 0)
    cfg = pipeline_config(cuda_lib, 2)
    res = gpu.detect(sc.left, sc.right, cfg)
    h, w = res.d1.shape
    rig = gpu.rig_from_config(cfg, w, h)
    assert (rig.cu, rig.cv) == (w / 2.0, h / 2.0)
    n = int(res.labels.max())
    ga = gpu.reproject_instances(res.d1, res.labels, n, rig)
    oa = oracle.reproject_instances(res.d1, res.labels, n, rig)
    assert len(ga) == len(oa) == n
    for a, b in zip(ga, oa):
        assert a.tobytes() == b.tobytes()
    full_g, full_o = gpu.reproject(res.d1, rig), oracle.reproject(res.d1, rig)
    assert full_g.tobytes() == full_o.tobytes()
    # cloud error of the noisy reprojection against the ground-truth one
    truth = gpu.reproject(sc.gt_disparity.astype(np.float32), rig)
    test = full_g[::97]
    e_g = gpu.closest_distance_error(test, truth[::13])
    e_o = oracle.closest_distance_error(test, truth[::13])
    assert abs(e_g - e_o) <= 1e-10 * e_o


@pytest.mark.parametrize("seed", [0, 1])
def test_closest_distance_error_matches_oracle(gpu, oracle, seed):
    rng = np.random.default_rng(900 + seed)
    truth = rng.normal(0.0, 3.0, (3000, 3)).astype(np.float32)
    test = (truth[rng.integers(0, 3000, 5000)] + rng.normal(0, 0.05, (5000, 3))).astype(np.float32)
    a, b = gpu.closest_distance_error(test, truth), oracle.closest_distance_error(test, truth)
    assert abs(a - b) <= 1e-10 * b

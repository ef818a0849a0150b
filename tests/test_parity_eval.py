"""Evaluation metrics: device vs oracle.

Counts are exact on both sides, so pep, the confusion counts and every
derived ratio, and the instance report are compared bit for bit.  rmse: the
device sums the squared errors in double-double (block partials in a fixed
order), the oracle sequentially in double as evaluation.hpp:35-40 does, so the
two differ by the oracle's rounding only (<= ~n ulp): 1e-10 relative.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2012_10802_b200.synth import make_scene, pipeline_config

pytestmark = pytest.mark.gpu


def blobs(rng, h, w, n):
    """Instance map of n random axis-aligned rectangles (later ids overwrite)."""
    m = np.zeros((h, w), np.int32)
    for i in range(1, n + 1):
        v0, u0 = rng.integers(0, h - 8), rng.integers(0, w - 8)
        m[v0:v0 + rng.integers(4, 60), u0:u0 + rng.integers(4, 90)] = i
    return m


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_disparity_metrics_match_oracle(gpu, oracle, seed):
    rng = np.random.default_rng(700 + seed)
    h, w = 800, 1312
    gt = rng.uniform(0.0, 120.0, (h, w)).astype(np.float32)
    est = (gt + rng.normal(0.0, 1.5, (h, w))).astype(np.float32)
    gt[rng.random((h, w)) < 0.1] = -1.0
    est[rng.random((h, w)) < 0.2] = -1.0
    for eps in (0.5, 1.0, 3.0):
        assert gpu.pep(est, gt, eps) == oracle.pep(est, gt, eps)
    a, b = gpu.rmse(est, gt), oracle.rmse(est, gt)
    assert abs(a - b) <= 1e-10 * b


@pytest.mark.parametrize("seed", [0, 1])
def test_label_metrics_match_oracle(gpu, oracle, seed):
    rng = np.random.default_rng(800 + seed)
    h, w = 480, 640
    pred, gt = blobs(rng, h, w, 25), blobs(rng, h, w, 18)
    a, b = gpu.pixel_metrics(pred, gt), oracle.pixel_metrics(pred, gt)
    assert bytes(a) == bytes(b)
    for iou in (0.1, 0.5, 0.9):
        ra, rb = gpu.instance_metrics(pred, gt, iou), oracle.instance_metrics(pred, gt, iou)
        assert (ra.correct, ra.incorrect, ra.misdetection) == \
               (rb.correct, rb.incorrect, rb.misdetection)


def test_pipeline_outputs_against_scene_truth(gpu, oracle, cuda_lib):
    """The metrics `bench`/acceptance compute (rpd_cli.cpp:130-165): d1 vs the
    scene's ground-truth disparity, labels vs its pothole instances."""
    sc = make_scene(2, 0)
    res = gpu.detect(sc.left, sc.right, pipeline_config(cuda_lib, 2))
    gt_d = sc.gt_disparity.astype(np.float32)
    assert gpu.pep(res.d1, gt_d, 3.0) == oracle.pep(res.d1, gt_d, 3.0)
    a, b = gpu.rmse(res.d1, gt_d), oracle.rmse(res.d1, gt_d)
    assert abs(a - b) <= 1e-10 * b
    pa, pb = gpu.pixel_metrics(res.labels, sc.gt_mask), oracle.pixel_metrics(res.labels, sc.gt_mask)
    assert bytes(pa) == bytes(pb)
    ia, ib = gpu.instance_metrics(res.labels, sc.gt_mask), oracle.instance_metrics(res.labels, sc.gt_mask)
    assert (ia.correct, ia.incorrect, ia.misdetection) == (ib.correct, ib.incorrect, ib.misdetection)


def test_image_io_transforms_match_oracle(gpu, oracle):
    """image_io.cpp per-pixel transforms, bit-exact."""
    rng = np.random.default_rng(42)
    h, w = 600, 800
    d = rng.uniform(0.0, 250.0, (h, w)).astype(np.float32)
    d[rng.random((h, w)) < 0.1] = -1.0
    assert np.array_equal(gpu.encode_disparity_u16(d), oracle.encode_disparity_u16(d))
    s = rng.integers(0, 65536, (h, w)).astype(np.uint16)
    assert gpu.decode_disparity_u16(s).tobytes() == oracle.decode_disparity_u16(s).tobytes()
    lab = rng.integers(0, 40, (h, w)).astype(np.int32)
    assert np.array_equal(gpu.encode_labels_u16(lab), oracle.encode_labels_u16(lab))
    img = rng.uniform(-20.0, 280.0, (h, w)).astype(np.float32)
    assert np.array_equal(gpu.encode_gray_u8(img), oracle.encode_gray_u8(img))
    rgb = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    assert gpu.gray_from_rgb8(rgb).tobytes() == oracle.gray_from_rgb8(rgb).tobytes()
    assert np.array_equal(gpu.overlay_rgb8(img, lab), oracle.overlay_rgb8(img, lab))

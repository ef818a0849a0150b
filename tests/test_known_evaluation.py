"""Known answers of the reference evaluation suite,
both implementations.

Restates the cases of /root/reference/proj/tests/test_evaluation.cpp
(pep, rmse, fscore, pixel_metrics, instance_metrics) with our own inputs for
the randomised properties.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2012_10802_b200.api import DegenerateError, InvalidArgument

INV = -1.0


def test_pep_strict_violations_over_valid_overlap(ctx):
    gt = np.full((2, 5), 10.0, np.float32)
    est = gt.copy()
    est[0, 0] = 13.5   # err 3.5
    est[0, 1] = 12.0   # err exactly 2: not a violation at eps = 2
    est[1, 0] = INV
    gt[1, 1] = INV
    assert ctx.pep(est, gt, 2.0) == pytest.approx(100.0 / 8.0)
    assert ctx.pep(est, gt, 3.0) == pytest.approx(100.0 / 8.0)
    assert ctx.pep(est, gt, 4.0) == pytest.approx(0.0)
    with pytest.raises(DegenerateError):
        ctx.pep(est, np.full((2, 5), INV, np.float32), 2.0)
    with pytest.raises(InvalidArgument):
        ctx.pep(est, np.ones((1, 1), np.float32), 2.0)


def test_rmse(ctx):
    gt = np.full((1, 4), 5.0, np.float32)
    est = np.array([[5.0, 8.0, 1.0, INV]], np.float32)
    assert ctx.rmse(est, gt) == pytest.approx(math.sqrt(25.0 / 3.0))  # errors 0, 3, -4
    assert ctx.rmse(gt, gt) == 0.0


def test_pep_monotone_rmse_dominates_mean_abs(ctx):
    rng = np.random.default_rng(3)
    gt = rng.uniform(5.0, 40.0, (12, 12)).astype(np.float32)
    est = (gt + rng.normal(0.0, 2.0, (12, 12))).astype(np.float32)
    prev = 100.0
    for eps in (0.5, 1.0, 2.0, 3.0):
        p = ctx.pep(est, gt, eps)
        assert p <= prev
        prev = p
    mean_abs = float(np.mean(np.abs(est.astype(np.float64) - gt)))
    assert ctx.rmse(est, gt) >= mean_abs - 1e-12


def test_fscore_harmonic_mean(ctx):
    assert ctx.fscore(0.8982, 0.8903) == pytest.approx(0.8942, rel=5e-4)
    assert ctx.fscore(1.0, 1.0) == 1.0
    assert ctx.fscore(0.0, 0.0) == 0.0
    assert ctx.fscore(0.0, 0.9) == 0.0


def test_pixel_metrics_hand_counted(ctx):
    pred = np.array([[1, 1, 0, 0], [2, 0, 0, 0]], np.int32)
    gt = np.array([[1, 0, 1, 0], [1, 1, 0, 0]], np.int32)
    m = ctx.pixel_metrics(pred, gt)
    assert (m.counts.n_tp, m.counts.n_fp, m.counts.n_fn, m.counts.n_tn) == (2, 1, 2, 3)
    assert m.precision == pytest.approx(2.0 / 3.0)
    assert m.recall == pytest.approx(0.5)
    assert m.accuracy == pytest.approx(5.0 / 8.0)
    assert m.fscore == pytest.approx(ctx.fscore(2.0 / 3.0, 0.5))


def test_pixel_metrics_perfect_and_degenerate(ctx):
    gt = np.array([[0, 1, 0], [2, 2, 0], [0, 0, 3]], np.int32)
    m = ctx.pixel_metrics(gt, gt)
    assert (m.precision, m.recall, m.accuracy, m.fscore) == (1.0, 1.0, 1.0, 1.0)
    empty = np.zeros((2, 2), np.int32)
    some = np.array([[1, 0], [0, 0]], np.int32)
    m = ctx.pixel_metrics(empty, some)
    assert m.degenerate_precision and not m.degenerate_recall
    assert m.precision == 0.0 and m.recall == 0.0
    both = ctx.pixel_metrics(empty, empty)
    assert both.degenerate_precision and both.degenerate_recall
    assert both.accuracy == 1.0


def test_pixel_metrics_counts_partition(ctx):
    rng = np.random.default_rng(9)
    pred = rng.integers(0, 3, (7, 9)).astype(np.int32)
    gt = rng.integers(0, 3, (7, 9)).astype(np.int32)
    m = ctx.pixel_metrics(pred, gt)
    assert m.counts.total() == 63
    assert 0.0 <= m.accuracy <= 1.0


def test_instance_exact_match(ctx):
    m = np.zeros((4, 6), np.int32)
    m[0:2, 0:2] = 1
    m[2:4, 4:6] = 2
    r = ctx.instance_metrics(m, m)
    assert (r.correct, r.incorrect, r.misdetection) == (2, 0, 0)


def test_instance_best_iou_wins(ctx):
    gt = np.zeros((3, 20), np.int32)
    gt[1, 0:10] = 1
    pred = np.zeros((3, 20), np.int32)
    pred[1, 2:8] = 1       # inter 6, union 10
    pred[0, 8:12] = 2      # no overlap (other row)
    pred[1, 8:10] = 2      # inter 2, union 10 + 6 - 2
    r = ctx.instance_metrics(pred, gt, 0.5)
    assert (r.correct, r.incorrect, r.misdetection) == (1, 1, 0)


def test_instance_unmatched_truth_is_misdetection(ctx):
    gt = np.zeros((5, 5), np.int32)
    gt[0:2, 0:2] = 1
    gt[3:5, 3:5] = 2
    pred = np.zeros((5, 5), np.int32)
    pred[0:2, 0:2] = 1
    r = ctx.instance_metrics(pred, gt)
    assert (r.correct, r.incorrect, r.misdetection) == (1, 0, 1)


def test_instance_iou_gate(ctx):
    gt = np.zeros((1, 12), np.int32)
    gt[0, 0:8] = 1
    pred = np.zeros((1, 12), np.int32)
    pred[0, 4:12] = 1      # inter 4, union 12: IoU 1/3
    low = ctx.instance_metrics(pred, gt, 0.5)
    assert (low.correct, low.incorrect, low.misdetection) == (0, 1, 1)
    assert ctx.instance_metrics(pred, gt, 1.0 / 3.0).correct == 1


def test_instance_one_to_one(ctx):
    gt = np.zeros((2, 8), np.int32)
    gt[0, :] = 1
    pred = np.zeros((2, 8), np.int32)
    pred[0, 0:4] = 1
    pred[0, 4:8] = 2       # both IoU 0.5 against the same truth
    r = ctx.instance_metrics(pred, gt, 0.5)
    assert (r.correct, r.incorrect, r.misdetection) == (1, 1, 0)

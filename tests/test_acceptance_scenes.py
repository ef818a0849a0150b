"""The reference acceptance gate's scene-based checks, end to end on the device
(SURVEY.md §8(f) rows 1 and 4): scenes from the device generator, the CUDA
detect pipeline, the device evaluation metrics.

* check 4 (acceptance.cpp:220-266): scene_batch(20, 7100), delta_pd = 0.48,
  2400 superpixels -> pixel accuracy >= 0.99, F >= 0.85, instance rate >= 0.9
  (greedy IoU >= 0.5, match_truth :182-218), no missed pothole >= 2 px deep,
  slowest frame <= 5 s;
* check 5 (acceptance.cpp:268-300): plane-only scenes, seeds 11-13 -> the
  transformed disparity has std <= 1 px and mean within 0.5 px of delta_dt.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2012_10802_b200.scenes import SceneSpec, generate_scene, scene_batch

pytestmark = pytest.mark.gpu


def match_truth(pred: np.ndarray, gt: np.ndarray, iou_min: float) -> np.ndarray:
    """acceptance.cpp:182-218: greedy one-to-one by descending IoU (ties: lower
    prediction, then lower truth); returns matched[g] for g = 0..max(gt)."""
    np_, ng = int(pred.max()), int(gt.max())
    ap = np.bincount(pred.ravel(), minlength=np_ + 1)
    ag = np.bincount(gt.ravel(), minlength=ng + 1)
    both = (pred > 0) & (gt > 0)
    inter = np.zeros((np_ + 1, ng + 1), np.int64)
    np.add.at(inter, (pred[both], gt[both]), 1)
    pairs = [(inter[p, g] / (ap[p] + ag[g] - inter[p, g]), p, g)
             for p in range(1, np_ + 1) for g in range(1, ng + 1) if inter[p, g] > 0]
    pairs.sort(key=lambda t: (-t[0], t[1], t[2]))
    matched = np.zeros(ng + 1, bool)
    used = np.zeros(np_ + 1, bool)
    for iou, p, g in pairs:
        if iou < iou_min:
            break
        if used[p] or matched[g]:
            continue
        used[p] = matched[g] = True
    return matched


def test_check4_detection_batch(gpu):
    cfg = gpu.lib.default_config(delta_pd=0.48, superpixels=2400)
    tp = fp = fn = tn = 0
    gt_total = gt_matched = deep_missed = 0
    worst_ms = 0.0
    for sc in scene_batch(gpu, 20, 7100):
        res = gpu.detect(sc.left, sc.right, cfg, want=("labels",))
        worst_ms = max(worst_ms, res.total_ms)
        pm = gpu.pixel_metrics(res.labels, sc.gt_mask)
        tp += pm.counts.n_tp
        fp += pm.counts.n_fp
        fn += pm.counts.n_fn
        tn += pm.counts.n_tn
        matched = match_truth(res.labels, sc.gt_mask, 0.5)
        for g in range(1, matched.size):
            gt_total += 1
            if matched[g]:
                gt_matched += 1
            elif sc.spec.potholes[g - 1].depth >= 2.0:
                deep_missed += 1
    accuracy = (tp + tn) / (tp + fp + fn + tn)
    precision, recall = tp / (tp + fp), tp / (tp + fn)
    f = gpu.fscore(precision, recall)
    rate = gt_matched / gt_total
    detail = (f"accuracy {accuracy:.4f}, F {f:.4f}, instance rate {rate:.3f} "
              f"({gt_matched}/{gt_total}), deep misses {deep_missed}, slowest {worst_ms:.1f} ms")
    print(detail)
    assert accuracy >= 0.99 and f >= 0.85 and rate >= 0.90, detail
    assert deep_missed == 0 and worst_ms <= 5000.0, detail


def test_check5_flatness(gpu):
    cfg = gpu.lib.default_config()
    worst_std = worst_mean = 0.0
    for seed in (11, 12, 13):
        spec = SceneSpec(a0=5.5, a1=0.08, phi_true=(seed - 12.0) * 0.02, texture_seed=seed)
        sc = generate_scene(gpu, spec)
        d2 = gpu.detect(sc.left, sc.right, cfg, want=("d2",)).d2
        x = d2[d2 != -1.0].astype(np.float64)
        mean = x.sum() / x.size
        sd = np.sqrt(max(0.0, (x * x).sum() / x.size - mean * mean))
        worst_std = max(worst_std, sd)
        worst_mean = max(worst_mean, abs(mean - cfg.delta_dt))
    assert worst_std <= 1.0 and worst_mean <= 0.5, (worst_std, worst_mean)

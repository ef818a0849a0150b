"""Known answers of the reference segmentation suite, both implementations.

Ports /root/reference/proj/tests/test_segmentation.cpp and acceptance.cpp
checks 6-8 (:305-454) with our own seeded inputs.
"""
from __future__ import annotations

from collections import deque

import numpy as np
import pytest

from paper_2012_10802_b200.api import DegenerateError, Histogram2D, InvalidArgument, threshold

DU = (1, -1, 0, 0, 1, 1, -1, -1)
DV = (0, 0, 1, -1, 1, -1, 1, -1)


def ccl_oracle(mask, conn):
    """Stack flood fill, labels in first-encounter scan order (test_segmentation.cpp:14-42)."""
    h, w = mask.shape
    out = np.zeros((h, w), np.int32)
    nxt = 0
    nd = 4 if conn == 4 else 8
    for v in range(h):
        for u in range(w):
            if mask[v, u] == 0 or out[v, u] != 0:
                continue
            nxt += 1
            out[v, u] = nxt
            st = [(u, v)]
            while st:
                pu, pv = st.pop()
                for i in range(nd):
                    nu, nv = pu + DU[i], pv + DV[i]
                    if 0 <= nu < w and 0 <= nv < h and mask[nv, nu] != 0 and out[nv, nu] == 0:
                        out[nv, nu] = nxt
                        st.append((nu, nv))
    return out


def is_connected_partition(labels, count):
    if labels.min() < 1 or labels.max() > count:
        return False
    if len(np.unique(labels)) != count:
        return False
    for k in range(1, count + 1):
        if ccl_oracle((labels == k).astype(np.int32), 8).max() != 1:
            return False
    return True


# ------------------------------------------------------------------- SLIC --
def test_slic_constant_square_exact_grid(ctx):
    flat = np.full((120, 120), 30.0, np.float32)
    labels, _, count, _ = ctx.slic(flat, 36, 10.0, 10)
    assert count == 36
    _, sizes = np.unique(labels, return_counts=True)
    assert np.all(sizes == 400)
    vv, uu = np.meshgrid(np.arange(120), np.arange(120), indexing="ij")
    assert np.array_equal(labels, labels[(vv // 20) * 20, (uu // 20) * 20])


def test_slic_edge_adherence(ctx):
    m = np.zeros((96, 96), np.float32)
    m[:, 48:] = 100.0
    labels, _, _, _ = ctx.slic(m, 64, 0.5, 10)
    assert np.all(labels[1:95, 47] != labels[1:95, 48])


def test_slic_connected_partition_near_count(ctx):
    rng = np.random.default_rng(5)
    for trial in range(5):
        m = rng.uniform(0.0, 50.0, (60 + trial * 7, 80 + trial * 5)).astype(np.float32)
        labels, _, count, _ = ctx.slic(m, 48, 10.0, 10)
        assert is_connected_partition(labels, count)
        assert 48 * 0.8 <= count <= 48 * 1.2


def test_slic_deterministic_and_bounded(ctx):
    vv, uu = np.meshgrid(np.arange(40), np.arange(40), indexing="ij")
    m = ((uu * 7 + vv * 3) % 23).astype(np.float32)
    a = ctx.slic(m, 16, 5.0, 10)[0]
    b = ctx.slic(m, 16, 5.0, 10)[0]
    assert np.array_equal(a, b)
    with pytest.raises(InvalidArgument):
        ctx.slic(m, 40 * 40 + 1, 5.0, 10)
    with pytest.raises(InvalidArgument):
        ctx.slic(m, 3, 5.0, 10)


def test_acceptance_slic_partitions(ctx):
    """acceptance.cpp:379-420 — SLIC maps are connected partitions within ±20%."""
    rng = np.random.default_rng(6000)
    for _ in range(10):
        h, w = int(rng.integers(40, 90)), int(rng.integers(40, 90))
        p = int(rng.integers(16, 64))
        m = rng.uniform(0.0, 60.0, (h, w)).astype(np.float32)
        m[rng.random((h, w)) < 0.1] = -1.0
        labels, _, count, _ = ctx.slic(m, p, 8.0, 10)
        assert is_connected_partition(labels, count)
        assert p * 0.8 <= count <= p * 1.2


# ---------------------------------------------------------------- pooling --
def test_pool_superpixels(ctx):
    m = np.array([[28.0, 30.0, 32.0], [-1.0, -1.0, 10.0]], np.float32)
    lab = np.array([[1, 1, 1], [2, 2, 1]], np.int32)
    d3 = ctx.pool_superpixels(m, lab, 2)
    assert d3[0, 0] == pytest.approx(25.0)
    assert d3[0, 2] == d3[0, 0]
    assert d3[1, 0] == -1.0
    assert np.array_equal(ctx.pool_superpixels(d3, lab, 2), d3)
    flat = np.full((2, 3), 4.0, np.float32)
    assert np.array_equal(ctx.pool_superpixels(flat, lab, 2), flat)


# -------------------------------------------------------------- histogram --
def test_histogram_constant_diagonal_bin(ctx):
    hist = ctx.build_histogram(np.full((5, 5), 12.0, np.float32), 0.5)
    assert hist.total == 9
    occ = np.argwhere(hist.counts > 0)
    assert occ.shape[0] == 1 and occ[0, 0] == occ[0, 1]
    assert hist.center(occ[0, 0]) == pytest.approx(12.25)


def test_histogram_single_interior_vector(ctx):
    m = np.full((3, 3), 20.0, np.float32)
    m[1, 1] = 10.0
    hist = ctx.build_histogram(m, 1.0)
    assert hist.total == 1 and hist.counts[0, 10] == 1


def test_histogram_partial_neighbourhood_skipped(ctx):
    m = np.full((4, 4), 20.0, np.float32)
    m[0, 0] = -1.0
    assert ctx.build_histogram(m, 1.0).total == 3


def test_histogram_checkerboard(ctx):
    vv, uu = np.meshgrid(np.arange(6), np.arange(6), indexing="ij")
    m = ((uu + vv) % 2).astype(np.float32)
    hist = ctx.build_histogram(m, 0.125)
    assert hist.total == 16
    at0 = at1 = 0
    for i, j in np.argwhere(hist.counts > 0):
        assert hist.center(j) == pytest.approx(0.5 + 0.0625)
        if i == 0:
            at0 += hist.counts[i, j]
        else:
            at1 += hist.counts[i, j]
    assert at0 == 8 and at1 == 8


def test_histogram_empty_and_error(ctx):
    hist = ctx.build_histogram(np.full((2, 2), 5.0, np.float32), 0.25)
    assert hist.total == 0 and hist.counts.shape == (0, 0)
    with pytest.raises(InvalidArgument):
        ctx.build_histogram(np.zeros((4, 4), np.float32), 0.0)


# -------------------------------------------------------------- threshold --
def test_threshold_bimodal(ctx):
    m = np.full((22, 50), 30.0, np.float32)
    m[:4, :] = 20.0
    thr = ctx.find_road_threshold(ctx.build_histogram(m, 0.5), 2.36, 3.0)
    assert thr.mu1 == pytest.approx(20.25, rel=1e-9)
    assert thr.mu2 == pytest.approx(30.25, rel=1e-9)
    assert thr.t_r == pytest.approx(30.25, rel=1e-9)
    assert thr.t_s == pytest.approx(27.89, rel=1e-9)


def test_threshold_constant_degenerate(ctx):
    thr = ctx.find_road_threshold(ctx.build_histogram(np.full((6, 6), 25.0, np.float32), 0.5),
                                  2.36, 3.0)
    assert thr.degenerate
    assert thr.t_r == pytest.approx(25.25)


def test_threshold_off_diagonal_excluded(ctx):
    counts = np.zeros((50, 50), np.int64)
    counts[10, 40] = 5
    counts[20, 20] = 3
    counts[30, 30] = 3
    thr = ctx.find_road_threshold(Histogram2D(1.0, 0.0, counts, 11), 1.0, 3.0)
    assert thr.excluded_fraction == pytest.approx(5.0 / 11.0)
    assert thr.mu1 == pytest.approx(20.5)
    assert thr.mu2 == pytest.approx(30.5)
    counts[:] = 0
    counts[10, 40] = 5
    with pytest.raises(DegenerateError):
        ctx.find_road_threshold(Histogram2D(1.0, 0.0, counts, 5), 1.0, 3.0)


def exhaustive_mu2(counts, origin, bw, tau):
    diag = {}
    for i, j in np.argwhere(counts > 0):
        g1 = origin + (i + 0.5) * bw
        g2 = origin + (j + 0.5) * bw
        if abs(g1 - g2) > tau:
            continue
        key = (g1 + g2) / 2.0
        diag[key] = diag.get(key, 0) + int(counts[i, j])
    pts = sorted(diag.items())
    best, best_mu2 = 1e300, 0.0
    for s in range(1, len(pts)):
        n1 = sum(c for _, c in pts[:s])
        n2 = sum(c for _, c in pts[s:])
        m1 = sum(c * x for x, c in pts[:s]) / n1
        m2 = sum(c * x for x, c in pts[s:]) / n2
        sse = sum(c * (x - (m1 if i < s else m2)) ** 2 for i, (x, c) in enumerate(pts))
        if sse < best:
            best, best_mu2 = sse, m2
    return best_mu2


def test_threshold_exhaustive_equivalence(ctx):
    """test_segmentation.cpp:225-275 and acceptance.cpp:346-375."""
    rng = np.random.default_rng(11)
    checked = 0
    for _ in range(200):
        counts = np.zeros((20, 20), np.int64)
        for _ in range(12):
            counts[rng.integers(0, 20), rng.integers(0, 20)] += rng.integers(1, 51)
        hist = Histogram2D(0.5, 10.0, counts, int(counts.sum()))
        try:
            thr = ctx.find_road_threshold(hist, 1.0, 3.0)
        except DegenerateError:
            continue
        if thr.degenerate:
            continue
        assert thr.mu2 == pytest.approx(exhaustive_mu2(counts, 10.0, 0.5, 3.0), rel=1e-9)
        checked += 1
    assert checked > 50


def test_threshold_shift_invariance(ctx):
    vv, uu = np.meshgrid(np.arange(24), np.arange(40), indexing="ij")
    m = (30.0 + ((uu + vv) % 2) * 0.25).astype(np.float32)
    m[8:12, 10:18] = 24.0
    c = np.float32(4.0)
    t1 = ctx.find_road_threshold(ctx.build_histogram(m, 0.25), 2.0, 3.0)
    t2 = ctx.find_road_threshold(ctx.build_histogram(m + c, 0.25), 2.0, 3.0)
    assert t2.t_r == pytest.approx(t1.t_r + 4.0, rel=1e-12)
    assert np.array_equal(m < t1.t_s, (m + c) < t2.t_s)


# -------------------------------------------------------------------- CCL --
def test_ccl_empty(ctx):
    assert np.all(ctx.connected_components(np.zeros((4, 4), np.int32), 8) == 0)


def test_ccl_diagonal_touch(ctx):
    m = np.zeros((3, 3), np.int32)
    m[0, 0] = m[1, 1] = 1
    assert ctx.connected_components(m, 8).max() == 1
    assert ctx.connected_components(m, 4).max() == 2


def test_ccl_random_masks_equal_flood_fill(ctx):
    rng = np.random.default_rng(17)
    for trial in range(20):
        h, w = (32, 32) if trial < 10 else (int(rng.integers(1, 70)), int(rng.integers(1, 70)))
        m = (rng.random((h, w)) < 0.4).astype(np.int32)
        for conn in (4, 8):
            assert np.array_equal(ctx.connected_components(m, conn), ccl_oracle(m, conn))


# ----------------------------------------------------------------- detect --
def _detect_fixture():
    n = 90
    vv, uu = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    sp = ((vv // 10) * 9 + uu // 10 + 1).astype(np.int32)
    thr = threshold(t_r=30.0, t_s=27.64)

    def pooled(low):
        d3 = np.full((n, n), 30.0, np.float32)
        for k in low:
            d3[sp == k] = 25.0
        return d3
    return sp, thr, pooled


def test_detect_nothing_below(ctx):
    sp, thr, pooled = _detect_fixture()
    assert np.all(ctx.detect_potholes(pooled([]), sp, 10.0, thr, 5, 2) == 0)


def test_detect_interior_blob(ctx):
    sp, thr, pooled = _detect_fixture()
    out = ctx.detect_potholes(pooled([31, 32, 40]), sp, 10.0, thr, 5, 2)
    assert out.max() == 1 and (out != 0).sum() == 300


def test_detect_single_superpixel_rejected(ctx):
    sp, thr, pooled = _detect_fixture()
    assert np.all(ctx.detect_potholes(pooled([40]), sp, 10.0, thr, 5, 2) == 0)


def test_detect_border_rejected(ctx):
    sp, thr, pooled = _detect_fixture()
    assert np.all(ctx.detect_potholes(pooled([1, 2, 10]), sp, 10.0, thr, 5, 2) == 0)


def test_detect_lower_threshold_monotone(ctx):
    sp, thr, pooled = _detect_fixture()
    d3 = pooled([31, 32, 40, 57])
    base = ctx.detect_potholes(d3, sp, 10.0, thr, 5, 2)
    low = ctx.detect_potholes(d3, sp, 10.0, threshold(30.0, 20.0), 5, 2)
    assert np.all(base[low != 0] != 0)


def test_detect_scan_order_relabel(ctx):
    sp, thr, pooled = _detect_fixture()
    out = ctx.detect_potholes(pooled([31, 32, 58, 59, 22, 23]), sp, 10.0, thr, 5, 2)
    # components are renumbered by first pixel in scan order
    firsts = [np.argmax((out == k).ravel()) for k in range(1, out.max() + 1)]
    assert firsts == sorted(firsts) and out.max() >= 2

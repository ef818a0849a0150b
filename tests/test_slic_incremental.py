"""SLIC incremental rounds (slic.cu, TileDirty / delta_pixel).

After round 0 the per-label sums persist: a round moves only the terms of the
pixels whose label changed (RPD_SLIC_INCREMENTAL = 2, the product default), and
optionally skips the tiles that no moved centre's window reaches (= 1).  Both
must give exactly the labels and centres of the full re-summation (= 0) and of
the oracle (segmentation.cpp:30-93, 170-229): on noisy rasters (every centre
moves every round), on flat rasters (the rounds converge and tiles are
skipped), with orphan rounds (every tile is re-assigned after a round with
orphans) and for 0, 1 and 2 iterations.  The modes are switched through the
checked build's environment knob; the product library ignores it."""
from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import pytest

from paper_2012_10802_b200.api import Library
from test_slic_orphans import blocky_cases

pytestmark = pytest.mark.gpu
DBG_LIB = Path(__file__).resolve().parents[1] / "paper_2012_10802_b200" / "_lib_dbg" / \
    "librpd_b200.so"
MODES = (0, 1, 2)


@pytest.fixture(scope="module")
def dbg():
    if not DBG_LIB.exists():
        pytest.fail("checked build missing: make -C paper_2012_10802_b200/csrc DEBUG_KNOBS=1")
    return Library(str(DBG_LIB)).context(0)


def slic_mode(ctx, mode, d2, p, comp, it, large=None):
    os.environ["RPD_SLIC_INCREMENTAL"] = str(mode)
    if large is not None:  # tile height: the large-raster kernels on a small raster, or the reverse
        os.environ["RPD_SLIC_LARGE_TILES"] = str(int(large))
    try:
        return ctx.slic(d2, p, comp, it)
    finally:
        del os.environ["RPD_SLIC_INCREMENTAL"]
        os.environ.pop("RPD_SLIC_LARGE_TILES", None)


def same(a, b):
    la, ca, na, sa = a
    lb, cb, nb, sb = b
    assert na == nb and sa == sb
    assert np.array_equal(la, lb), f"{int((la != lb).sum())} labels differ"
    assert np.array_equal(ca.view(np.uint64), cb.view(np.uint64))


def noisy(h, w, seed):
    rng = np.random.default_rng(seed)
    v, u = np.mgrid[0:h, 0:w]
    d2 = (0.03 * v + 0.01 * u + rng.normal(0, 0.4, (h, w))).astype(np.float32)
    d2[rng.random((h, w)) < 0.02] = -1.0  # invalid pixels (values_or_zero)
    return d2


@pytest.mark.parametrize("h,w,p,it", [(200, 300, 150, 10), (97, 131, 40, 4), (240, 320, 300, 10),
                                      (64, 64, 16, 1), (64, 64, 16, 2), (50, 70, 12, 0)])
def test_modes_equal_oracle_noisy(dbg, oracle, h, w, p, it):
    d2 = noisy(h, w, h * 1000 + w)
    ref = oracle.slic(d2, p, 8.0, it)
    for mode in MODES:
        same(slic_mode(dbg, mode, d2, p, 8.0, it), ref)
        same(slic_mode(dbg, mode, d2, p, 8.0, it, large=True), ref)


def test_flat_raster_converges_and_skips_tiles(dbg, oracle):
    # piecewise-constant values: the cells settle, later rounds move no centre
    h, w = 240, 320
    d2 = np.zeros((h, w), np.float32)
    d2[:, w // 2:] = 3.0
    ref = oracle.slic(d2, 120, 8.0, 10)
    before = dbg.stats()
    same(slic_mode(dbg, 1, d2, 120, 8.0, 10, large=False), ref)
    after = dbg.stats()
    assigned = after.slic_tiles_assigned - before.slic_tiles_assigned
    skipped = after.slic_tiles_skipped - before.slic_tiles_skipped
    tiles = ((w + 31) // 32) * ((h + 23) // 24)
    assert assigned + skipped == 10 * tiles  # rounds 1..10 visit every tile once
    assert skipped > 0, "no tile was skipped on a converging raster"
    for mode in (0, 2):
        same(slic_mode(dbg, mode, d2, 120, 8.0, 10), ref)


def test_partly_moving_raster_skips_some_tiles(dbg, oracle):
    # flat left half (settles), noisy right half (keeps moving)
    h, w = 192, 384
    d2 = noisy(h, w, 7)
    d2[:, : w // 2] = 1.0
    ref = oracle.slic(d2, 200, 8.0, 10)
    before = dbg.stats()
    same(slic_mode(dbg, 1, d2, 200, 8.0, 10, large=True), ref)
    after = dbg.stats()
    skipped = after.slic_tiles_skipped - before.slic_tiles_skipped
    assigned = after.slic_tiles_assigned - before.slic_tiles_assigned
    assert skipped > 0 and assigned > skipped
    # checked-build counters: some centres moved and some pixels changed label, far from all
    moved = after.slic_centres_moved - before.slic_centres_moved
    changed = after.slic_pixels_changed - before.slic_pixels_changed
    assert 0 < moved < 10 * 200 and 0 < changed < h * w
    n, who = dbg.guard_check()  # the tile flag / counter buffers of the skipping mode included
    assert n == 0, f"{n} guard bytes overwritten (first: {who})"


ORPHAN_CASES = blocky_cases()[:48]  # orphans before the last round in 3 of these (test_slic_orphans)


@pytest.mark.parametrize("i", range(len(ORPHAN_CASES)))
def test_orphan_rounds_all_modes(dbg, oracle, i):
    d2, p, comp = ORPHAN_CASES[i]
    ref = oracle.slic(d2, p, comp, 10)
    for mode in MODES:
        same(slic_mode(dbg, mode, d2, p, comp, 10), ref)
    same(slic_mode(dbg, 2, d2, p, comp, 10, large=True), ref)  # 40-row tiles (large rasters)
    same(slic_mode(dbg, 1, d2, p, comp, 10, large=True), ref)


@pytest.mark.parametrize("large", [False, True])
def test_brute_force_walk_with_persistent_sums(dbg, oracle, large):
    # the per-pixel scan of every centre (bucket / tile overflow path) under both tile heights
    d2 = noisy(120, 170, 11)
    ref = oracle.slic(d2, 150, 8.0, 5)
    os.environ["RPD_SLIC_FORCE_WALK"] = "1"
    try:
        for mode in MODES:
            same(slic_mode(dbg, mode, d2, 150, 8.0, 5, large=large), ref)
    finally:
        del os.environ["RPD_SLIC_FORCE_WALK"]


def test_product_ignores_the_knob(gpu, oracle):
    d2 = noisy(120, 160, 3)
    ref = oracle.slic(d2, 60, 8.0, 5)
    os.environ["RPD_SLIC_INCREMENTAL"] = "0"
    try:
        same(gpu.slic(d2, 60, 8.0, 5), ref)
    finally:
        del os.environ["RPD_SLIC_INCREMENTAL"]

"""Segmented path aggregation (sgm_tma.cu, agg_body): horizontal / vertical
chains longer than the longest diagonal are cut into segments, one CTA each;
a segment starts a warm-up before its first stored step, and is recomputed
from its predecessor's true state whenever its warm-up state differs.  The
outputs must stay bit-identical to aggregate_costs (sgm.cpp:70-110) in every
case, including the adversarial one where the warm-up cannot converge
(uniform costs across the cut keep the true state's shape forever)."""
from __future__ import annotations

import numpy as np
import pytest

import os
from pathlib import Path

from paper_2012_10802_b200.api import AGG_KERNELS, EIGHT_DIRECTIONS, Library, model

pytestmark = pytest.mark.gpu


def aggregate_both(gpu, oracle, vol, paths=8, l1=10.0, l2=120.0):
    dirs = EIGHT_DIRECTIONS[:paths]
    before = gpu.stats().agg_segment_reruns
    a = gpu.aggregate_costs(vol, l1, l2, dirs)
    st = gpu.stats()
    assert AGG_KERNELS[st.last_agg_kernel] == "u8_tma"
    b = oracle.aggregate_costs(vol, l1, l2, dirs)
    mism = a.view(np.uint32) != b.view(np.uint32)
    assert not mism.any(), f"{int(mism.sum())} cells differ, first {np.argwhere(mism)[0].tolist()}"
    return st.agg_segmented_ctas, st.agg_segment_reruns - before


@pytest.mark.parametrize("shape", [(200, 600, 17), (96, 800, 17), (600, 200, 17),
                                   (150, 700, 29), (130, 900, 33)])
def test_segmented_random_volumes_exact(gpu, oracle, shape):
    """Textured (random) costs: segments are active and converge."""
    h, w, n = shape
    rng = np.random.default_rng(h * 1000 + w + n)
    vol = rng.integers(0, 61, size=(h, w, n)).astype(np.float32)
    segs, _ = aggregate_both(gpu, oracle, vol)
    assert segs > 0, "the long chains were not segmented"


@pytest.mark.parametrize("orient", ["rows", "cols"])
def test_segmented_uniform_band_forces_recompute(gpu, oracle, orient):
    """Uniform costs over a band that contains the cuts: the warm-up state
    (all zero) never meets the true state shaped by the texture before the
    band, so the segments must be recomputed, and the result stays exact."""
    h, w, n = 200, 600, 17
    rng = np.random.default_rng(77)
    vol = rng.integers(0, 61, size=(h, w, n)).astype(np.float32)
    vol[:, 120:480, :] = 30.0
    if orient == "cols":
        vol = np.ascontiguousarray(vol.transpose(1, 0, 2))
    segs, reruns = aggregate_both(gpu, oracle, vol)
    assert segs > 0
    assert reruns > 0, "the recompute path was not exercised"


def test_segmented_match_pair_dump_exact(gpu, oracle):
    """The production match_pair buffers (both reference volumes, u8 cost
    kernel, right-reference overrides) on a raster whose rows are segmented."""
    h, w = 180, 640
    rng = np.random.default_rng(5)
    left = rng.integers(0, 256, (h, w)).astype(np.float32)
    right = np.roll(left, 4, axis=1) + rng.normal(0, 2, (h, w)).astype(np.float32)
    right = np.clip(np.rint(right), 0, 255).astype(np.float32)
    m = model(3.0, 0.02, 0.01)
    cfg = gpu.lib.default_config(lambda1=10.0, lambda2=120.0)
    a = gpu.match_pair_dump_ex(left, right, m, cfg, 16)
    assert gpu.stats().agg_segmented_ctas > 0
    b = oracle.match_pair_dump_ex(left, right, m, oracle.lib.default_config(
        lambda1=10.0, lambda2=120.0), 16)
    for k in ("cost", "cost_right", "agg_left", "agg_right", "disp_left", "disp_right"):
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k


def test_segmented_replays_are_deterministic(gpu, oracle):
    """Flags and tickets rearm between launches: repeated launches (including
    ones that recompute) give identical results."""
    h, w, n = 200, 600, 17
    rng = np.random.default_rng(9)
    vol = rng.integers(0, 61, size=(h, w, n)).astype(np.float32)
    vol[:, 150:470, :] = 12.0
    first = gpu.aggregate_costs(vol, 10.0, 120.0)
    for _ in range(5):
        again = gpu.aggregate_costs(vol, 10.0, 120.0)
        assert np.array_equal(first.view(np.uint32), again.view(np.uint32))


DBG_LIB = Path(__file__).resolve().parents[1] / "paper_2012_10802_b200" / "_lib_dbg" / \
    "librpd_b200.so"


@pytest.mark.parametrize("levels", [65, 129, 200])
@pytest.mark.parametrize("nseg", [2, 3])
def test_forced_segments_multi_lane_layouts(oracle, levels, nseg):
    """The product segments only one-lane chains; the checked build can force
    segments on every layout (RPD_AGG_SPLIT=n): the G = 4 / 8 lane groups
    (shuffle-coupled chains) must stay exact too, converged or recomputed."""
    if not DBG_LIB.exists():
        pytest.fail("checked build missing: make -C paper_2012_10802_b200/csrc DEBUG_KNOBS=1")
    ctx = Library(str(DBG_LIB)).context(0)
    h, w = 40, 700
    rng = np.random.default_rng(levels + nseg)
    vol = rng.integers(0, 61, size=(h, w, levels)).astype(np.float32)
    vol[:, 180:500, :] = 20.0  # the cuts inside a uniform band: recompute there
    os.environ["RPD_AGG_SPLIT"] = str(nseg)
    try:
        segs, _ = aggregate_both(ctx, oracle, vol)
    finally:
        del os.environ["RPD_AGG_SPLIT"]
    assert segs > 0

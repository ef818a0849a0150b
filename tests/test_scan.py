"""The single-pass exclusive scan (scan.cuh): ticketed tiles of 2048 elements,
warp-parallel decoupled look-back, descriptors tagged per launch (no clearing
between launches).  Exact prefix sums and totals at tile-boundary sizes, for
sparse, dense and multi-valued flags, over many consecutive launches (the
tags advance, stale descriptors of earlier launches must never match)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [1, 2, 7, 2047, 2048, 2049, 4096, 3 * 2048 + 5, 100_003, 1_049_601]


@pytest.mark.parametrize("n", SIZES)
def test_scan_exact(gpu, n):
    rng = np.random.default_rng(n)
    for flags in (rng.integers(0, 2, n), (rng.random(n) < 0.01).astype(np.int64),
                  np.ones(n, np.int64), np.zeros(n, np.int64), rng.integers(0, 4, n)):
        flags = flags.astype(np.int32)
        out, total = gpu.debug_scan(flags)
        exp = np.concatenate([[0], np.cumsum(flags, dtype=np.int64)[:-1]]).astype(np.int32)
        assert np.array_equal(out, exp)
        assert total == int(flags.sum())


def test_scan_many_consecutive_launches(gpu):
    rng = np.random.default_rng(5)
    for i in range(40):
        n = int(rng.integers(1, 300_000))
        flags = rng.integers(0, 2, n).astype(np.int32)
        out, total = gpu.debug_scan(flags)
        assert total == int(flags.sum())
        assert out[-1] == total - flags[-1]
        assert np.array_equal(out[: min(n, 5000)],
                              np.concatenate([[0], np.cumsum(flags[: min(n, 5000)])[:-1]]))


def test_scan_empty(gpu):
    out, total = gpu.debug_scan(np.zeros(0, np.int32))
    assert out.size == 0 and total == 0

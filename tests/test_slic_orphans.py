"""SLIC rounds with orphans: pixels that no centre window covers
(segmentation.cpp:59-71) take the spatially nearest centre.  The device
handles an intermediate round's orphans inside the next round's centre kernel
(their sums must land before any centre is finalised) and the last round's in
a separate fallback.  Blocky high-contrast rasters with few superpixels make
centres drift apart, which opens such gaps in intermediate rounds (a numpy
restatement of the reference rounds, seed nudge included, finds orphans before
the last round in 3 of the first 48 cases of this generator, e.g. case 29 in
rounds 7-10); the device must equal the oracle exactly on all of them."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def blocky_cases(n=120, seed=1):
    rng = np.random.default_rng(seed)
    cases = []
    while len(cases) < n:
        h, w = int(rng.integers(20, 70)), int(rng.integers(20, 120))
        bh, bw = int(rng.integers(3, 15)), int(rng.integers(3, 15))
        base = rng.integers(0, 4, size=(h // bh + 1, w // bw + 1)).astype(np.float32) * \
            np.float32(rng.choice([5, 50, 500]))
        d2 = np.kron(base, np.ones((bh, bw), np.float32))[:h, :w]
        p = int(rng.integers(4, 40))
        comp = float(rng.choice([0.01, 0.1, 1.0, 10.0]))
        if p <= h * w:
            cases.append((np.ascontiguousarray(d2), p, comp))
    return cases


CASES = blocky_cases()


@pytest.mark.parametrize("i", range(len(CASES)))
def test_slic_rounds_with_orphans_exact(gpu, oracle, i):
    d2, p, comp = CASES[i]
    la, ca, na, sa = gpu.slic(d2, p, comp, 10)
    lb, cb, nb, sb = oracle.slic(d2, p, comp, 10)
    assert na == nb and sa == sb
    assert np.array_equal(la, lb), f"{int((la != lb).sum())} labels differ"
    assert np.array_equal(ca.view(np.uint64), cb.view(np.uint64))

"""The device roll-angle sin/cos (road.cu dd_sincos) is correctly rounded:
compared with 40-digit decimal references on seeded angles covering the
golden-section brackets (|phi| <= 0.75) and the pi/2-reduction path."""
from decimal import Decimal, getcontext

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref(x):
    """Correctly rounded sin/cos from a 45-digit Taylor series (40 terms: the
    remainder is < 1e-60 for |x| <= 3)."""
    getcontext().prec = 45
    d = Decimal(float(x))
    s, t = Decimal(0), d
    c, tc = Decimal(0), Decimal(1)
    for n in range(40):
        s += t
        c += tc
        t = -t * d * d / ((2 * n + 2) * (2 * n + 3))
        tc = -tc * d * d / ((2 * n + 1) * (2 * n + 2))
    return float(s), float(c)


def test_device_sincos_correctly_rounded(gpu):
    rng = np.random.default_rng(20121080)
    x = np.concatenate([rng.uniform(-0.27, 0.27, 3000), rng.uniform(-0.75, 0.75, 1000),
                        rng.uniform(-3.0, 3.0, 500), [0.0, 1e-300, -1e-12, 0.75, -0.75]])
    s, c = gpu.debug_sincos(x)
    ref = [_ref(v) for v in x]
    assert np.array_equal(s, np.array([r[0] for r in ref]))
    assert np.array_equal(c, np.array([r[1] for r in ref]))

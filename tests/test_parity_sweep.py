"""Full BASELINE sweep against the literal reference build (BASELINE.md §3
coverage): configs 1, 2, 4 and all 64 frames of config 3, every 64th frame of
config 5 (64 frames).  Bars: d0/d1 bit-exact, phi identical, D2 within 1e-4
relative, SLIC >= 99.9 %, pothole labels identical — on every frame."""
from __future__ import annotations

import json
import os
from pathlib import Path

import pytest

from sweep import run_sweep, sweep_cases

pytestmark = pytest.mark.gpu


def test_sweep_against_literal_reference(gpu, ref_lib):
    report = run_sweep(gpu, ref_lib, sweep_cases())
    out = os.environ.get("RPD_SWEEP_JSON")
    if out:
        Path(out).write_text(json.dumps(report, indent=1))
    s = report["summary"]
    bad = [r for r in report["records"] if not r["ok"]]
    assert not bad, (s, bad[:3])
    assert s["frames"] == 3 + 64 + 64

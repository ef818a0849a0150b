"""The reference's OWN test suite — /root/reference/proj/tests/{test_sgm,
test_perspective, test_road_geometry, test_segmentation}.cpp and the
acceptance gate (acceptance.cpp), compiled UNMODIFIED (tests/cpp/refsuite):

  * lit_*  against the literal reference build (untouched src/*.cpp + the
           Eigen subset in oracle/ref_shim): pins the shims themselves;
  * gpu_*  against the B200 library through the reference-API adapter
           (paper_2012_10802_b200/dropin/rpd_dropin.cpp -> librpd_b200.so): the drop-in
           proof — the reference's own known answers, exact DP / QR /
           flood-fill / 2-means oracles and acceptance checks 1-8 on the CUDA
           kernels.

The binaries are built here by __graft_entry__.build() (make -C
tests/cpp/refsuite) and travel to the GPU box prebuilt."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

BUILD = Path(__file__).resolve().parent / "cpp" / "refsuite" / "_build"
SUITES = ["test_sgm", "test_perspective", "test_road_geometry", "test_segmentation",
          "acceptance"]


def _run(binary: Path):
    if not binary.exists():
        pytest.fail(f"{binary} not built (make -C tests/cpp/refsuite; needs /root/reference "
                    "at build time)")
    out = subprocess.run([str(binary)], capture_output=True, text=True, timeout=900,
                         cwd=str(binary.parent))
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-3000:]
    if binary.name.endswith("acceptance"):
        lines = [ln for ln in text.splitlines() if ln.startswith(("PASS", "FAIL", "SKIP"))]
        assert sum(ln.startswith("PASS") for ln in lines) == 8, lines
        assert not any(ln.startswith("FAIL") for ln in lines), lines
    else:
        assert " 0 failed" in text, text[-3000:]
    return text


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_literal_build(suite):
    _run(BUILD / f"lit_{suite}")


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200(suite):
    _run(BUILD / f"gpu_{suite}")

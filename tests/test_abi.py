"""CPU-side checks of the C-ABI boundary (no GPU needed).

* include/rpd_b200.h is the contract: both shared libraries (the sm_100a CUDA
  product and the CPU oracle) export every entry point it declares.
* The CUDA library loads on a machine without a GPU and fails loudly
  (RPD_ECUDA) at context creation instead of falling back to the CPU.
* Host-only entry points (config defaults / validation / key=value parsing)
  behave like the reference (config.cpp:9-77).
"""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2012_10802_b200.api import (ABI_SYMBOLS, EXTENSION_SYMBOLS, Config, Library,
                                       RPD_ECUDA, RPD_EINVAL, RPD_OK)

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "rpd_b200.h"
CUDA_LIB = ROOT / "paper_2012_10802_b200" / "_lib" / "librpd_b200.so"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(rpd_[a-z0-9_]+)\s*\(", text)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True,
                         text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if " T " in ln}


def test_header_declares_the_binding_set():
    declared = set(header_symbols())
    assert set(ABI_SYMBOLS) <= declared
    assert set(EXTENSION_SYMBOLS) <= declared


@pytest.fixture(scope="module")
def cuda_lib_path():
    if not CUDA_LIB.exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_2012_10802_b200" / "csrc"), "-j8"],
                       check=True, stdout=subprocess.DEVNULL)
    return CUDA_LIB


def test_cuda_library_exports_every_declared_symbol(cuda_lib_path):
    missing = set(header_symbols()) - exported(cuda_lib_path)
    assert not missing, f"missing exports: {sorted(missing)}"


def test_oracle_exports_the_reference_entry_points(oracle_lib):
    missing = set(ABI_SYMBOLS) - exported(oracle_lib.path)
    assert not missing, f"oracle misses: {sorted(missing)}"


def test_cuda_library_loads_and_is_sm100a_only(cuda_lib_path):
    lib = Library(str(cuda_lib_path))
    assert lib.dll.rpd_abi_version() == 1
    assert lib.has_streaming
    sass = subprocess.run(["cuobjdump", "-lelf", str(cuda_lib_path)], capture_output=True,
                          text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", sass))
    assert arches == {"100a"}, arches


def test_cuda_library_has_tma_and_dpx_sass(cuda_lib_path):
    sass = subprocess.run(["cuobjdump", "-sass", str(cuda_lib_path)], capture_output=True,
                          text=True).stdout
    assert "UTMALDG" in sass and "UTMASTG" in sass  # TMA tensor loads / stores
    assert "VIADDMNMX" in sass                      # DPX fused add+min (SGM recurrence)
    # road fit: flag-tagged 128-bit partial exchange between the cooperative CTAs
    assert "STG.E.128.STRONG.GPU" in sass and "LDG.E.128.STRONG.GPU" in sass


def test_no_cpu_fallback_without_gpu(cuda_lib_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = Library(str(cuda_lib_path))
    h = C.c_void_p()
    assert lib.dll.rpd_ctx_create(0, 0, 0, 0, C.byref(h)) == RPD_ECUDA
    assert not h.value


def test_config_defaults_match_reference(cuda_lib_path, oracle_lib):
    for lib in (Library(str(cuda_lib_path)), oracle_lib):
        c = lib.default_config()
        assert (c.delta_pt, c.delta_dt, c.delta_pd) == (5.0, 30.0, 2.36)
        assert (c.d_max, c.d_max_pt, c.lambda1, c.lambda2) == (64, 16, 8.0, 32.0)
        assert (c.census_window, c.lr_threshold, c.superpixels) == (5, 1.0, 1365)
        assert (c.compactness, c.slic_iterations, c.hist_bin_width) == (8.0, 10, 0.25)
        assert (c.tau_diag, c.border_margin, c.min_superpixels, c.connectivity) == (3.0, 5, 2, 8)
        assert (c.roll_bracket, c.roll_tol, c.focal, c.baseline) == (0.261799, 1e-4, 700.0, 0.12)
        assert (c.cu, c.cv, c.sgm_paths) == (-1.0, -1.0, 8)


def _validate(lib, **kw):
    cfg = lib.default_config(**kw)
    return lib.dll.rpd_config_validate(None, C.byref(cfg))


@pytest.mark.parametrize("bad", [dict(delta_pt=-1.0), dict(delta_dt=0.0), dict(delta_pd=0.0),
                                 dict(d_max=0), dict(d_max_pt=0), dict(lambda1=0.0),
                                 dict(lambda1=40.0, lambda2=32.0), dict(census_window=4),
                                 dict(superpixels=3), dict(compactness=0.0),
                                 dict(connectivity=6), dict(roll_bracket=0.0),
                                 dict(roll_tol=0.0), dict(focal=0.0), dict(sgm_paths=6)])
def test_config_validation_rejects(oracle_lib, bad):
    ctx = oracle_lib.context()
    cfg = oracle_lib.default_config(**bad)
    with pytest.raises(ValueError):
        ctx.validate(cfg)


def test_config_set_key_value(oracle_lib):
    ctx = oracle_lib.context()
    cfg = oracle_lib.default_config()
    ctx.config_set(cfg, "delta_pd", "1.25")
    ctx.config_set(cfg, "superpixels", "777")
    assert cfg.delta_pd == 1.25 and cfg.superpixels == 777
    with pytest.raises(ValueError):
        ctx.config_set(cfg, "nope", "1")


def test_cpp_dropin_header_compiles():
    """The header-only C++ drop-in (include/rpd_b200.hpp) compiles as C++17."""
    src = ROOT / "tests" / "cpp" / "dropin_smoke.cpp"
    out = Path("/tmp") / "rpd_dropin_smoke"
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
                    str(src), "-o", str(out), "-L", str(CUDA_LIB.parent), "-lrpd_b200",
                    f"-Wl,-rpath,{CUDA_LIB.parent}"], check=True)

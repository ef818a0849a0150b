"""Runs the C++ drop-in smoke program (tests/cpp/dropin_smoke.cpp) on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2012_10802_b200" / "_lib"


@pytest.mark.gpu
def test_cpp_dropin_runs(tmp_path):
    exe = tmp_path / "dropin"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "dropin_smoke.cpp"), "-o", str(exe),
                    "-L", str(LIBDIR), "-lrpd_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout

"""B200-native stereo road-pothole detection (arxiv 2012.10802), drop-in for the
reference `rpd` C++ library's hot path (detect / sgm / transform / slic).

The compute path is `_lib/librpd_b200.so`: hand-written sm_100a CUDA kernels
behind the C-ABI in include/rpd_b200.h.  There is no CPU fallback: if the
library is missing or no CUDA device is present, `load_library()` raises.
"""
from __future__ import annotations

import os
from pathlib import Path

from . import api
from .api import (CapacityError, Config, Context, CudaError, DegenerateError, InvalidArgument,
                  Library, RoadModel, Threshold, model)

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "_lib"
CUDA_LIB = LIB_DIR / "librpd_b200.so"
SYNTH_LIB = LIB_DIR / "librpd_synth.so"

_loaded = None


def load_library(path: str | os.PathLike | None = None) -> Library:
    """Load the sm_100a CUDA library.  Fails loudly when it is absent."""
    global _loaded
    p = Path(path) if path else CUDA_LIB
    if _loaded is not None and Path(_loaded.path) == p:
        return _loaded
    if not p.exists():
        raise ImportError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (the CUDA extension is the only compute path)")
    lib = Library(str(p))
    _loaded = lib
    return lib


def context(device: int = 0, **kw) -> Context:
    return load_library().context(device, **kw)


__all__ = ["api", "Config", "Context", "CudaError", "DegenerateError", "InvalidArgument",
           "CapacityError", "Library", "RoadModel", "Threshold", "model", "load_library",
           "context", "CUDA_LIB", "SYNTH_LIB"]

"""BASELINE.json configurations: seeded synthetic scenes + pipeline settings.

The paper's datasets and KITTI are not available; these seeded synthetic
inputs with the BASELINE shapes, disparity ranges, roll angles and pothole
statistics stand in for them.  Scenes come from
synth/rpd_synth.cpp (built into _lib/librpd_synth.so).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import SYNTH_LIB

DEG = math.pi / 180.0
SEED_BASE = 20121080


class SceneParams(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("seed", C.c_uint64),
        ("texture", C.c_int32), ("d_min", C.c_double), ("d_max", C.c_double),
        ("quad_share", C.c_double), ("phi", C.c_double), ("n_potholes", C.c_int32),
        ("axis_min", C.c_double), ("axis_max", C.c_double), ("depth_min", C.c_double),
        ("depth_max", C.c_double), ("centred", C.c_int32), ("n_cracks", C.c_int32),
        ("crack_w_min", C.c_double), ("crack_w_max", C.c_double),
        ("crack_depth_min", C.c_double), ("crack_depth_max", C.c_double),
        ("noise_sigma", C.c_double), ("margin", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


@dataclass
class Scene:
    left: np.ndarray   # uint8 H x W
    right: np.ndarray  # uint8 H x W
    gt_disparity: np.ndarray
    gt_mask: np.ndarray
    params: dict


# Pipeline overrides per config (everything else = config.hpp defaults).
# D = disparity range -> d_max = D - 1 (the bootstrap pass uses (d_max+1)/2).
PIPELINE = {
    1: dict(d_max=63, sgm_paths=4, lambda1=10.0, lambda2=120.0, superpixels=300,
            slic_iterations=10),
    2: dict(d_max=127, sgm_paths=8, lambda1=10.0, lambda2=120.0, superpixels=2000),
    3: dict(d_max=127, sgm_paths=8, lambda1=10.0, lambda2=120.0, superpixels=1365),
    4: dict(d_max=255, sgm_paths=8, lambda1=10.0, lambda2=120.0, superpixels=8000,
            slic_iterations=10),
    5: dict(d_max=127, sgm_paths=8, lambda1=10.0, lambda2=120.0, superpixels=2000),
}
SHAPES = {1: (240, 320), 2: (800, 1312), 3: (1024, 1280), 4: (1080, 1920), 5: (800, 1312)}
FRAMES = {1: 1, 2: 1, 3: 64, 4: 1, 5: 4096}


def seed_of(config: int, frame: int) -> int:
    return SEED_BASE + 1000 * config + frame


def scene_params(config: int, frame: int = 0) -> SceneParams:
    h, w = SHAPES[config]
    seed = seed_of(config, frame)
    p = SceneParams()
    p.width, p.height, p.seed = w, h, seed
    p.quad_share = 0.25
    p.margin = 40
    p.crack_w_min, p.crack_w_max, p.crack_depth_min, p.crack_depth_max = 3.0, 6.0, 1.0, 2.0
    if config == 1:
        p.texture, p.d_min, p.d_max, p.phi = 0, 8.0, 40.0, 2.0 * DEG
        p.n_potholes, p.centred = 1, 1
        p.axis_min, p.axis_max, p.depth_min, p.depth_max = 20.0, 30.0, 4.0, 4.0
        p.noise_sigma = 2.0
    elif config in (2, 5):
        p.texture, p.d_min, p.d_max, p.phi = 1, 20.0, 110.0, 3.0 * DEG
        p.n_potholes, p.axis_min, p.axis_max, p.depth_min, p.depth_max = 3, 30.0, 120.0, 3.0, 8.0
        p.noise_sigma = 3.0
    elif config == 3:
        rng = np.random.default_rng(seed)
        p.texture = 1
        p.d_min = float(rng.uniform(20.0, 40.0))
        p.d_max = float(rng.uniform(80.0, 110.0))
        p.phi = float(rng.uniform(-5.0, 5.0)) * DEG
        p.n_potholes = int(rng.integers(0, 6))
        p.axis_min, p.axis_max, p.depth_min, p.depth_max = 20.0, 100.0, 2.0, 8.0
        p.noise_sigma = 3.0
    elif config == 4:
        p.texture, p.d_min, p.d_max, p.phi = 1, 30.0, 230.0, 4.0 * DEG
        p.n_potholes, p.axis_min, p.axis_max, p.depth_min, p.depth_max = 6, 30.0, 120.0, 3.0, 8.0
        p.n_cracks = 20
        p.noise_sigma = 3.0
    else:
        raise ValueError(f"unknown config {config}")
    return p


_lib = None


def _synth():
    global _lib
    if _lib is None:
        if not SYNTH_LIB.exists():
            raise ImportError(f"{SYNTH_LIB} not built (run __graft_entry__.build())")
        _lib = C.CDLL(str(SYNTH_LIB))
        _lib.rpd_synth_scene.restype = C.c_int
        _lib.rpd_synth_scene.argtypes = [C.POINTER(SceneParams), C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
    return _lib


def make_scene(config: int, frame: int = 0, params: SceneParams | None = None) -> Scene:
    p = params if params is not None else scene_params(config, frame)
    h, w = p.height, p.width
    left = np.empty((h, w), np.uint8)
    right = np.empty((h, w), np.uint8)
    gt = np.empty((h, w), np.float32)
    mask = np.empty((h, w), np.int32)
    rc = _synth().rpd_synth_scene(C.byref(p), left.ctypes.data, right.ctypes.data,
                                  gt.ctypes.data, mask.ctypes.data)
    if rc != 0:
        raise ValueError("rpd_synth_scene: bad parameters")
    return Scene(left, right, gt, mask, p.as_dict())


def small_scene(h: int, w: int, seed: int, *, d_min=6.0, d_max=30.0, phi_deg=2.0, potholes=2,
                texture=0, noise=2.0, depth=(4.0, 6.0), axes=(15.0, 40.0)) -> Scene:
    """A reduced-size scene with the config-1 recipe (for fast parity tests)."""
    p = SceneParams()
    p.width, p.height, p.seed = w, h, seed
    p.texture, p.d_min, p.d_max, p.phi = texture, d_min, d_max, phi_deg * DEG
    p.quad_share = 0.25
    p.n_potholes = potholes
    p.axis_min, p.axis_max = axes
    p.depth_min, p.depth_max = depth
    p.noise_sigma = noise
    p.margin = 20
    return make_scene(0, 0, p)


def pipeline_config(lib, config: int):
    return lib.default_config(**PIPELINE[config])

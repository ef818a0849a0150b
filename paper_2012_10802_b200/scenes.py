"""The reference's synthetic-scene API (synth.hpp:1-64).

`generate_scene` / `scene_batch` run on the device through the C-ABI
(abi_synth.cu) and reproduce the reference's scenes exactly: same
std::mt19937 streams, same float / double expression order.  `write_scene` /
`load_scene` are the scene-directory I/O of synth.cpp:198-260 (PNG via
image_io.py).  This is distinct from synth.py, the BASELINE-config generator
used by the benchmark.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np

from . import image_io
from .api import BatchRangesC, PotholeSpecC, SceneSpecC, StereoRig


@dataclass
class PotholeSpec:
    """synth.hpp:12-18."""
    cu: float = 0.0
    cv: float = 0.0
    ru: float = 10.0
    rv: float = 10.0
    depth: float = 2.0


@dataclass
class Rig:
    """StereoRig, types.hpp:25-30."""
    focal: float = 700.0
    baseline: float = 0.12
    cu: float = 0.0
    cv: float = 0.0


@dataclass
class SceneSpec:
    """synth.hpp:20-30."""
    width: int = 640
    height: int = 480
    rig: Rig = field(default_factory=Rig)
    a0: float = 5.0
    a1: float = 0.08
    phi_true: float = 0.0
    potholes: List[PotholeSpec] = field(default_factory=list)
    texture_seed: int = 1
    noise_sigma: float = 0.0


@dataclass
class BatchRanges:
    """synth.hpp:45-53."""
    depth_min: float = 1.5
    depth_max: float = 4.0
    radius_min: float = 22.0
    radius_max: float = 48.0
    a0_min: float = 4.0
    a0_max: float = 7.0
    a1_min: float = 0.07
    a1_max: float = 0.09
    phi_abs_max: float = 0.035
    noise_sigma: float = 0.0
    margin: int = 40


@dataclass
class SceneTruth:
    """synth.hpp:32-38."""
    left: np.ndarray
    right: np.ndarray
    gt_disparity: np.ndarray
    gt_mask: np.ndarray
    spec: SceneSpec


def generate_scene(ctx, spec: SceneSpec) -> SceneTruth:
    """synth.hpp:43 / synth.cpp:94-149."""
    left, right, gt, mask = ctx.generate_scene(spec)
    return SceneTruth(left, right, gt, mask, dataclasses.replace(spec))


def _spec_from_c(cs: SceneSpecC) -> SceneSpec:
    pots = [PotholeSpec(cs.potholes[i].cu, cs.potholes[i].cv, cs.potholes[i].ru,
                        cs.potholes[i].rv, cs.potholes[i].depth) for i in range(cs.n_potholes)]
    r = cs.rig
    return SceneSpec(cs.width, cs.height, Rig(r.focal, r.baseline, r.cu, r.cv), cs.a0, cs.a1,
                     cs.phi_true, pots, cs.texture_seed, cs.noise_sigma)


def batch_spec(lib, base_seed: int, index: int, ranges: Optional[BatchRanges] = None) -> SceneSpec:
    """The spec of scene `index` of scene_batch (synth.cpp:151-192); host only."""
    r = ranges or BatchRanges()
    rc = BatchRangesC(*[getattr(r, f.name) for f in dataclasses.fields(BatchRanges)])
    cs = SceneSpecC()
    pots = (PotholeSpecC * 3)()
    st = lib.dll.rpd_scene_batch_spec(C.c_uint32(base_seed & 0xFFFFFFFF), index, C.byref(rc),
                                      C.byref(cs), pots)
    if st != 0:
        raise ValueError("scene_batch: bad arguments")
    return _spec_from_c(cs)


def scene_batch(ctx, count: int, base_seed: int,
                ranges: Optional[BatchRanges] = None) -> List[SceneTruth]:
    """synth.hpp:56-57: scene i uses seed base_seed + i and 1-3 potholes."""
    if count < 1:
        raise ValueError("scene_batch: count must be >= 1")
    return [generate_scene(ctx, batch_spec(ctx.lib, base_seed, i, ranges)) for i in range(count)]


def write_scene(scene: SceneTruth, directory, ctx) -> None:
    """synth.cpp:198-226: left/right/disp_gt/mask_gt PNGs + spec.txt."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    image_io.save_gray_image(scene.left, d / "left.png", ctx)
    image_io.save_gray_image(scene.right, d / "right.png", ctx)
    image_io.save_disparity(scene.gt_disparity, d / "disp_gt.png", ctx)
    image_io.save_labels(scene.gt_mask, d / "mask_gt.png", ctx)
    s = scene.spec
    lines = [f"width={s.width}", f"height={s.height}", f"a0={_g(s.a0)}", f"a1={_g(s.a1)}",
             f"phi={_g(s.phi_true)}", f"seed={s.texture_seed}", f"noise_sigma={_g(s.noise_sigma)}",
             f"focal={_g(s.rig.focal)}", f"baseline={_g(s.rig.baseline)}", f"cu={_g(s.rig.cu)}",
             f"cv={_g(s.rig.cv)}", f"potholes={len(s.potholes)}"]
    for i, p in enumerate(s.potholes):
        lines.append(f"pothole{i}={_g(p.cu)},{_g(p.cv)},{_g(p.ru)},{_g(p.rv)},{_g(p.depth)}")
    (d / "spec.txt").write_text("\n".join(lines) + "\n")


def _g(x: float) -> str:
    """operator<< on a double with the default precision 6 (%g)."""
    return "%g" % x


def load_scene(directory, ctx) -> SceneTruth:
    """synth.cpp:228-260."""
    d = Path(directory)
    left = image_io.load_gray_image(d / "left.png", ctx)
    right = image_io.load_gray_image(d / "right.png", ctx)
    gt = image_io.load_disparity(d / "disp_gt.png", ctx)
    mask = image_io.load_labels(d / "mask_gt.png")
    p = d / "spec.txt"
    if not p.exists():
        raise RuntimeError(f"not found: {p}")
    s = SceneSpec()
    n_potholes = 0
    for line in p.read_text().splitlines():
        if "=" not in line:
            continue
        key, value = line.split("=", 1)
        if key == "width":
            s.width = int(value)
        elif key == "height":
            s.height = int(value)
        elif key == "a0":
            s.a0 = float(value)
        elif key == "a1":
            s.a1 = float(value)
        elif key == "phi":
            s.phi_true = float(value)
        elif key == "seed":
            s.texture_seed = int(value)
        elif key == "noise_sigma":
            s.noise_sigma = float(value)
        elif key == "focal":
            s.rig.focal = float(value)
        elif key == "baseline":
            s.rig.baseline = float(value)
        elif key == "cu":
            s.rig.cu = float(value)
        elif key == "cv":
            s.rig.cv = float(value)
        elif key == "potholes":
            n_potholes = int(value)
        elif key.startswith("pothole"):
            cu, cv, ru, rv, depth = (float(x) for x in value.split(","))
            s.potholes.append(PotholeSpec(cu, cv, ru, rv, depth))
    if len(s.potholes) != n_potholes:
        raise RuntimeError(f"corrupt spec.txt in {d}")
    return SceneTruth(left, right, gt, mask, s)


__all__ = ["PotholeSpec", "Rig", "SceneSpec", "BatchRanges", "SceneTruth", "generate_scene",
           "batch_spec", "scene_batch", "write_scene", "load_scene", "StereoRig"]

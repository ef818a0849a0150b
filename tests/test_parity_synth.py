"""Device scene generator vs the CPU oracle: bit-exact
left / right / truth disparity / mask on the same specs, and the batched
device entry point equal to one-at-a-time generation."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2012_10802_b200.scenes import (BatchRanges, PotholeSpec, SceneSpec, batch_spec,
                                          generate_scene)

pytestmark = pytest.mark.gpu

SPECS = [
    SceneSpec(),  # 640 x 480 defaults
    SceneSpec(width=160, height=120, texture_seed=42, phi_true=0.02, noise_sigma=2.0,
              potholes=[PotholeSpec(80.0, 60.0, 18.0, 12.0, 3.0)]),
    SceneSpec(width=97, height=61, texture_seed=7, a0=9.0, a1=0.05, phi_true=-0.04,
              noise_sigma=5.0,
              potholes=[PotholeSpec(30.0, 30.0, 10.0, 8.0, 2.0),
                        PotholeSpec(36.0, 33.0, 9.0, 6.0, 1.5)]),  # overlapping: last wins
    SceneSpec(width=5, height=3, texture_seed=3),
    SceneSpec(width=1312, height=800, texture_seed=20121080, a0=12.0, a1=0.09, phi_true=0.03,
              noise_sigma=3.0, potholes=[PotholeSpec(500.0, 600.0, 80.0, 40.0, 4.0)]),
]


def assert_same_scene(a, b):
    for name, x, y in zip(("left", "right", "gt_disparity", "gt_mask"), a, b):
        assert x.dtype == y.dtype and x.shape == y.shape, name
        diff = np.flatnonzero(x.view(np.uint32) != y.view(np.uint32)) if x.dtype != np.int32 \
            else np.flatnonzero(x != y)
        assert diff.size == 0, f"{name}: {diff.size} pixels differ, first {diff[:5]}"


@pytest.mark.parametrize("k", range(len(SPECS)))
def test_generate_scene_bit_exact(gpu, oracle, k):
    spec = SPECS[k]
    assert_same_scene(gpu.generate_scene(spec), oracle.generate_scene(spec))


def test_scene_batch_specs_and_scenes_match(gpu, oracle):
    ranges = BatchRanges(noise_sigma=1.5)
    for i in range(6):
        sg = batch_spec(gpu.lib, 7100, i, ranges)
        so = batch_spec(oracle.lib, 7100, i, ranges)
        assert sg == so
    for i in (0, 3):
        s = batch_spec(gpu.lib, 7100, i, ranges)
        assert_same_scene(gpu.generate_scene(s), oracle.generate_scene(s))


def test_generate_scenes_device_equals_single(gpu):
    import torch
    specs = [batch_spec(gpu.lib, 900, i, BatchRanges(noise_sigma=2.0 if i % 2 else 0.0))
             for i in range(3)]
    h, w = specs[0].height, specs[0].width
    dev = torch.device("cuda", 0)
    left = torch.empty((3, h, w), dtype=torch.float32, device=dev)
    right = torch.empty_like(left)
    gt = torch.empty_like(left)
    mask = torch.empty((3, h, w), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    gpu.generate_scenes_device(specs, left.data_ptr(), right.data_ptr(), gt.data_ptr(),
                               mask.data_ptr())
    for i, s in enumerate(specs):
        one = generate_scene(gpu, s)
        assert_same_scene((left[i].cpu().numpy(), right[i].cpu().numpy(), gt[i].cpu().numpy(),
                           mask[i].cpu().numpy()),
                          (one.left, one.right, one.gt_disparity, one.gt_mask))

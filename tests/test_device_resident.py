"""Device-resident C-ABI arguments (abi_util.hpp, pipeline.cu fetch): the
detect entry points, the evaluation metrics (evaluation.hpp:14-149), the
reprojections (road_geometry.cpp:153-228) and the image_io transforms take
device memory of the context's GPU wherever they take a host buffer, with
results identical to the host-buffer calls.  This is how a frame's outputs are
evaluated or reprojected without a host round trip."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2012_10802_b200.api import DetectOut
from paper_2012_10802_b200.synth import make_scene, pipeline_config

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def frame(cuda_lib):
    ctx = cuda_lib.context(0)
    sc = make_scene(1, 0)
    cfg = pipeline_config(cuda_lib, 1)
    host = ctx.detect(sc.left, sc.right, cfg)
    return ctx, sc, cfg, host


def test_detect_device_inputs_and_outputs(frame):
    ctx, sc, cfg, host = frame
    h, w = sc.left.shape
    dev = torch.device("cuda", 0)
    left = torch.from_numpy(sc.left).to(dev)
    right = torch.from_numpy(sc.right).to(dev)
    outs = {k: torch.empty((h, w), dtype=torch.float32, device=dev) for k in ("d0", "d1", "d2")}
    outs["labels"] = torch.empty((h, w), dtype=torch.int32, device=dev)
    o = DetectOut()
    for k, t in outs.items():
        setattr(o, k, C.cast(t.data_ptr(), C.POINTER(C.c_int32 if k == "labels" else C.c_float)))
    ctx.detect_raw(left.data_ptr(), right.data_ptr(), h, w, cfg, o)
    torch.cuda.synchronize()
    for k in ("d0", "d1", "d2"):
        assert np.array_equal(outs[k].cpu().numpy().view(np.uint32),
                              getattr(host, k).view(np.uint32)), k
    assert np.array_equal(outs["labels"].cpu().numpy(), host.labels)
    assert o.n_potholes == host.n_potholes


def test_evaluation_on_device_outputs(frame):
    ctx, sc, cfg, host = frame
    dev = torch.device("cuda", 0)
    d1 = torch.from_numpy(host.d1).to(dev)
    lab = torch.from_numpy(host.labels).to(dev)
    gt = torch.from_numpy(sc.gt_disparity.astype(np.float32)).to(dev)
    mask = torch.from_numpy(sc.gt_mask.astype(np.int32)).to(dev)
    assert ctx.pep(d1, gt, 3.0) == ctx.pep(host.d1, sc.gt_disparity, 3.0)
    assert ctx.rmse(d1, gt) == ctx.rmse(host.d1, sc.gt_disparity)
    a = ctx.pixel_metrics(lab, mask)
    b = ctx.pixel_metrics(host.labels, sc.gt_mask)
    assert (a.counts.n_tp, a.counts.n_fp, a.counts.n_fn, a.counts.n_tn) == \
        (b.counts.n_tp, b.counts.n_fp, b.counts.n_fn, b.counts.n_tn)
    assert a.fscore == b.fscore
    a = ctx.instance_metrics(lab, mask)
    b = ctx.instance_metrics(host.labels, sc.gt_mask)
    assert (a.correct, a.incorrect, a.misdetection) == (b.correct, b.incorrect, b.misdetection)


def test_reprojection_and_io_on_device_outputs(frame):
    ctx, sc, cfg, host = frame
    h, w = host.d1.shape
    dev = torch.device("cuda", 0)
    d1 = torch.from_numpy(host.d1).to(dev)
    lab = torch.from_numpy(host.labels).to(dev)
    rig = ctx.rig_from_config(cfg, w, h)
    n = int(host.labels.max())
    a = ctx.reproject_instances(d1, lab, n, rig)
    b = ctx.reproject_instances(host.d1, host.labels, n, rig)
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(ctx.reproject(d1, rig), ctx.reproject(host.d1, rig))
    assert np.array_equal(ctx.encode_disparity_u16(d1), ctx.encode_disparity_u16(host.d1))


def test_device_arrays_must_match_dtype(frame):
    ctx, _, _, host = frame
    d = torch.zeros((8, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        ctx.rmse(d, d)

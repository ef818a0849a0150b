"""Known answers of the reference on-disk format tests (SURVEY.md §8(f) row
3), both implementations of the per-pixel transforms: test_core_io.cpp:24-137
restated over paper_2012_10802_b200.image_io."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2012_10802_b200 import image_io as io
from paper_2012_10802_b200.api import DegenerateError

INV = -1.0


def test_pgm_round_trip_preserves_bytes(ctx, tmp_path):
    path = tmp_path / "small.pgm"
    path.write_bytes(b"P5\n2 2\n255\n" + bytes([0, 255, 128, 64]))
    img = io.load_gray_image(path, ctx)
    assert img.shape == (2, 2)
    assert img.tolist() == [[0.0, 255.0], [128.0, 64.0]]
    out = tmp_path / "small_out.pgm"
    io.save_gray_image(img, out, ctx)
    assert out.read_bytes() == path.read_bytes()


def test_missing_and_tiny(ctx, tmp_path):
    with pytest.raises(RuntimeError, match="not found"):
        io.load_gray_image("/nonexistent/image.png", ctx)
    tiny = tmp_path / "tiny.pgm"
    tiny.write_bytes(b"P5\n1 1\n255\n\x40")
    with pytest.raises(RuntimeError, match="too small"):
        io.load_gray_image(tiny, ctx)


def test_gray_png_round_trip(ctx, tmp_path):
    img = np.array([[17 * v + 5 * u for u in range(4)] for v in range(3)], np.float32)
    path = tmp_path / "gray.png"
    io.save_gray_image(img, path, ctx)
    assert np.array_equal(io.load_gray_image(path, ctx), img)


def test_disparity_encoding(ctx, tmp_path):
    m = np.array([[1.0, 50.0, INV], [0.5, 0.0, 255.5]], np.float32)
    path = tmp_path / "disp.png"
    io.save_disparity(m, path, ctx)
    back = io.load_disparity(path, ctx)
    assert back.tolist() == [[1.0, 50.0, INV], [0.5, INV, 255.5]]  # 0 encodes no-estimate
    assert ctx.encode_disparity_u16(m).tolist() == [[256, 12800, 0], [128, 0, 65408]]


def test_disparity_exact_for_multiples_of_1_256(ctx, tmp_path):
    rng = np.random.default_rng(7)
    m = (rng.integers(1, 65536, (16, 16)) / 256.0).astype(np.float32)
    path = tmp_path / "disp_rt.png"
    io.save_disparity(m, path, ctx)
    assert np.array_equal(io.load_disparity(path, ctx), m)


def test_disparity_overflow_and_8bit_rejected(ctx, tmp_path):
    with pytest.raises(DegenerateError, match="encoding range"):
        io.save_disparity(np.full((2, 2), 300.0, np.float32), tmp_path / "x.png", ctx)
    path = tmp_path / "gray8.png"
    io.save_gray_image(np.full((2, 2), 9.0, np.float32), path, ctx)
    with pytest.raises(RuntimeError, match="16-bit"):
        io.load_disparity(path, ctx)


def test_label_round_trip(ctx, tmp_path):
    labels = np.array([[0, 1], [512, 65535]], np.int32)
    path = tmp_path / "labels.png"
    io.save_labels(labels, path, ctx)
    assert np.array_equal(io.load_labels(path), labels)
    with pytest.raises(DegenerateError, match="encoding range"):
        ctx.encode_labels_u16(np.array([[70000]], np.int32))


def test_overlay(ctx, tmp_path):
    img = np.full((4, 4), 100.0, np.float32)
    labels = np.zeros((4, 4), np.int32)
    labels[1, 1] = 1
    labels[2, 2] = 13  # same palette slot as label 1
    assert io.overlay_palette(1) == io.overlay_palette(13)
    path = tmp_path / "overlay.png"
    io.save_overlay(img, labels, path, ctx)
    assert path.exists()
    rgb = ctx.overlay_rgb8(img, labels)
    assert rgb[0, 0].tolist() == [100, 100, 100]
    assert rgb[1, 1].tolist() == [165, 63, 88]  # round((100 + (230, 25, 75)) * 0.5)
    assert rgb[1, 1].tolist() == rgb[2, 2].tolist()
    with pytest.raises(DegenerateError):
        io.save_overlay(img, np.zeros((3, 3), np.int32), tmp_path / "bad.png", ctx)


def test_rgb_png_luminance(ctx, tmp_path):
    rgb = np.array([[[255, 0, 0], [0, 255, 0]], [[0, 0, 255], [10, 20, 30]]], np.uint8)
    path = tmp_path / "rgb.png"
    io._write_png(io.Raw(rgb.astype(np.uint16), 8), path)
    g = io.load_gray_image(path, ctx)
    exp = (np.float32(0.299) * rgb[..., 0].astype(np.float32) +
           np.float32(0.587) * rgb[..., 1].astype(np.float32) +
           np.float32(0.114) * rgb[..., 2].astype(np.float32))
    assert np.array_equal(g, exp.astype(np.float32))

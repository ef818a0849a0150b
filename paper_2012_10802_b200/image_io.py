"""On-disk formats of the reference (image_io.hpp / image_io.cpp:1-339;
SURVEY.md §8(f) row 3).

The per-pixel transforms (KITTI x256 disparity, 16-bit labels, 8-bit gray,
RGB luminance, overlay tint) run on the device through the C-ABI
(`Context.encode_disparity_u16`, ...); this module holds the file codecs
around them.  libpng is absent from the image, so PNG is a minimal codec over
zlib: writing emits unfiltered scanlines (8/16-bit gray, 8-bit RGB, like
the reference's writer); reading accepts non-interlaced 8/16-bit gray, gray +
alpha, RGB, RGBA and palette images with all five scanline filters, with the
reference's conversions (palette -> RGB, alpha stripped).  Binary PGM (P5,
8/16-bit) is read and written as image_io.cpp:42-110.  `.pgm` paths write PGM,
anything else PNG (:163-166).
"""
from __future__ import annotations

import struct
import zlib
from pathlib import Path

import numpy as np

_PNG_SIG = b"\x89PNG\r\n\x1a\n"


class Raw:
    """RawImage (image_io.cpp:16-26): samples (h, w, channels) uint16."""

    def __init__(self, samples: np.ndarray, bit_depth: int):
        self.samples = samples
        self.bit_depth = bit_depth

    @property
    def channels(self) -> int:
        return self.samples.shape[2]


# ---------------------------------------------------------------- PGM (P5) --
def _read_pgm(path) -> Raw:
    data = Path(path).read_bytes()
    pos = 2
    vals = []
    while len(vals) < 3:
        while pos < len(data) and (data[pos:pos + 1].isspace() or data[pos:pos + 1] == b"#"):
            if data[pos:pos + 1] == b"#":
                pos = data.index(b"\n", pos) + 1
            else:
                pos += 1
        end = pos
        while end < len(data) and data[end:end + 1].isdigit():
            end += 1
        if end == pos:
            raise RuntimeError(f"bad PGM header in {path}")
        vals.append(int(data[pos:end]))
        pos = end
    w, h, maxval = vals
    pos += 1  # single whitespace before the raster
    if w <= 0 or h <= 0:
        raise RuntimeError(f"zero-dimension image: {path}")
    n = w * h
    if maxval > 255:
        raw = np.frombuffer(data, ">u2", n, pos)
        bd = 16
    else:
        raw = np.frombuffer(data, np.uint8, n, pos)
        bd = 8
    if raw.size != n:
        raise RuntimeError(f"truncated PGM raster in {path}")
    return Raw(raw.astype(np.uint16).reshape(h, w, 1), bd)


def _write_pgm(raw: Raw, path) -> None:
    h, w = raw.samples.shape[:2]
    head = b"P5\n%d %d\n%d\n" % (w, h, 65535 if raw.bit_depth == 16 else 255)
    body = raw.samples[:, :, 0].astype(">u2" if raw.bit_depth == 16 else np.uint8).tobytes()
    Path(path).write_bytes(head + body)


# --------------------------------------------------------------------- PNG --
def _chunk(tag: bytes, payload: bytes) -> bytes:
    return (struct.pack(">I", len(payload)) + tag + payload +
            struct.pack(">I", zlib.crc32(tag + payload) & 0xFFFFFFFF))


def _write_png(raw: Raw, path) -> None:
    h, w, ch = raw.samples.shape
    color = 2 if ch == 3 else 0
    ihdr = struct.pack(">IIBBBBB", w, h, raw.bit_depth, color, 0, 0, 0)
    px = raw.samples.astype(">u2" if raw.bit_depth == 16 else np.uint8).reshape(h, -1)
    rows = np.concatenate([np.zeros((h, 1), np.uint8), px.view(np.uint8).reshape(h, -1)], 1)
    Path(path).write_bytes(_PNG_SIG + _chunk(b"IHDR", ihdr) +
                           _chunk(b"IDAT", zlib.compress(rows.tobytes(), 6)) +
                           _chunk(b"IEND", b""))


def _unfilter(data: bytes, h: int, stride: int, bpp: int) -> np.ndarray:
    buf = np.frombuffer(data, np.uint8)
    if buf.size < h * (stride + 1):
        raise RuntimeError("truncated PNG data")
    buf = buf[: h * (stride + 1)].reshape(h, stride + 1)
    out = np.zeros((h, stride), np.uint8)
    prev = np.zeros(stride, np.int32)
    for y in range(h):
        f, line = buf[y, 0], buf[y, 1:].astype(np.int32)
        if f == 0:
            cur = line
        elif f == 2:  # Up
            cur = (line + prev) & 0xFF
        elif f == 1:  # Sub: prefix sums with stride bpp
            cur = np.empty(stride, np.int32)
            for c in range(bpp):
                cur[c::bpp] = np.cumsum(line[c::bpp]) & 0xFF
        else:  # Average / Paeth: sequential along the row
            cur = np.zeros(stride, np.int32)
            for x in range(stride):
                a = cur[x - bpp] if x >= bpp else 0
                b = prev[x]
                if f == 3:
                    p = (a + b) >> 1
                else:
                    c = prev[x - bpp] if x >= bpp else 0
                    pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                    p = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
                cur[x] = (line[x] + p) & 0xFF
        out[y] = cur
        prev = cur
    return out


def _read_png(path) -> Raw:
    data = Path(path).read_bytes()
    if data[:8] != _PNG_SIG:
        raise RuntimeError(f"failed to decode PNG: {path}")
    pos, idat, plte = 8, [], None
    w = h = bd = color = interlace = None
    while pos < len(data):
        (ln,) = struct.unpack(">I", data[pos:pos + 4])
        tag, payload = data[pos + 4:pos + 8], data[pos + 8:pos + 8 + ln]
        pos += 12 + ln
        if tag == b"IHDR":
            w, h, bd, color, _, _, interlace = struct.unpack(">IIBBBBB", payload)
        elif tag == b"PLTE":
            plte = np.frombuffer(payload, np.uint8).reshape(-1, 3)
        elif tag == b"IDAT":
            idat.append(payload)
        elif tag == b"IEND":
            break
    if w is None or interlace:
        raise RuntimeError(f"failed to decode PNG: {path}")
    ch = {0: 1, 2: 3, 3: 1, 4: 2, 6: 4}[color]
    if bd not in (8, 16) and not (color in (0, 3) and bd in (1, 2, 4)):
        raise RuntimeError(f"unsupported bit depth in {path}")
    bits = bd * ch
    stride = (w * bits + 7) // 8
    rows = _unfilter(zlib.decompress(b"".join(idat)), h, stride, max(1, bits // 8))
    if bd == 16:
        s = rows.view(">u2").reshape(h, w, ch).astype(np.uint16)
    elif bd == 8:
        s = rows.reshape(h, w, ch).astype(np.uint16)
    else:  # 1/2/4-bit gray or palette indices
        per = 8 // bd
        bitsarr = np.unpackbits(rows, axis=1).reshape(h, -1, bd)
        vals = np.zeros(bitsarr.shape[:2], np.uint16)
        for k in range(bd):
            vals = (vals << 1) | bitsarr[:, :, k]
        s = vals[:, :w].reshape(h, w, 1)
        if color == 0:  # png_set_expand_gray_1_2_4_to_8
            s = s * (255 // ((1 << bd) - 1))
        del per
    if color == 3:  # png_set_palette_to_rgb
        if plte is None:
            raise RuntimeError(f"failed to decode PNG: {path}")
        s = plte[s[:, :, 0]].astype(np.uint16)
        bd = 8
    elif color in (4, 6):  # png_set_strip_alpha
        s = s[:, :, : ch - 1]
    if bd < 8:
        bd = 8
    return Raw(np.ascontiguousarray(s), bd)


def _read_any(path) -> Raw:
    p = Path(path)
    if not p.exists():
        raise RuntimeError(f"not found: {path}")
    return _read_pgm(p) if p.read_bytes()[:2] == b"P5" else _read_png(p)


def _write_any(raw: Raw, path) -> None:
    (_write_pgm if str(path).endswith(".pgm") else _write_png)(raw, path)


# ------------------------------------------------------ image_io.hpp API --
def load_gray_image(path, ctx) -> np.ndarray:
    """image_io.cpp:171-185 (RGB -> 0.299 R + 0.587 G + 0.114 B on the device)."""
    raw = _read_any(path)
    if raw.bit_depth != 8:
        raise RuntimeError(f"unsupported bit depth for gray image: {path}")
    h, w = raw.samples.shape[:2]
    if w < 2 or h < 2:
        raise RuntimeError(f"image too small: {path}")
    if raw.channels == 3:
        return ctx.gray_from_rgb8(raw.samples.astype(np.uint8))
    return raw.samples[:, :, 0].astype(np.float32)


def save_gray_image(img, path, ctx) -> None:
    """image_io.cpp:187-199."""
    _write_any(Raw(ctx.encode_gray_u8(img)[:, :, None].astype(np.uint16), 8), path)


def load_disparity(path, ctx) -> np.ndarray:
    """image_io.cpp:202-213: stored / 256, 0 = no estimate."""
    raw = _read_any(path)
    if raw.bit_depth != 16 or raw.channels != 1:
        raise RuntimeError(f"disparity file must be 16-bit single channel: {path}")
    return ctx.decode_disparity_u16(raw.samples[:, :, 0])


def save_disparity(disp, path, ctx) -> None:
    """image_io.cpp:215-235: round(d * 256), 0 = invalid."""
    _write_any(Raw(ctx.encode_disparity_u16(disp)[:, :, None], 16), path)


def load_labels(path) -> np.ndarray:
    """image_io.cpp:237-243."""
    raw = _read_any(path)
    if raw.channels != 1:
        raise RuntimeError(f"label file must be single channel: {path}")
    return raw.samples[:, :, 0].astype(np.int32)


def save_labels(labels, path, ctx) -> None:
    """image_io.cpp:245-259."""
    _write_any(Raw(ctx.encode_labels_u16(labels)[:, :, None], 16), path)


_PALETTE = ((230, 25, 75), (60, 180, 75), (255, 225, 25), (0, 130, 200), (245, 130, 48),
            (145, 30, 180), (70, 240, 240), (240, 50, 230), (210, 245, 60), (250, 190, 190),
            (0, 128, 128), (170, 110, 40))


def overlay_palette(label: int):
    """image_io.cpp:261-268 (C++ % semantics for label >= 1)."""
    return _PALETTE[(label - 1) % 12]


def save_overlay(img, labels, path, ctx) -> None:
    """image_io.cpp:291-312 (always PNG)."""
    rgb = ctx.overlay_rgb8(img, labels)
    _write_png(Raw(rgb.astype(np.uint16), 8), path)

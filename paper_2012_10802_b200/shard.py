"""Frame sharding across GPUs and streams.

Stereo frames are independent: there is no exchange step, hence no collective
on the data path.  Each rank (one process per GPU, launched by torchrun) owns
a fixed subset of the frames and processes them with its own rpd_ctx; only a
small per-frame summary travels to rank 0 at the end (gather_object).

Within a GPU, `StreamingRunner` keeps several frames in flight: every worker
thread owns a context (its own CUDA stream), so the upload, the pipeline and
the download of different frames overlap (ctypes releases the GIL inside the
library calls).  The reference's `rpd bench --workers` does the same with
std::async threads on the CPU (rpd_cli.cpp:293-302).
"""
from __future__ import annotations

import ctypes as C
import hashlib
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Iterable, List, Optional, Sequence

import numpy as np


def frames_for_rank(n_frames: int, rank: int, world: int, scheme: str = "round_robin"):
    """Frame ids owned by `rank`: round-robin (config 5 streaming) or
    contiguous blocks (config 3 batch)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if scheme == "round_robin":
        return list(range(rank, n_frames, world))
    if scheme == "block":
        per = (n_frames + world - 1) // world
        return list(range(rank * per, min(n_frames, (rank + 1) * per)))
    raise ValueError(f"unknown scheme {scheme}")


@dataclass
class FrameSummary:
    frame: int
    n_potholes: int
    labels_sha1: str
    fit: tuple
    stage_ms: dict = field(default_factory=dict)


def summarize(frame: int, res) -> FrameSummary:
    sha = hashlib.sha1(np.ascontiguousarray(res.labels).tobytes()).hexdigest()
    m = res.fit.model
    return FrameSummary(frame, int(res.n_potholes), sha, (m.a0, m.a1, m.phi),
                        dict(res.stage_ms))


class StreamingRunner:
    """Processes frames with `n_streams` concurrent contexts of one library.

    With the CUDA library every worker thread owns a context (its own CUDA
    stream) and two pinned host slots (rpd_host_alloc): while frame k runs on
    the device — its H2D copy enqueued asynchronously from slot k % 2 — the
    thread builds frame k + 1 into the other slot, then fetches k's outputs
    into pinned result buffers (BASELINE config 5: "pinned double-buffered
    host upload").  Libraries without the streaming extension (the CPU
    oracle) run plain synchronous detect calls per thread."""

    def __init__(self, lib, device: int = 0, n_streams: int = 2):
        self.lib = lib
        self.ctxs = [lib.context(device) for _ in range(max(1, n_streams))]

    def run(self, frame_ids: Sequence[int], make_frame: Callable[[int], tuple], cfg,
            want=("labels",)) -> List[FrameSummary]:
        out: List[Optional[FrameSummary]] = [None] * len(frame_ids)
        errors: list = []
        next_idx = [0]
        lock = threading.Lock()

        def take():
            with lock:
                i = next_idx[0]
                next_idx[0] += 1
            return i if i < len(frame_ids) else None

        def worker_sync(ctx):
            while (i := take()) is not None:
                left, right = make_frame(frame_ids[i])
                out[i] = summarize(frame_ids[i], ctx.detect(left, right, cfg, want=want))

        def worker_pinned(ctx):
            from .api import DetectOut, Threshold  # noqa: F401
            slots, outs = None, None
            i = take()
            if i is None:
                return
            left, right = make_frame(frame_ids[i])
            h, w = left.shape
            slots = [(self.lib.pinned_empty((h, w), np.uint8),
                      self.lib.pinned_empty((h, w), np.uint8)) for _ in range(2)]
            labels = self.lib.pinned_empty((h, w), np.int32)
            o = DetectOut()
            o.labels = labels.ctypes.data_as(C.POINTER(C.c_int32))
            cur = 0
            slots[cur][0][...] = left
            slots[cur][1][...] = right
            ctx.detect_async_host_u8(slots[cur][0].ctypes.data, slots[cur][1].ctypes.data, h, w,
                                     cfg)
            while True:
                j = take()
                if j is not None:  # build the next frame while this one runs
                    nl, nr = make_frame(frame_ids[j])
                    slots[1 - cur][0][...] = nl
                    slots[1 - cur][1][...] = nr
                ctx.fetch(o)
                out[i] = _summary_from_out(frame_ids[i], o, labels)
                if j is None:
                    return
                i, cur = j, 1 - cur
                ctx.detect_async_host_u8(slots[cur][0].ctypes.data, slots[cur][1].ctypes.data,
                                         h, w, cfg)

        pinned = getattr(self.lib, "has_streaming", False) and "rpd_detect_async_host_u8" \
            not in getattr(self.lib, "missing", ())

        def worker(ctx):
            try:
                (worker_pinned if pinned else worker_sync)(ctx)
            except Exception as e:  # surfaced after join
                errors.append(e)

        threads = [threading.Thread(target=worker, args=(c,)) for c in self.ctxs]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return [s for s in out if s is not None]


def _summary_from_out(frame: int, o, labels) -> FrameSummary:
    from .api import STAGE_NAMES
    sha = hashlib.sha1(np.ascontiguousarray(labels).tobytes()).hexdigest()
    m = o.fit.model
    return FrameSummary(frame, int(o.n_potholes), sha, (m.a0, m.a1, m.phi),
                        dict(zip(STAGE_NAMES, list(o.stage_ms))))


def run_sharded(lib, make_frame: Callable[[int], tuple], cfg, n_frames: int, rank: int,
                world: int, device: int = 0, n_streams: int = 2, scheme: str = "round_robin",
                group=None):
    """Each rank processes its frames; rank 0 returns every summary sorted by
    frame id (others return None).  Uses torch.distributed only to gather the
    small summaries."""
    mine = frames_for_rank(n_frames, rank, world, scheme)
    t0 = time.perf_counter()
    local = StreamingRunner(lib, device, n_streams).run(mine, make_frame, cfg)
    dt = time.perf_counter() - t0
    if world == 1:
        return sorted(local, key=lambda s: s.frame), [dt]
    import torch.distributed as dist
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((local, dt), gathered, dst=0, group=group)
    if rank != 0:
        return None, None
    allf = [s for part, _ in gathered for s in part]
    return sorted(allf, key=lambda s: s.frame), [t for _, t in gathered]

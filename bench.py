#!/usr/bin/env python
"""bench.py — stereo pothole detection (arxiv 2012.10802 pipeline) on B200.

Workload (default): BASELINE.json configs[4] ("cfg5"), the streaming run:
seeded 800x1312 uint8 stereo pairs from the config-2 generator (D=128:
d_max=127, bootstrap L=65 at half resolution, PT pass L=17; 8 SGM paths,
P1=10, P2=120, SLIC p=2000), frames round-robined across the ranks.  The
paper's datasets are unavailable: every frame is a distinct seeded synthetic
scene (paper_2012_10802_b200/synth.py, seed 20121080 + 1000*c + frame).
`--config 3` runs cfg3 (64 frames 1024x1280, contiguous blocks per rank),
`--config 1|2|4` the single-pair configs as replicas.

A step = F detect_potholes_pipeline runs (pipeline.cpp:47-109) per GPU on F
distinct frames of the rank's shard (a pool of up to --pool distinct frames,
pre-generated before timing and cycled): bootstrap SGM, road fit, PT SGM,
road refit, DT, SLIC + pooling, threshold, labelling.  A GPU keeps S pipeline
contexts (one CUDA stream + workspace + captured graph each) in flight.
N GPUs = N ranks, one process per GPU (torchrun; spawned by this script when
--gpus N > 1 and WORLD_SIZE is unset), no collective on the data path
(weak scaling; max-over-ranks timing).

  value   frames/s, frames resident in HBM, device time per step from CUDA
          events (start on a master stream every context stream waits on,
          end after all of them), L2 flushed (256 MiB write) between steps
          outside the events, max over ranks.
  value_serial  one frame at a time on one stream (the pass the per-stage
          times and the roofline come from).
  e2e     frames/s through the C-ABI call rpd_detect_u8 with pinned HOST
          buffers (S host threads, one context each): H2D of the pair, the
          pipeline, D2H of labels + d1 + d2 every call.
  roofline  the SGM path aggregation (dominant kernel): SURVEY.md §8(d)
          algorithmic bytes 2*(5P-2)*cells and ops 2*P*9*cells per frame over
          its CUDA-event time; peaks from MEASURED_PEAKS.json (HBM) and
          profiles/int_peak.json (tools/int_peak.cu, integer pipes).
  cpu_baseline  the LITERAL reference (untouched reference sources,
          oracle/_ref/librpd_ref.so) on all host cores, one distinct frame per
          thread; plus its 1-thread latency and StageClock stage times.

`--impl reference` times that CPU path alone and prints the same JSON line.
`--backend oracle` runs the multi-rank orchestration on CPU with the oracle
library and gloo (tests only; no GPU numbers).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes as C
import itertools
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# A frame server keeps many pipeline contexts (streams) in flight; the default
# 8 hardware work queues serialise their launches.  Must be set before CUDA
# initialises (measured: 16 contexts, 8 -> 32 queues, +4 % frames/s).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "stereo frames/s end-to-end and SGM GDE/s at 1/2/4/8 B200 vs CPU oracle"
ORACLE_LIB = ROOT / "oracle" / "_build" / "librpd_oracle.so"
REF_LIB = ROOT / "oracle" / "_ref" / "librpd_ref.so"
STAGES = ("sgm_bootstrap", "road_fit", "sgm_pt", "road_refit", "disparity_transform", "slic",
          "detect")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, help="BASELINE config index (1-5)")
    ap.add_argument("--streams", type=int, default=16,
                    help="concurrent pipeline contexts (one CUDA stream each) per GPU")
    ap.add_argument("--frames", type=int, default=0,
                    help="frames per step per GPU (0 = 2 x streams)")
    ap.add_argument("--pool", type=int, default=128,
                    help="distinct frames pre-generated per rank (cycled)")
    ap.add_argument("--cpu-threads", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the SURVEY §8(f) measurements (eval, reproject, scenes)")
    ap.add_argument("--backend", default="cuda", choices=["cuda", "oracle"],
                    help="oracle: CPU dry run of the orchestration (tests only)")
    ap.add_argument("--lib", default=None, help="A/B experiments: alternative product .so")
    ap.add_argument("--e2e-outputs", default="labels,d1,d2",
                    help="outputs copied back per e2e call (rpd_detect_out fields)")
    ap.add_argument("--e2e-threads", type=int, default=0, help="0 = --streams")
    ap.add_argument("--e2e-contexts", type=int, default=0,
                    help="pipeline contexts of the e2e run (0 = max(--streams, e2e threads)); more "
                         "contexts than threads: each thread streams several frames "
                         "(rpd_detect_async_host_u8 + rpd_detect_fetch)")
    return ap.parse_args(argv)


def env_rank():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: one process per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def int_peak():
    try:
        return json.loads((ROOT / "profiles" / "int_peak.json").read_text())
    except Exception:
        return None


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def gde_per_frame(h, w, cfg):
    """GDE: sum over passes of H_p * W_p * L_p."""
    if h >= 64 and w >= 64:
        boot = (h // 2) * (w // 2) * ((cfg.d_max + 1) // 2 + 1)
    else:
        boot = h * w * (cfg.d_max + 1)
    return boot + h * w * (cfg.d_max_pt + 1)


def workload_name(c, h, w, cfg, ids_total, scheme):
    return ("cfg%d: %dx%d uint8 pairs, D=%d, P=%d, P1=%g, P2=%g, SLIC p=%d; %s" % (
        c, h, w, cfg.d_max + 1, cfg.sgm_paths, cfg.lambda1, cfg.lambda2, cfg.superpixels,
        "%d distinct seeded frames, %s across ranks" % (ids_total, scheme) if ids_total > 1
        else "one pair, replicas on every rank"))


# ------------------------------------------------------------- frame sets --
def shard(config, rank, world):
    """Frame ids of this rank: cfg5 round-robin, cfg3
    contiguous blocks, single-pair configs replicated."""
    from paper_2012_10802_b200.shard import frames_for_rank
    from paper_2012_10802_b200.synth import FRAMES
    n = FRAMES[config]
    if n == 1:
        return [0], "replicas", 1
    scheme = "round_robin" if config == 5 else "block"
    return frames_for_rank(n, rank, world, scheme), scheme.replace("_", "-"), n


def make_pool(config, ids, threads):
    """Pre-generates the frames (host threads; the generator releases the GIL)."""
    from paper_2012_10802_b200.synth import make_scene

    def gen(i):
        sc = make_scene(config, i)
        return sc.left, sc.right
    with cf.ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        return list(ex.map(gen, ids))


# ----------------------------------------------------------- clock sampling --
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- CPU path ----
def cpu_lib():
    """The reference's own CPU implementation: the literal build when present
    (kind "reference"), else the restated oracle (kind "port")."""
    from paper_2012_10802_b200.api import Library
    if REF_LIB.exists():
        return Library(str(REF_LIB)), "reference"
    return Library(str(ORACLE_LIB)), "port"


def cpu_run(lib, config, pool, threads, offset=0, min_wall=0.0):
    """Rounds of one detect per host thread on pool frames (distinct where the
    config has several) until `min_wall` seconds have passed; returns
    (frames/s, wall s, frames, stage ms of the first frame)."""
    from paper_2012_10802_b200.synth import pipeline_config
    ctxs = [lib.context() for _ in range(threads)]
    cfg = pipeline_config(lib, config)
    out = [None] * threads
    rounds = [0]

    def work(j):
        left, right = pool[(offset + rounds[0] * threads + j) % len(pool)]
        out[j] = ctxs[j].detect(left, right, cfg, want=("labels",))

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        while True:
            list(ex.map(work, range(threads)))
            rounds[0] += 1
            if time.perf_counter() - t0 >= min_wall:
                break
    dt = time.perf_counter() - t0
    return rounds[0] * threads / dt, dt, rounds[0] * threads, out[0].stage_ms


def cpu_threads(args):
    return args.cpu_threads or (os.cpu_count() or 1)


def cpu_baseline(args, config, pool):
    lib, kind = cpu_lib()
    thr = cpu_threads(args)
    fps, dt, frames, _ = cpu_run(lib, config, pool, thr, min_wall=2.0)
    t0 = time.perf_counter()
    _, _, _, stage = cpu_run(lib, config, pool, 1, offset=thr)
    lat = (time.perf_counter() - t0) * 1e3
    what = "distinct cfg%d frames" % config if len(pool) > 1 else "replicas of the cfg%d pair" % config
    return {"value": round(fps, 4), "unit": "frames/s", "cores": thr, "kind": kind,
            "sample": f"{frames} {what}, one per host thread at a time "
                      f"({dt:.1f} s wall, {dt * thr:.0f} core-s)",
            "cpu_model": cpu_model(), "latency_ms_1thread": round(lat, 1),
            "stage_ms_1thread": {k: round(v, 2) for k, v in stage.items()}}


# ---------------------------------------------------------------- GPU arm ---
class Dist:
    def __init__(self, world, backend, local):
        self.world = world
        self.dist = None
        if world > 1:
            import torch
            import torch.distributed as dist
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group("gloo")
            self.dist = dist
        self.backend = backend

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()
        if self.backend == "nccl" or (self.dist is None and self.backend == "cuda"):
            import torch
            torch.cuda.synchronize()

    def allmax(self, x):
        return self._reduce(x, "max")

    def allsum(self, x):
        return self._reduce(x, "sum")

    def _reduce(self, x, op):
        if self.dist is None:
            return x
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else
                             self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


def gpu_arm(args, rank, world, local):
    import numpy as np
    import torch

    import paper_2012_10802_b200 as pkg
    from paper_2012_10802_b200.api import DetectOut
    from paper_2012_10802_b200.synth import SHAPES, pipeline_config

    torch.cuda.set_device(local)
    D = Dist(world, "nccl", local)
    lib = pkg.load_library(args.lib) if args.lib else pkg.load_library()
    c = args.config
    h, w = SHAPES[c]
    cfg = pipeline_config(lib, c)
    gde = gde_per_frame(h, w, cfg)
    ids, scheme, ids_total = shard(c, rank, world)
    ids = ids[:max(1, args.pool)]
    host_threads = max(1, (os.cpu_count() or 1) // world)
    pool = make_pool(c, ids, host_threads)
    P = len(pool)
    n = h * w

    # ---- pool resident in HBM (value) and pinned host memory (e2e)
    left_h = torch.from_numpy(np.stack([p[0] for p in pool])).pin_memory()
    right_h = torch.from_numpy(np.stack([p[1] for p in pool])).pin_memory()
    left_d = left_h.cuda()
    right_d = right_h.cuda()
    lp = [left_d[i].data_ptr() for i in range(P)]
    rp = [right_d[i].data_ptr() for i in range(P)]

    # ---- serial pass: one frame at a time, aggregation events on
    ctx = lib.context(local)
    ctx.set_profiling(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for i in range(args.warmup):
        ctx.detect_async_u8(lp[i % P], rp[i % P], h, w, cfg)
        ctx.fetch()
    kernels = ctx.stats().kernels_last_frame
    clocks = Clocks(local)
    D.barrier()
    clocks.start()
    step_ms, agg_ms, agg_bytes, agg_cells, sgm_ms, npot = [], [], [], [], [], []
    stage_acc = [0.0] * len(STAGES)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for k in range(args.steps):
        i = k % P
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush, ordered before the frame, outside the events
        e0.record(stream)
        ctx.detect_async_u8(lp[i], rp[i], h, w, cfg)
        e1.record(stream)
        out = ctx.fetch()  # waits + checks the device status (not timed)
        step_ms.append(e0.elapsed_time(e1))
        st = ctx.stats()
        agg_ms.append(sum(st.sgm_agg_ms[j] for j in range(st.sgm_passes)))
        agg_bytes.append(sum(st.sgm_agg_alg_bytes[j] for j in range(st.sgm_passes)))
        agg_cells.append(sum(st.sgm_cells[j] for j in range(st.sgm_passes)))
        sgm_ms.append(out.stage_ms[0] + out.stage_ms[2])
        for j in range(len(STAGES)):
            stage_acc[j] += out.stage_ms[j]
        npot.append(out.n_potholes)
    serial_ms = D.allmax(sum(step_ms))
    value_serial = world * args.steps / (serial_ms / 1e3)
    sgm_total_ms = D.allmax(sum(sgm_ms))
    sgm_gdes = world * args.steps * gde / (sgm_total_ms / 1e3) / 1e9

    # ---- throughput: F distinct frames per step over S concurrent contexts
    S = max(1, args.streams)
    F = args.frames or 2 * S
    ctx.set_profiling(False)
    ctxs = [ctx] + [lib.context(local) for _ in range(S - 1)]
    streams = [torch.cuda.ExternalStream(c_.stream) for c_ in ctxs]
    master = torch.cuda.current_stream()
    for s_ in range(args.warmup):
        for i in range(F):
            f = (s_ * F + i) % P
            ctxs[i % S].detect_async_u8(lp[f], rp[f], h, w, cfg)
        for c_ in ctxs:
            c_.fetch()
    D.barrier()
    conc_ms = []
    for s_ in range(args.steps):
        flush.zero_()  # on the master stream, before e0
        e0.record(master)
        for st_ in streams:
            st_.wait_event(e0)
        for i in range(F):
            f = (s_ * F + i) % P
            ctxs[i % S].detect_async_u8(lp[f], rp[f], h, w, cfg)
        for st_ in streams:
            ev = torch.cuda.Event()
            ev.record(st_)
            master.wait_event(ev)
        e1.record(master)
        e1.synchronize()
        conc_ms.append(e0.elapsed_time(e1))
        for c_ in ctxs:
            npot.append(c_.fetch().n_potholes)  # checks every context's device status
    D.barrier()
    clk = clocks.stop()
    total_ms = D.allmax(sum(conc_ms))
    frames_done = D.allsum(args.steps * F)
    value = frames_done / (total_ms / 1e3)

    # ---- e2e through the C-ABI with pinned host buffers: S host threads, one
    # context each, every call = H2D pair + pipeline + D2H labels/d1/d2
    e2e_fields = [f for f in args.e2e_outputs.split(",") if f]
    ctype = {"labels": (torch.int32, C.c_int32), "sp_labels": (torch.int32, C.c_int32),
             "d0": (torch.float32, C.c_float), "d1": (torch.float32, C.c_float),
             "d2": (torch.float32, C.c_float), "d3": (torch.float32, C.c_float)}

    def make_out():
        o = DetectOut()
        bufs = []
        for name in e2e_fields:
            tdt, cdt = ctype[name]
            b = torch.empty(n, dtype=tdt).pin_memory()
            bufs.append(b)
            setattr(o, name, C.cast(b.data_ptr(), C.POINTER(cdt)))
        return o, bufs
    # Host threads: one per context when the host has the cores, else each
    # thread keeps several contexts in flight through the streaming C-ABI
    # (rpd_detect_async_host_u8: async H2D from pinned memory + the frame;
    # rpd_detect_fetch: D2H of the outputs), so a many-GPU box with few host
    # cores per rank is not measured as a host-thread limit.
    ET = args.e2e_threads or min(S, max(1, (os.cpu_count() or 1) // world))
    NE = args.e2e_contexts or max(S, ET)
    ectxs = ctxs[:NE] + [lib.context(local) for _ in range(max(0, NE - S))]
    outs = [make_out() for _ in ectxs]
    lhp = [left_h[i].data_ptr() for i in range(P)]
    rhp = [right_h[i].data_ptr() for i in range(P)]

    def e2e_run(nframes):
        # frames are handed out from one shared counter (a frame server's work
        # queue): host threads finish within about one frame of each other
        ticket = itertools.count()

        def work(j):
            mine = list(range(j, NE, ET))
            if len(mine) == 1:  # the synchronous call: H2D, frame, D2H
                c_ = mine[0]
                while True:
                    q = next(ticket)  # atomic under the GIL
                    if q >= nframes:
                        return
                    f = q % P
                    ectxs[c_].detect_raw(lhp[f], rhp[f], h, w, cfg, outs[c_][0])
            busy = []
            for c_ in mine:  # one frame in flight per context
                q = next(ticket)
                if q >= nframes:
                    break
                ectxs[c_].detect_async_host_u8(lhp[q % P], rhp[q % P], h, w, cfg)
                busy.append(c_)
            while busy:
                c_ = busy.pop(0)
                ectxs[c_].fetch(outs[c_][0])
                q = next(ticket)
                if q < nframes:
                    ectxs[c_].detect_async_host_u8(lhp[q % P], rhp[q % P], h, w, cfg)
                    busy.append(c_)
        ths = [threading.Thread(target=work, args=(j,)) for j in range(ET)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    total_frames = args.steps * F
    e2e_run(max(1, args.warmup) * NE)
    D.barrier()
    t0 = time.perf_counter()
    e2e_run(total_frames)
    e2e_s = D.allmax(time.perf_counter() - t0)
    D.barrier()
    e2e = D.allsum(total_frames) / e2e_s

    # ---- rooflines of the aggregation kernel
    pk = peaks()
    peak = pk.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json)" if peak else "fallback (B200_PROFILING.md)"
    peak = peak or 6650.0
    t_agg = sum(agg_ms) / 1e3
    achieved = (sum(agg_bytes) / 1e9) / t_agg
    traffic = None
    tf = ROOT / "profiles" / "agg_traffic.json"
    if tf.exists():
        try:
            # per config: both aggregation launches of one frame (ncu)
            traffic = json.loads(tf.read_text())["configs"][str(c)]["bytes_per_frame"]
        except Exception:
            traffic = None
    ops_agg = 2.0 * cfg.sgm_paths * 9.0 * sum(agg_cells)  # OPS_agg
    ip = int_peak()
    int_ops = None
    if ip:
        lane_peak = ip["iadd3"]["lane_ops_per_s"]
        simd_peak = ip["viaddmnmx_u16x2"]["cell_ops_per_s"]
        a_ops = ops_agg / t_agg
        int_ops = {"achieved_tops": round(a_ops / 1e12, 3),
                   "peak_tops": round(lane_peak / 1e12, 3),
                   "frac": round(a_ops / lane_peak, 4),
                   "peak_simd2_tops": round(simd_peak / 1e12, 3),
                   "frac_simd2": round(a_ops / simd_peak, 4),
                   "ops_per_frame": ops_agg / args.steps,
                   "peak_source": "profiles/int_peak.json (tools/int_peak.cu): IADD3 lane ops; "
                                  "simd2 = VIADDMNMX.U16x2 cell ops (2 halves x add+min)",
                   "note": "OPS_agg = 2*P*9 ops per cell (SURVEY §8(d)); the u16x2 DPX "
                           "recurrence packs two cells per lane, so frac can exceed 1"}

    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "value_serial": round(value_serial, 3),
        "scaling": "weak", "vs_baseline": None, "dtype": "u8/u16 (SGM), f32/f64 (fit, SLIC)",
        "data": "synthetic (seeded BASELINE cfg%d scenes, synth.py; paper datasets "
                "unavailable)" % c,
        "config": {"workload": workload_name(c, h, w, cfg, ids_total, scheme),
                   "frames_per_step_per_gpu": F, "streams_per_gpu": S,
                   "distinct_frames_per_rank": P, "frame_ids_rank0": [ids[0], ids[-1]],
                   "l2": "flushed (256 MiB write) between timed steps",
                   "cuda_device_max_connections":
                       os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"),
                   "parallelism": "independent frames: %d concurrent pipeline contexts per "
                                  "GPU, %d rank(s) = GPUs, no collective" % (S, world)},
        "sgm_gdes": round(sgm_gdes, 3),
        "gdes_pipeline": round(value * gde / 1e9, 3),
        "gde_per_frame": gde,
        "stage_ms": {k: round(v / args.steps, 4) for k, v in zip(STAGES, stage_acc)},
        "n_potholes_last": npot[-1] if npot else None,
        "e2e": {"value": round(e2e, 3), "unit": "frames/s", "h2d_bytes_per_step": 2 * n * F,
                "d2h_bytes_per_step": 4 * n * F * len(e2e_fields),
                "outputs": e2e_fields, "host_threads": ET, "contexts": NE},
        "gpu_launches": int(kernels * args.steps * F),
        "roofline": {"bound": "hbm", "kernel": "k_aggregate_tma (SGM path aggregation, 2P "
                                               "paths, both passes)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_src,
                     "dram_gbs_actual": round(traffic / 1e9 / (t_agg / args.steps), 1)
                     if traffic else None,
                     "agg_ms_per_frame": round(sum(agg_ms) / len(agg_ms), 4),
                     "alg_bytes_per_frame": agg_bytes[0] if agg_bytes else None,
                     "int_ops": int_ops,
                     "note": "achieved = SURVEY §8(d) algorithmic bytes / event time; the u8 "
                             "formulation moves ~1/3 of them (dram_gbs_actual = ncu DRAM "
                             "bytes of both launches / the same time)"},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_extras:
        result.update(widening_extras(args, ctx, pool[0], c, cfg, h, w))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, c, pool)
    if rank == 0:
        print(json.dumps(result), flush=True)
    D.close()


def widening_extras(args, ctx, frame, c, cfg, h, w):
    """SURVEY §8(f) rows measured through the C-ABI with host buffers."""
    import numpy as np
    import torch

    from paper_2012_10802_b200.synth import make_scene
    extra = {}
    # the first of the config's frames with detections (clouds to reproject)
    for fi in range(8):
        scene = make_scene(c, fi)
        res = ctx.detect(scene.left, scene.right, cfg, want=("d1", "labels"))
        if res.n_potholes > 0:
            break
    extra["frame"] = fi
    gt_d = scene.gt_disparity.astype(np.float32)

    def eval_all(c_):
        c_.pep(res.d1, gt_d, 3.0)
        c_.rmse(res.d1, gt_d)
        c_.pixel_metrics(res.labels, scene.gt_mask)
        return c_.instance_metrics(res.labels, scene.gt_mask)

    for _ in range(3):
        eval_all(ctx)
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        rep = eval_all(ctx)
    extra["eval"] = {"metrics": "pep(eps=3) + rmse of d1, pixel + instance metrics of labels",
                     "ms_per_frame_gpu_c_abi": round((time.perf_counter() - t0) * 1e3 / reps, 3),
                     "instance_report": [rep.correct, rep.incorrect, rep.misdetection]}
    # the same calls on device-resident buffers (a frame's outputs kept in HBM,
    # the ground truth uploaded once): no host round trip per call
    dv = torch.device("cuda", torch.cuda.current_device())
    dres = {"d1": torch.from_numpy(res.d1).to(dv), "labels": torch.from_numpy(res.labels).to(dv),
            "gt": torch.from_numpy(gt_d).to(dv),
            "mask": torch.from_numpy(np.ascontiguousarray(scene.gt_mask, np.int32)).to(dv)}

    def eval_dev(c_):
        c_.pep(dres["d1"], dres["gt"], 3.0)
        c_.rmse(dres["d1"], dres["gt"])
        c_.pixel_metrics(dres["labels"], dres["mask"])
        return c_.instance_metrics(dres["labels"], dres["mask"])
    for _ in range(3):
        eval_dev(ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        rep_d = eval_dev(ctx)
    extra["eval"]["ms_per_frame_gpu_device_resident"] = \
        round((time.perf_counter() - t0) * 1e3 / reps, 3)
    assert (rep_d.correct, rep_d.incorrect, rep_d.misdetection) == \
        (rep.correct, rep.incorrect, rep.misdetection)
    rig = ctx.rig_from_config(cfg, w, h)
    n_pot = int(res.labels.max())

    def clouds(c_):
        return c_.reproject_instances(res.d1, res.labels, n_pot, rig)
    clouds(ctx)
    t0 = time.perf_counter()
    for _ in range(reps):
        pts = clouds(ctx)
    extra["reproject"] = {"clouds": n_pot, "points": int(sum(len(p) for p in pts)),
                          "ms_per_frame_gpu_c_abi":
                              round((time.perf_counter() - t0) * 1e3 / reps, 3)}
    ctx.reproject_instances(dres["d1"], dres["labels"], n_pot, rig)
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.reproject_instances(dres["d1"], dres["labels"], n_pot, rig)
    extra["reproject"]["ms_per_frame_gpu_device_resident"] = \
        round((time.perf_counter() - t0) * 1e3 / reps, 3)
    from paper_2012_10802_b200.scenes import BatchRanges, batch_spec
    nb = 20
    sb = {}
    for sigma in (0.0, 2.0):
        specs = [batch_spec(ctx.lib, 7100, i, BatchRanges(noise_sigma=sigma)) for i in range(nb)]
        sh, sw = specs[0].height, specs[0].width
        dv = torch.device("cuda", 0)
        bl = torch.empty((nb, sh, sw), dtype=torch.float32, device=dv)
        br, bg = torch.empty_like(bl), torch.empty_like(bl)
        bm = torch.empty((nb, sh, sw), dtype=torch.int32, device=dv)
        torch.cuda.synchronize()
        for _ in range(2):
            ctx.generate_scenes_device(specs, bl.data_ptr(), br.data_ptr(), bg.data_ptr(),
                                       bm.data_ptr())
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.generate_scenes_device(specs, bl.data_ptr(), br.data_ptr(), bg.data_ptr(),
                                       bm.data_ptr())
        sb["noise%g" % sigma] = round(nb * reps / (time.perf_counter() - t0), 1)
    acfg = ctx.lib.default_config(delta_pd=0.48, superpixels=2400)
    per = sh * sw * 4
    for i in range(2):
        ctx.detect_async(bl.data_ptr() + i * per, br.data_ptr() + i * per, sh, sw, acfg)
        ctx.fetch()
    t0 = time.perf_counter()
    ctx.generate_scenes_device(specs, bl.data_ptr(), br.data_ptr(), bg.data_ptr(), bm.data_ptr())
    for i in range(nb):
        ctx.detect_async(bl.data_ptr() + i * per, br.data_ptr() + i * per, sh, sw, acfg)
    ctx.fetch()
    extra["scenes"] = {"batch": "scene_batch(20, 7100), 640x480 (acceptance.cpp:221)",
                       "scenes_per_s_gpu": sb["noise0"], "scenes_per_s_gpu_noise2": sb["noise2"],
                       "generate_detect_stream_frames_per_s":
                           round(nb / (time.perf_counter() - t0), 1)}
    if ORACLE_LIB.exists() and not args.no_cpu_baseline:
        from paper_2012_10802_b200.api import Library
        octx = Library(str(ORACLE_LIB)).context()
        t0 = time.perf_counter()
        octx.generate_scene(specs[0])
        extra["scenes"]["scenes_per_s_oracle_1core_noise2"] = \
            round(1.0 / (time.perf_counter() - t0), 2)
        t0 = time.perf_counter()
        eval_all(octx)
        extra["eval"]["ms_per_frame_oracle_1core"] = round((time.perf_counter() - t0) * 1e3, 3)
        t0 = time.perf_counter()
        clouds(octx)
        extra["reproject"]["ms_per_frame_oracle_1core"] = \
            round((time.perf_counter() - t0) * 1e3, 3)
    return extra


# ------------------------------------------------- CPU dry run (tests) ------
def oracle_dry_run(args, rank, world):
    """The same sharding / max-over-ranks / JSON path with the CPU oracle
    library and gloo: exercises the multi-rank orchestration without a GPU.
    Its numbers are NOT GPU measurements (`backend` says so)."""
    from paper_2012_10802_b200.api import Library
    from paper_2012_10802_b200.synth import SHAPES, pipeline_config
    D = Dist(world, "gloo", 0)
    lib = Library(str(ORACLE_LIB))
    c = args.config
    h, w = SHAPES[c]
    cfg = pipeline_config(lib, c)
    ids, scheme, ids_total = shard(c, rank, world)
    ids = ids[:max(1, args.pool)]
    pool = make_pool(c, ids, 2)
    S = max(1, args.streams)
    F = args.frames or 2 * S
    ctxs = [lib.context() for _ in range(S)]
    import hashlib
    labels = []

    def step(s_):
        def work(j):
            for i in range(j, F, S):
                left, right = pool[(s_ * F + i) % len(pool)]
                r = ctxs[j].detect(left, right, cfg, want=("labels",))
                labels.append(hashlib.sha1(r.labels.tobytes()).hexdigest()[:8])
        with cf.ThreadPoolExecutor(max_workers=S) as ex:
            list(ex.map(work, range(S)))
    for s_ in range(args.warmup):
        step(s_)
    D.barrier()
    t0 = time.perf_counter()
    for s_ in range(args.steps):
        step(s_)
    dt = D.allmax(time.perf_counter() - t0)
    frames = D.allsum(args.steps * F)
    result = {"metric": METRIC, "value": round(frames / dt, 4), "unit": "frames/s",
              "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
              "ms_per_step": round(dt * 1e3 / args.steps, 3), "higher_is_better": True,
              "scaling": "weak", "backend": "oracle (CPU dry run of the orchestration; not a "
                                            "GPU measurement)",
              "config": {"workload": workload_name(c, h, w, cfg, ids_total, scheme),
                         "frames_per_step_per_gpu": F, "streams_per_gpu": S,
                         "distinct_frames_per_rank": len(pool)},
              "frames_processed": int(frames)}
    if D.dist is not None:
        gathered = [None] * world
        D.dist.all_gather_object(gathered, ids)
        result["frame_ids_per_rank"] = gathered
    else:
        result["frame_ids_per_rank"] = [ids]
    if rank == 0:
        print(json.dumps(result), flush=True)
    D.close()


# ---------------------------------------------------------- reference arm ---
def reference_arm(args, rank, world):
    """The reference's own CPU implementation on this box's host cores, on
    the same config / metric / unit as the GPU arm: each step = one distinct
    frame per host thread.  Rank 0 only."""
    if rank != 0:
        return
    from paper_2012_10802_b200.synth import SHAPES, pipeline_config
    c = args.config
    h, w = SHAPES[c]
    lib, kind = cpu_lib()
    cfg = pipeline_config(lib, c)
    ids, scheme, ids_total = shard(c, 0, 1)
    thr = cpu_threads(args)
    pool = make_pool(c, ids[:max(thr, min(args.pool, len(ids)))], thr)
    for s_ in range(args.warmup):
        cpu_run(lib, c, pool, thr, offset=s_ * thr)
    tot_frames, tot_s = 0, 0.0
    for s_ in range(args.steps):
        _, dt, frames, _ = cpu_run(lib, c, pool, thr, offset=(args.warmup + s_) * thr,
                                   min_wall=0.5)
        tot_frames += frames
        tot_s += dt
    fps = tot_frames / tot_s
    result = {
        "impl": "reference", "metric": METRIC, "value": round(fps, 4), "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot_s / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (reference arithmetic)",
        "data": "synthetic (seeded BASELINE cfg%d scenes, synth.py)" % c,
        "config": {"workload": workload_name(c, h, w, cfg, ids_total, scheme),
                   "implementation": ("literal reference: untouched /root/reference/proj/src "
                                      "sources + Eigen shim (oracle/_ref/librpd_ref.so)")
                   if kind == "reference" else "CPU oracle restatement of the reference"},
        "sgm_gdes": None,
        "cpu_baseline": {"value": round(fps, 4), "unit": "frames/s", "cores": thr, "kind": kind,
                         "sample": f"per step >= {thr} %s, one per host thread at a time"
                                   % ("distinct cfg%d frames" % c if len(pool) > 1 else
                                      "replicas of the cfg%d pair" % c),
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(fps, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(result), flush=True)


def main():
    args = parse()
    rank, world, local = env_rank()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        reference_arm(args, rank, world)
    elif args.backend == "oracle":
        oracle_dry_run(args, rank, world)
    else:
        gpu_arm(args, rank, world, local)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — stereo pothole detection (arxiv 2012.10802 pipeline) on B200.

Workload: BASELINE.json configs[1] ("cfg2"): one 800x1312 uint8 stereo pair,
D=128 (d_max=127, bootstrap L=65 at half resolution, PT pass L=17), 8 SGM
paths, P1=10, P2=120, SLIC p=2000.  Seeded synthetic scene (the paper's
datasets are not available; paper_2012_10802_b200/synth.py).

A step = F full detect_potholes_pipeline runs (pipeline.cpp:47-109; default
F = 2 x streams) on the pair: bootstrap SGM, road fit, PT SGM, road refit,
DT, SLIC + pooling, threshold, labelling.  The frames are independent, so a
GPU keeps S pipeline contexts (one CUDA stream + workspace + captured graph
each) in flight, as a stream server would.  N GPUs = N independent ranks
(weak scaling, no collective on the data path).

  value  frames/s with the pair resident in HBM; device time per step from
         CUDA events (start on a master stream that every context stream
         waits on, end after all of them); L2 flushed (256 MiB write) between
         steps outside the timed events; max over ranks.
  value_serial  the same with one frame at a time on one stream (also the
         pass the per-stage times and the roofline come from).
  e2e    frames/s through the C-ABI call rpd_detect_u8 with pinned HOST
         buffers (S host threads, one context each): H2D of the pair, the
         pipeline, D2H of labels + d1 + d2 every call.
  roofline  the SGM path-aggregation kernel (dominant): SURVEY.md §8(d)
         algorithmic bytes 2*(5P-2)*cells per launch / its CUDA-event time
         in the serial pass.
  cpu_baseline  the CPU oracle (scalar restatement of the reference) on all
         host cores, one frame per thread.

`--impl reference` times that CPU path alone and prints the same JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "stereo frames/s end-to-end and SGM GDE/s at 1/2/4/8 B200 vs CPU oracle"
ORACLE_LIB = ROOT / "oracle" / "_build" / "librpd_oracle.so"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, help="BASELINE config index (1-5)")
    ap.add_argument("--cpu-threads", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=16,
                    help="concurrent pipeline contexts (one CUDA stream each) per GPU")
    ap.add_argument("--frames", type=int, default=0,
                    help="frames per step per GPU (0 = 2 x streams)")
    return ap.parse_args()


def env_rank():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def gde_per_frame(h, w, cfg):
    """Sum over passes of H_p * W_p * L_p."""
    if h >= 64 and w >= 64:
        boot = (h // 2) * (w // 2) * ((cfg.d_max + 1) // 2 + 1)
    else:
        boot = h * w * (cfg.d_max + 1)
    return boot + h * w * (cfg.d_max_pt + 1)


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


# --------------------------------------------------------------- CPU oracle --
def cpu_oracle_run(scene, cfg_fields, threads, frames_per_thread=1):
    """Oracle detect on `threads` host threads, one frame each; returns
    (frames/s, wall s, frames)."""
    from paper_2012_10802_b200.api import Library
    lib = Library(str(ORACLE_LIB))
    ctxs = [lib.context() for _ in range(threads)]
    cfg = lib.default_config(**cfg_fields)
    errors = []

    def work(c):
        try:
            for _ in range(frames_per_thread):
                c.detect(scene.left, scene.right, cfg, want=("labels",))
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=work, args=(c,)) for c in ctxs]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    if errors:
        raise errors[0]
    frames = threads * frames_per_thread
    return frames / dt, dt, frames


def cpu_threads(args):
    return args.cpu_threads or (os.cpu_count() or 1)


# ---------------------------------------------------------------- GPU arm ---
def gpu_arm(args, rank, world, local):
    import numpy as np
    import torch

    import paper_2012_10802_b200 as pkg
    from paper_2012_10802_b200.api import Center, DetectOut
    from paper_2012_10802_b200.synth import PIPELINE, SHAPES, make_scene, pipeline_config

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    lib = pkg.load_library()
    ctx = lib.context(local)
    c = args.config
    h, w = SHAPES[c]
    scene = make_scene(c, 0)  # replicas of the config's pair on every rank
    cfg = pipeline_config(lib, c)
    override = os.environ.get("RPD_BENCH_CFG")  # experiments only: "key=value,..." (marked in config)
    if override:
        for kv in override.split(","):
            k, v = kv.split("=")
            setattr(cfg, k, type(getattr(cfg, k))(v))
    gde = gde_per_frame(h, w, cfg)

    # ---- device-resident value
    left_d = torch.from_numpy(scene.left).cuda()
    right_d = torch.from_numpy(scene.right).cuda()
    ctx.set_profiling(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        ctx.detect_async_u8(left_d.data_ptr(), right_d.data_ptr(), h, w, cfg)
        ctx.fetch()
    kernels = ctx.stats().kernels_last_frame
    clocks = Clocks(local)
    barrier()
    clocks.start()
    step_ms, agg_ms, agg_bytes, sgm_ms, npot = [], [], [], [], []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush, ordered before the step, outside the events
        e0.record(stream)
        ctx.detect_async_u8(left_d.data_ptr(), right_d.data_ptr(), h, w, cfg)
        e1.record(stream)
        out = ctx.fetch()  # waits + checks the device status (not timed)
        step_ms.append(e0.elapsed_time(e1))
        st = ctx.stats()
        agg_ms.append(sum(st.sgm_agg_ms[i] for i in range(st.sgm_passes)))
        agg_bytes.append(sum(st.sgm_agg_alg_bytes[i] for i in range(st.sgm_passes)))
        sgm_ms.append(out.stage_ms[0] + out.stage_ms[2])
        npot.append(out.n_potholes)
    serial_ms = allmax(sum(step_ms))
    value_serial = world * args.steps / (serial_ms / 1e3)
    sgm_total_ms = allmax(sum(sgm_ms))
    sgm_gdes = world * args.steps * gde / (sgm_total_ms / 1e3) / 1e9

    # ---- throughput: F frames per step over S concurrent contexts (streams)
    S = max(1, args.streams)
    F = args.frames or 2 * S
    ctx.set_profiling(False)
    ctxs = [ctx] + [lib.context(local) for _ in range(S - 1)]
    streams = [torch.cuda.ExternalStream(c.stream) for c in ctxs]
    master = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for i in range(F):
            ctxs[i % S].detect_async_u8(left_d.data_ptr(), right_d.data_ptr(), h, w, cfg)
        for c_ in ctxs:
            c_.fetch()
    barrier()
    conc_ms = []
    for _ in range(args.steps):
        flush.zero_()  # on the master stream, before e0
        e0.record(master)
        for st_ in streams:
            st_.wait_event(e0)
        for i in range(F):
            ctxs[i % S].detect_async_u8(left_d.data_ptr(), right_d.data_ptr(), h, w, cfg)
        for st_ in streams:
            ev = torch.cuda.Event()
            ev.record(st_)
            master.wait_event(ev)
        e1.record(master)
        e1.synchronize()
        conc_ms.append(e0.elapsed_time(e1))
        for c_ in ctxs:
            npot.append(c_.fetch().n_potholes)  # checks every context's device status
    barrier()
    clk = clocks.stop()
    total_ms = allmax(sum(conc_ms))
    value = world * args.steps * F / (total_ms / 1e3)

    # ---- e2e through the C-ABI with pinned host buffers: S host threads, one
    # context each, every call = H2D pair + pipeline + D2H labels/d1/d2
    n = h * w
    lh = torch.from_numpy(scene.left).pin_memory()
    rh = torch.from_numpy(scene.right).pin_memory()

    def make_out():
        bufs = (torch.empty(n, dtype=torch.int32).pin_memory(),
                torch.empty(n, dtype=torch.float32).pin_memory(),
                torch.empty(n, dtype=torch.float32).pin_memory())
        o = DetectOut()
        o.labels = C.cast(bufs[0].data_ptr(), C.POINTER(C.c_int32))
        o.d1 = C.cast(bufs[1].data_ptr(), C.POINTER(C.c_float))
        o.d2 = C.cast(bufs[2].data_ptr(), C.POINTER(C.c_float))
        return o, bufs
    outs = [make_out() for _ in ctxs]

    def e2e_run(frames_per_ctx):
        def work(j):
            for _ in range(frames_per_ctx[j]):
                ctxs[j].detect_raw(lh.data_ptr(), rh.data_ptr(), h, w, cfg, outs[j][0])
        ths = [threading.Thread(target=work, args=(j,)) for j in range(S)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    total_frames = args.steps * F
    per_ctx = [total_frames // S + (1 if j < total_frames % S else 0) for j in range(S)]
    e2e_run([max(1, args.warmup)] * S)
    barrier()
    t0 = time.perf_counter()
    e2e_run(per_ctx)
    e2e_s = allmax(time.perf_counter() - t0)
    barrier()
    e2e = world * total_frames / e2e_s

    # ---- roofline of the aggregation kernel
    pk = peaks()
    peak = pk.get("hbm_gbs")
    peak_src = "measured" if peak else "fallback"
    peak = peak or 6650.0
    achieved = (sum(agg_bytes) / 1e9) / (sum(agg_ms) / 1e3)
    traffic = None
    tf = ROOT / "profiles" / "agg_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None

    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "value_serial": round(value_serial, 3),
        "scaling": "weak", "vs_baseline": None, "dtype": "u8/u16 (SGM), f32/f64 (fit, SLIC)",
        "data": "synthetic (seeded BASELINE cfg%d scene, synth.py; paper datasets unavailable)" % c,
        "config": {"workload": "cfg%d: %dx%d uint8 pair, D=%d, P=%d, P1=%g, P2=%g, SLIC p=%d" % (
            c, h, w, cfg.d_max + 1, cfg.sgm_paths, cfg.lambda1, cfg.lambda2, cfg.superpixels),
            "frames_per_step_per_gpu": F, "streams_per_gpu": S,
            "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": "independent frames: %d concurrent pipeline contexts per GPU, "
                           "ranks = GPUs, no collective" % S,
            **({"override": override} if override else {})},
        "sgm_gdes": round(sgm_gdes, 3),
        "gde_per_frame": gde,
        "stage_ms": {k: round(v, 4) for k, v in zip(
            ("sgm_bootstrap", "road_fit", "sgm_pt", "road_refit", "disparity_transform",
             "slic", "detect"), list(out.stage_ms))},
        "n_potholes": npot[-1] if npot else None,
        "e2e": {"value": round(e2e, 3), "unit": "frames/s", "h2d_bytes_per_step": 2 * n,
                "d2h_bytes_per_step": 12 * n},
        "gpu_launches": kernels * args.steps * F,
        "roofline": {"bound": "hbm", "kernel": "k_aggregate (SGM path aggregation, 2P paths)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_src,
                     "agg_ms_per_frame": round(sum(agg_ms) / len(agg_ms), 4),
                     "alg_bytes_per_frame": agg_bytes[0] if agg_bytes else None,
                     "note": "achieved = SURVEY §8(d) algorithmic bytes / event time; the "
                             "kernel moves ~1/3 of them (u8 per-path outputs, no u16 sums)"},
        "clocks": clk,
    }
    # ---- evaluation metrics of the frame (d1 vs the scene's
    # ground-truth disparity, labels vs its pothole instances) through the
    # C-ABI with host buffers, GPU vs the oracle on one host core
    if rank == 0:
        res = ctx.detect(scene.left, scene.right, cfg, want=("d1", "labels"))
        gt_d = scene.gt_disparity.astype(np.float32)

        def eval_all(c):
            c.pep(res.d1, gt_d, 3.0)
            c.rmse(res.d1, gt_d)
            c.pixel_metrics(res.labels, scene.gt_mask)
            return c.instance_metrics(res.labels, scene.gt_mask)

        for _ in range(3):
            eval_all(ctx)
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            rep = eval_all(ctx)
        gpu_eval_ms = (time.perf_counter() - t0) * 1e3 / reps
        result["eval"] = {"metrics": "pep(eps=3) + rmse of d1, pixel + instance metrics of labels",
                          "ms_per_frame_gpu_c_abi": round(gpu_eval_ms, 3),
                          "instance_report": [rep.correct, rep.incorrect, rep.misdetection]}
        # every pothole's point cloud (rpd_cli.cpp:96-104)
        rig = ctx.rig_from_config(cfg, w, h)
        n_pot = int(res.labels.max())

        def clouds(c):
            return c.reproject_instances(res.d1, res.labels, n_pot, rig)
        clouds(ctx)
        t0 = time.perf_counter()
        for _ in range(reps):
            pts = clouds(ctx)
        result["reproject"] = {"clouds": n_pot, "points": int(sum(len(p) for p in pts)),
                               "ms_per_frame_gpu_c_abi":
                                   round((time.perf_counter() - t0) * 1e3 / reps, 3)}
        # the reference scene generator on the device — the
        # acceptance batch scene_batch(20, 7100) (640 x 480), without and with
        # noise, generated straight into HBM; then generate -> detect streamed
        # with no host image traffic
        import torch
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
        ctx.generate_scenes_device(specs, bl.data_ptr(), br.data_ptr(), bg.data_ptr(),
                                   bm.data_ptr())
        for i in range(nb):
            ctx.detect_async(bl.data_ptr() + i * per, br.data_ptr() + i * per, sh, sw, acfg)
        ctx.fetch()
        stream_fps = nb / (time.perf_counter() - t0)
        result["scenes"] = {"batch": "scene_batch(20, 7100), 640x480 (acceptance.cpp:221)",
                            "scenes_per_s_gpu": sb["noise0"],
                            "scenes_per_s_gpu_noise2": sb["noise2"],
                            "generate_detect_stream_frames_per_s": round(stream_fps, 1)}
        if ORACLE_LIB.exists() and not args.no_cpu_baseline:
            from paper_2012_10802_b200.api import Library as _Lib
            octx = _Lib(str(ORACLE_LIB)).context()
            t0 = time.perf_counter()
            octx.generate_scene(specs[0])
            result["scenes"]["scenes_per_s_oracle_1core_noise2"] = \
                round(1.0 / (time.perf_counter() - t0), 2)
            t0 = time.perf_counter()
            eval_all(octx)
            result["eval"]["ms_per_frame_oracle_1core"] = round((time.perf_counter() - t0) * 1e3, 3)
            t0 = time.perf_counter()
            clouds(octx)
            result["reproject"]["ms_per_frame_oracle_1core"] = \
                round((time.perf_counter() - t0) * 1e3, 3)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr = cpu_threads(args)
        fps, dt, frames = cpu_oracle_run(scene, PIPELINE[c] | {}, thr)
        result["cpu_baseline"] = {"value": round(fps, 4), "unit": "frames/s", "cores": thr,
                                  "kind": "port",
                                  "sample": f"{frames} cfg{c} frames, one per thread "
                                            f"({dt:.1f} s wall)"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ---------------------------------------------------------- reference arm ---
def reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_2012_10802_b200.synth import PIPELINE, SHAPES, make_scene
    c = args.config
    h, w = SHAPES[c]
    scene = make_scene(c, 0)
    thr = cpu_threads(args)
    for _ in range(args.warmup):
        cpu_oracle_run(scene, PIPELINE[c], thr)
    tot_frames, tot_s = 0, 0.0
    for _ in range(args.steps):
        _, dt, frames = cpu_oracle_run(scene, PIPELINE[c], thr)
        tot_frames += frames
        tot_s += dt
    fps = tot_frames / tot_s

    class _Cfg:
        pass
    cfg = _Cfg()
    cfg.d_max = PIPELINE[c]["d_max"]
    cfg.d_max_pt = PIPELINE[c].get("d_max_pt", 16)
    result = {
        "impl": "reference", "metric": METRIC, "value": round(fps, 4), "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot_s / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (reference arithmetic)",
        "data": "synthetic (seeded BASELINE cfg%d scene)" % c,
        "config": {"workload": "cfg%d: %dx%d uint8 pair, D=%d, P=%d" % (
            c, h, w, PIPELINE[c]["d_max"] + 1, PIPELINE[c]["sgm_paths"]),
            "implementation": "CPU oracle restatement of the reference (reference build "
                              "impossible: Eigen3/libpng absent)"},
        "sgm_gdes": None,
        "cpu_baseline": {"value": round(fps, 4), "unit": "frames/s", "cores": thr, "kind": "port",
                         "sample": f"per step {thr} cfg{c} frames, one per host thread"},
        "e2e": {"value": round(fps, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(result), flush=True)


def main():
    args = parse()
    rank, world, local = env_rank()
    if args.impl == "reference":
        reference_arm(args, rank, world)
    else:
        gpu_arm(args, rank, world, local)


if __name__ == "__main__":
    main()

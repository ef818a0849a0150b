"""Config parity sweep: the CUDA product against the LITERAL reference
(oracle/_ref/librpd_ref.so — the untouched reference sources, SURVEY.md §8(c)
Route 2) on the BASELINE configurations (BASELINE.md §3 coverage: every frame
of configs 1-4, every 64th frame of config 5).

Per frame it records the north_star bars — d0 / d1 bit-exact, D2 within 1e-4
relative (and how many pixels are bit-identical), SLIC label agreement, pothole
labels identical — plus the road fit: roll angle phi equal and a0 / a1 relative
difference.  Used by tests/test_parity_sweep.py (asserts) and
tools/parity_sweep.py (writes the JSON report under profiles/).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import time

import numpy as np

from paper_2012_10802_b200.synth import FRAMES, make_scene, pipeline_config


def sweep_cases(cfg3_frames=None, cfg5_stride=64):
    cases = [(1, 0), (2, 0), (4, 0)]
    cases += [(3, f) for f in (range(FRAMES[3]) if cfg3_frames is None else cfg3_frames)]
    cases += [(5, f) for f in range(0, FRAMES[5], cfg5_stride)]
    return cases


def _bits(a):
    return a.view(np.uint32)


def _rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def compare(a, b) -> dict:
    """a = product result, b = literal reference result."""
    va = a.d2 != -1
    vb = b.d2 != -1
    both = va & vb
    d2_rel = 0.0
    if both.any():
        x = a.d2[both].astype(np.float64)
        y = b.d2[both].astype(np.float64)
        d2_rel = float(np.max(np.abs(x - y) / np.maximum(np.maximum(np.abs(x), np.abs(y)), 1e-30)))
    rec = {
        "d0_mismatch": int((_bits(a.d0) != _bits(b.d0)).sum()),
        "d1_mismatch": int((_bits(a.d1) != _bits(b.d1)).sum()),
        "d2_valid_mismatch": int((va != vb).sum()),
        "d2_max_rel": d2_rel,
        "d2_bit_mismatch": int((_bits(a.d2) != _bits(b.d2)).sum()),
        "sp_agree": float((a.sp_labels == b.sp_labels).mean()),
        "labels_mismatch": int((a.labels != b.labels).sum()),
        "n_potholes": [int(a.n_potholes), int(b.n_potholes)],
        "phi_equal": bool(a.fit.model.phi == b.fit.model.phi),
        "phi": [a.fit.model.phi, b.fit.model.phi],
        "a0_rel": _rel(a.fit.model.a0, b.fit.model.a0),
        "a1_rel": _rel(a.fit.model.a1, b.fit.model.a1),
        "used_equal": bool(a.fit.used == b.fit.used),
    }
    rec["ok"] = (rec["d0_mismatch"] == 0 and rec["d1_mismatch"] == 0 and
                 rec["d2_valid_mismatch"] == 0 and rec["d2_max_rel"] <= 1e-4 and
                 rec["sp_agree"] >= 0.999 and rec["labels_mismatch"] == 0 and
                 rec["phi_equal"])
    return rec


def run_sweep(gpu, ref_lib, cases, threads=None) -> dict:
    """Reference detections run on host threads (one context each, ctypes
    releases the GIL) while the device processes the same frames."""
    threads = threads or max(1, min(len(cases), os.cpu_count() or 1))
    t0 = time.time()

    def ref_run(case):
        c, f = case
        sc = make_scene(c, f)
        ctx = ref_lib.context()
        r = ctx.detect(sc.left, sc.right, pipeline_config(ref_lib, c),
                       want=("d0", "d1", "d2", "labels", "sp_labels"))
        return case, r

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        futs = [ex.submit(ref_run, case) for case in cases]
        records = []
        for fut in futs:
            (c, f), b = fut.result()
            sc = make_scene(c, f)
            a = gpu.detect(sc.left, sc.right, pipeline_config(gpu.lib, c),
                           want=("d0", "d1", "d2", "labels", "sp_labels"))
            rec = compare(a, b)
            rec.update(config=c, frame=f)
            records.append(rec)
    summary = {
        "frames": len(records),
        "frames_ok": sum(r["ok"] for r in records),
        "phi_mismatch_frames": sum(not r["phi_equal"] for r in records),
        "d0_mismatch_frames": sum(r["d0_mismatch"] > 0 for r in records),
        "d1_mismatch_frames": sum(r["d1_mismatch"] > 0 for r in records),
        "label_mismatch_frames": sum(r["labels_mismatch"] > 0 for r in records),
        "d2_bit_exact_frames": sum(r["d2_bit_mismatch"] == 0 for r in records),
        "d2_max_rel": max(r["d2_max_rel"] for r in records),
        "a0_max_rel": max(r["a0_rel"] for r in records),
        "a1_max_rel": max(r["a1_rel"] for r in records),
        "sp_agree_min": min(r["sp_agree"] for r in records),
        "reference_threads": threads,
        "wall_s": round(time.time() - t0, 1),
    }
    return {"summary": summary, "records": records}

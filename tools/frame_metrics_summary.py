"""Summarise tools/ncu_frame_metrics.sh: per kernel (launches merged) serial
time, DRAM GB/s and its fraction of the measured HBM peak, and pipe / issue
utilisation weighted by duration."""
import collections
import csv
import json
import sys
from pathlib import Path

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
peak = 6531.9
try:
    mp = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))
    peak = float(mp.get("hbm_gbs") or peak)
except Exception:
    pass
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}  # -> bytes, ns
by = collections.defaultdict(dict)
for r in rows:
    v = float(r["Metric Value"].replace(",", "") or 0) * SCALE.get(r.get("Metric Unit", ""), 1.0)
    by[int(r["ID"])][r["Metric Name"]] = v
    by[int(r["ID"])]["name"] = r["Kernel Name"]
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for i, d in by.items():
    nm = d["name"].replace("rpdg::", "").replace("<unnamed>::", "").split("(")[0][:44]
    a = agg[nm]
    t = d["gpu__time_duration.sum"] / 1e3  # ns -> us
    a["n"] += 1
    a["t"] += t
    a["rd"] += d["dram__bytes_read.sum"]
    a["wr"] += d["dram__bytes_write.sum"]
    a["inst"] += d["smsp__inst_executed.sum"]
    for k in ("alu", "fma", "fp64", "lsu"):
        a[k] += t * d[f"sm__inst_executed_pipe_{k}.avg.pct_of_peak_sustained_active"]
    a["issue"] += t * d["smsp__issue_active.avg.pct_of_peak_sustained_active"]
    a["occ"] += t * d["sm__warps_active.avg.pct_of_peak_sustained_active"]
tot = sum(a["t"] for a in agg.values())
print(f"one frame: {sum(a['n'] for a in agg.values()):.0f} launches, {tot:.1f} us serial (ncu, "
      f"cold-cache), HBM peak {peak:.0f} GB/s")
print(f"{'kernel':44s} {'n':>3s} {'us':>7s} {'share':>6s} {'DRAM GB/s':>9s} {'%HBM':>5s} "
      f"{'alu%':>5s} {'fma%':>5s} {'fp64%':>5s} {'lsu%':>5s} {'issue%':>6s} {'occ%':>5s} {'Minst':>6s}")
for nm, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
    t = a["t"]
    gbs = (a["rd"] + a["wr"]) / (t * 1e-6) / 1e9 if t else 0.0  # dram bytes are bytes
    print(f"{nm:44s} {a['n']:3.0f} {t:7.1f} {100 * t / tot:5.1f}% {gbs:9.0f} {100 * gbs / peak:5.1f} "
          f"{a['alu'] / t:5.1f} {a['fma'] / t:5.1f} {a['fp64'] / t:5.1f} {a['lsu'] / t:5.1f} "
          f"{a['issue'] / t:6.1f} {a['occ'] / t:5.1f} {a['inst'] / 1e6:6.2f}")

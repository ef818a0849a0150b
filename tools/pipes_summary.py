"""Summarises tools/pipes.sh output: per kernel (aggregated over launches)
warp instructions per pipe and the SMSP-cycles each pipe needs at its issue
rate (ALU / FMA-heavy / FP64: 16 lanes per SMSP per clock = 2 cycles per warp
instruction, measured in profiles/int_peak.json and tools/pipe_probe.cu)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ix = {k: i for i, k in enumerate(hdr)}
acc = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(int)
ids = set()
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    name = r[ix["Kernel Name"]][:60]
    m = r[ix["Metric Name"]]
    v = float(r[ix["Metric Value"]].replace(",", "") or 0)
    acc[name][m] += v
    key = (name, r[ix["ID"]])
    if key not in ids:
        ids.add(key)
        cnt[name] += 1
tot = defaultdict(float)
lines = []
for k, d in acc.items():
    for m, v in d.items():
        tot[m] += v
    lines.append((d["sm__inst_executed.sum"], k, d))
lines.sort(reverse=True)
P = ["alu", "fma", "fmaheavy", "fp64", "lsu", "uniform", "adu", "cbu", "xu"]
print("%-60s %5s %8s %7s | " % ("kernel", "n", "us", "Minst") + " ".join("%7s" % p for p in P)
      + " | alu_cyc% fma_cyc%")
for inst, k, d in lines[:40]:
    print("%-60s %5d %8.1f %7.2f | " % (k, cnt[k], d["gpu__time_duration.sum"] / 1e3, inst / 1e6)
          + " ".join("%7.2f" % (d["sm__inst_executed_pipe_%s.sum" % p] / 1e6) for p in P)
          + " | %6.1f %6.1f" % (100 * d["sm__pipe_alu_cycles_active.sum"] /
                                max(1, 4 * d["sm__cycles_elapsed.avg"] * 148),
                                100 * d["sm__pipe_fma_cycles_active.sum"] /
                                max(1, 4 * d["sm__cycles_elapsed.avg"] * 148)))
print("TOTAL Minst %.1f  " % (tot["sm__inst_executed.sum"] / 1e6) +
      " ".join("%s=%.1f" % (p, tot["sm__inst_executed_pipe_%s.sum" % p] / 1e6) for p in P))

"""Summarise tools/sm_time.sh output: per kernel name, SM-us consumed per frame."""
import collections, csv, sys
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
clk = float(sys.argv[2]) if len(sys.argv) > 2 else 1.965e3  # MHz
ids = sorted({int(r["ID"]) for r in rows})
# one frame = the last 1/frames of the launches: take launches between the last two k_half
by = collections.defaultdict(dict)
for r in rows:
    by[int(r["ID"])][r["Metric Name"]] = (r["Metric Value"].replace(",", ""), r["Metric Unit"])
    by[int(r["ID"])]["name"] = r["Kernel Name"]
halves = [i for i in ids if "k_half(" in by[i]["name"]]
lo, hi = halves[-2], halves[-1]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i in ids:
    if not (lo <= i < hi):
        continue
    d = by[i]
    nm = d["name"].replace("rpdg::", "").replace("<unnamed>::", "")[:50]
    a = agg[nm]
    a[0] += 1
    a[1] += float(d["gpu__time_duration.sum"][0]) / (1000.0 if d["gpu__time_duration.sum"][1] == "ns" else 1.0)
    a[2] += float(d["sm__cycles_active.sum"][0]) / clk  # SM-us
    a[3] += float(d["smsp__inst_executed.sum"][0])
tot_t = sum(a[1] for a in agg.values()); tot_sm = sum(a[2] for a in agg.values())
print(f"frame: {sum(a[0] for a in agg.values())} launches, {tot_t:.1f} us serial, {tot_sm:.0f} SM-us "
      f"(= {tot_sm / 148:.1f} us of the full GPU)")
for nm, a in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    print(f"{a[2]:9.0f} SM-us {100 * a[2] / tot_sm:5.1f}%  {a[1]:7.1f} us  {a[0]:3d}x  {a[3] / 1e6:7.2f} Mwarp-inst  {nm}")

"""Per-frame kernel time breakdown from an ncu --metrics gpu__time_duration.sum CSV."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
names = [d["Kernel Name"] for d in data]
idx = [i for i, n in enumerate(names) if "k_flat_model" in n]
s, e = idx[-2], idx[-1]
frame = data[s:e]
agg = collections.OrderedDict()
tot = 0.0
unit = frame[0]["Metric Unit"]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
for d in frame:
    n = d["Kernel Name"].split("(")[0].replace("rpdg::", "").replace("<unnamed>::", "")[:58]
    t = float(d["Metric Value"]) * scale
    tot += t
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += t
print(f"frame: {len(frame)} launches, {tot:.1f} us (serialised, cold-cache)")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{t:9.1f} us {100*t/tot:5.1f}% {c:4d}x  {n}")

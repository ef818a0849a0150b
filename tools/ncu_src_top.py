"""Top stalled SASS lines of an `ncu --page source --csv` dump."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
start = 1 if rows[0][0] == "Kernel Name" else 0
print(rows[0][1] if start else "")
hdr = rows[start]
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
data = [r for r in rows[start + 1:] if len(r) == len(hdr) and r[si].replace(".", "", 1).isdigit()]
tot = sum(float(r[si]) for r in data)
print("samples", tot, "sass lines", len(data), "warp-instr executed", sum(float(r[ei] or 0) for r in data))
order = sorted(range(len(data)), key=lambda i: -float(data[i][si]))[:n]
for i in sorted(order):
    r = data[i]
    print(f"{i:5d} {r[si]:>6s} {r[ei]:>9s}  {r[1][:96]}")

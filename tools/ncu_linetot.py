"""Per-source-line executed warp instructions (all files) of an ncu report: ncu_linetot.py REP [MIN]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 2e5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fp = None; tot = collections.defaultdict(float); stl = collections.defaultdict(float); src = {}
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "File Path":
        fp = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)")
        j = i + 1
        while j < len(rows) and not (rows[j] and rows[j][0] in ("File Path", "Function Name")):
            rr = rows[j]
            if len(rr) == len(hdr) and rr[0].isdigit():
                try:
                    tot[(fp, int(rr[0]))] += float(rr[ie] or 0)
                    stl[(fp, int(rr[0]))] += float(rr[si] or 0)
                except ValueError:
                    pass
                src.setdefault((fp, int(rr[0])), rr[1])
            j += 1
        i = j
        continue
    i += 1
T = sum(tot.values()); S = sum(stl.values())
print(f"total {T / 1e6:.2f}M warp-inst, {S:.0f} stall samples")
for k in sorted(tot):
    if tot[k] > mn or stl[k] > 0.02 * S:
        print(f"{k[0][:12]:12s} {k[1]:4d} {tot[k] / 1e6:6.2f}M {100 * stl[k] / max(S, 1):5.1f}%  {src[k].strip()[:80]}")

"""Instruction mix + top stalled SASS lines of one kernel in an ncu report.
usage: ncu_ops.py REP KERNEL_REGEX [N]"""
import collections, csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
his = [i for i, r in enumerate(rows) if "Instructions Executed" in r]
hi = his[0]
hdr = rows[hi]
end = his[1] - 1 if len(his) > 1 else len(rows)
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
si = hdr.index("Warp Stall Sampling (All Samples)")
def num(x):
    try:
        return float(x)
    except ValueError:
        return None
data = [r for r in rows[hi + 1:end] if len(r) == len(hdr) and num(r[ie]) is not None]
tot = sum(num(r[ie]) for r in data)
stot = sum(num(r[si]) or 0 for r in data)
print(f"warp-instr {tot:.0f}  stall samples {stot:.0f}  sass lines {len(data)}")
op = collections.Counter()
for r in data:
    t = r[src].strip().split()
    o = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    op[o.split(".")[0]] += num(r[ie])
print("  ".join(f"{k}:{100 * v / tot:.1f}%" for k, v in op.most_common(16)))
order = sorted(range(len(data)), key=lambda i: -(num(data[i][si]) or 0))[:n]
for i in sorted(order):
    r = data[i]
    print(f"{i:5d} {r[si]:>6s} {r[ie]:>9s}  {r[src][:90]}")

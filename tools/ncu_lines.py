"""Per-CUDA-source-line stall samples (and top stall reasons) of the kernels in
an ncu report: ncu_lines.py REP [N]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
func = None
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Function Name":
        func = r[1]
    if r and r[0] == "Line No" and len(r) > 4:
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        stall_cols = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_")]
        per = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter(), ""])
        j = i + 1
        while j < len(rows) and not (rows[j] and rows[j][0] in ("File Path", "Function Name")):
            rr = rows[j]
            if len(rr) == len(hdr) and rr[0].isdigit():
                e = per[int(rr[0])]
                try:
                    e[0] += float(rr[si] or 0)
                    e[1] += float(rr[ie] or 0)
                    for c, h in stall_cols:
                        e[2][h] += float(rr[c] or 0)
                except ValueError:
                    pass
                if not e[3]:
                    e[3] = rr[1]
            j += 1
        tot = sum(v[0] for v in per.values())
        print(f"== {func}  samples={tot:.0f}")
        for ln, (s, ins, st, src) in sorted(per.items(), key=lambda x: -x[1][0])[:n]:
            top = ", ".join(f"{k[6:]}={int(v)}" for k, v in st.most_common(3) if v)
            print(f"{ln:5d} {100 * s / max(tot, 1):5.1f}% ins={ins:10.0f}  {src.strip()[:60]:60s} {top}")
        i = j
        continue
    i += 1

"""Summarise the RPD_FIT_TRACE=1 clock64 trace of the last k_fit launch."""
import collections, sys
lines = open(sys.argv[1]).read().splitlines()
runs, cur, hruns, hcur = [], [], [], []
for l in lines:
    p = l.split()
    if p and p[0] == "FITTR":
        if int(p[1]) == 0 and cur:
            runs.append(cur); cur = []
            hruns.append(hcur); hcur = []
        cur.append((int(p[2]), int(p[3])))
    elif p and p[0] == "FITH":
        hcur.append(int(p[2]))
runs.append(cur); hruns.append(hcur)
r, h = runs[-1], hruns[-1]
print(len(runs), "launches; last:", len(r), "events, total", r[-1][1], "cycles")
d = collections.defaultdict(lambda: [0, 0])
for (a, ta), (b, tb) in zip(r, r[1:]):
    d[(a, b)][0] += 1
    d[(a, b)][1] += tb - ta
for k, (c, t) in sorted(d.items(), key=lambda x: -x[1][1]):
    print(f"{str(k):10s} n={c:3d} total={t:7d} avg={t // c}")
hd = [b - a for a, b in zip(h[0::2], h[1::2])]
if hd:
    print("helper sincos: n=%d avg=%d max=%d" % (len(hd), sum(hd) // len(hd), max(hd)))

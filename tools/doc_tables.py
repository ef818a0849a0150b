"""Regenerates the results tables of DESIGN.md §6.2 and BASELINE.md from
profiles/r2_bench_cfg{1..5}.json and profiles/agg_traffic.json."""
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
names = {5: "5 (default)", 1: "1 (240×320, P=4)", 2: "2", 3: "3 (64 × 1024×1280)",
         4: "4 (1080×1920, D=256)"}
bnames = {1: "1 (240×320, P=4)", 2: "2 (800×1312)", 3: "3 (64 × 1024×1280)",
          4: "4 (1080×1920, D=256)", 5: "5 (streaming, distinct frames)"}
tr = json.loads((ROOT / "profiles" / "agg_traffic.json").read_text())["configs"]
rows, brows = [], []
for c in (5, 1, 2, 3, 4):
    d = json.loads((ROOT / "profiles" / f"r2_bench_cfg{c}.json").read_text())
    r = d["roofline"]
    cpu = d["cpu_baseline"]["value"]
    dram = tr[str(c)]["bytes_per_frame"] / (r["agg_ms_per_frame"] * 1e-3) / 1e9 / r["peak"]
    dtxt = f"{dram:.2f}" + (" (L2-resident)" if c == 1 else "")
    rows.append(f"| {names[c]} | {d['value']:.0f} | {d['e2e']['value']:.0f} | {d['value_serial']:.0f} | "
                f"{d['sgm_gdes']:.1f} | {r['agg_ms_per_frame']:.3f} | {r['frac']:.2f} | {dtxt} | "
                f"{r['int_ops']['frac']:.2f} | {cpu:.1f} | {d['e2e']['value'] / cpu:.0f}× |")
for c in (1, 2, 3, 4, 5):
    d = json.loads((ROOT / "profiles" / f"r2_bench_cfg{c}.json").read_text())
    cb = d["cpu_baseline"]
    brows.append(f"| {bnames[c]} | {cb['value']:.1f} frames/s | {cb['latency_ms_1thread']:.0f} | "
                 f"{d['e2e']['value']:.0f} | {d['value']:.0f} |")


def replace_table(path, header, new_rows):
    text = path.read_text()
    i = text.index(header)
    j = text.index("\n\n", i)
    lines = text[i:j].split("\n")
    text = text[:i] + "\n".join(lines[:2] + new_rows) + text[j:]
    path.write_text(text)


replace_table(ROOT / "DESIGN.md", "| config | value (frames/s) | e2e | serial |", rows)
replace_table(ROOT / "BASELINE.md", "| config | literal reference, 16 threads |", brows)
print("\n".join(rows))
print("\n".join(brows))

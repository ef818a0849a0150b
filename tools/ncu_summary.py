"""Summarise an ncu report: per-kernel time, DRAM bytes, occupancy, top stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
def col(r, name):
    return r[hdr.index(name)] if name in hdr else "-"
for r in rows[2:]:
    name = col(r, "Kernel Name")[:48]
    t = col(r, "gpu__time_duration.sum"); tu = units[hdr.index("gpu__time_duration.sum")]
    rd = col(r, "dram__bytes_read.sum"); ru = units[hdr.index("dram__bytes_read.sum")]
    wr = col(r, "dram__bytes_write.sum"); wu = units[hdr.index("dram__bytes_write.sum")]
    act = col(r, "smsp__cycles_active.avg"); el = col(r, "sm__cycles_elapsed.avg")
    occ = col(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    ipc = col(r, "sm__inst_executed.avg.per_cycle_active")
    stalls = sorted(((float(r[i] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                     and not h.endswith("not_issued")), reverse=True)[:4]
    print(f"{name:48s} t={t}{tu} rd={rd}{ru} wr={wr}{wu} active/elapsed={act}/{el} occ%={occ} ipc={ipc}")
    print("      stalls:", ", ".join(f"{n}={int(v)}" for v, n in stalls))

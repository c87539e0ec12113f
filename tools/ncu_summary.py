"""Summarise an ncu report: key raw metrics + the hottest SASS lines (by warp-stall samples)."""
import csv, subprocess, sys, collections

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum.per_second"]
for v in rows[2:]:
    print("kernel:", v[h.index("Kernel Name")][:80])
    for i, name in enumerate(h):
        if name in want:
            print(f"  {name} = {v[i]} {u[i]}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    # one table per kernel; each starts with a header row holding the column names
    data, hh = [], None
    for r in rows:
        if "Source" in r and "Instructions Executed" in r:
            hh = r
            continue
        if hh is None or len(r) != len(hh):
            continue
        wcol = next((c for c in hh if c.startswith("Warp Stall Sampling (All")), None)
        if wcol is None:
            continue
        si, ci, wi = hh.index("Source"), hh.index("Instructions Executed"), hh.index(wcol)
        try:
            data.append((r[si], int(r[ci] or 0), int(r[wi] or 0)))
        except ValueError:
            continue
    if not data:
        print("(no source-level samples in the report)")
        sys.exit(0)
    tot = sum(d[2] for d in data)
    print("top stall lines (samples, executed, sass):")
    for d in sorted(data, key=lambda d: -d[2])[:int(sys.argv[2])]:
        print(f"  {d[2]:6d} {100*d[2]/max(tot,1):5.1f}% {d[1]:10d}  {d[0][:100]}")

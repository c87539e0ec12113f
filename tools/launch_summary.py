"""Summarise ncu launch lists (gpu__time_duration, dram bytes, instructions per kernel launch) of
the LAST call in each file: python tools/launch_summary.py profiles/round2_launches_*.csv"""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    if not rows:
        continue
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = {}
    for r in rows[1:]:
        d.setdefault(int(r[ii]), {"k": r[ki].split("(")[0].replace("rtk_b200::", "")})[r[mi]] = r[vi]
    ids = sorted(d)
    # the last call = the launches after the last k_sample_select / k_rows_fused / first kernel of a call
    starts = [i for i in ids if any(s in d[i]["k"] for s in ("k_sample_select", "k_rows_fused", "k_lsd_hist",
                                                               "k_scale_guess", "k_init_sel", "k_row_cluster"))]
    first = starts[-1] if starts else ids[0]
    if "k_scale_guess" not in d[first]["k"] and any("k_scale_guess" in d[i]["k"] for i in ids if i < first):
        first = max(i for i in ids if i < first and "k_scale_guess" in d[i]["k"])
    print(f"== {path.split('/')[-1]} (last call: launches {first}..{ids[-1]})")
    tot = 0.0
    for i in ids:
        if i < first:
            continue
        v = d[i]
        t = v.get("gpu__time_duration.sum", "nan")
        try:
            tus = float(t) / 1e3
            tot += tus
            ts = f"{tus:8.1f} us"
        except ValueError:
            ts = "  (not replayable: cooperative grid barrier)"
        rd = v.get("dram__bytes_read.sum", "")
        wr = v.get("dram__bytes_write.sum", "")
        rd = f"{float(rd) / 1e6:9.1f} MB rd" if rd not in ("", "nan") else ""
        wr = f"{float(wr) / 1e6:8.1f} MB wr" if wr not in ("", "nan") else ""
        print(f"   {v['k'][:44]:44s} {ts} {rd} {wr}")
    print(f"   {'sum (serialised, cold L2)':44s} {tot:8.1f} us")

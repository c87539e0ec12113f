"""Per-CUDA-source-line instruction / stall totals of an ncu report (source page with the
cuda,sass correlation). usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, hdr, fname = [], None, ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] in ("", "-"):
        continue  # SASS rows of a line carry an empty line number; the line row holds the totals
    try:
        n = int(r[hdr.index("Instructions Executed")] or 0)
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    rows.append((n, s, f"{fname}:{r[0]}", r[1].strip()[:80]))
ti = sum(r[0] for r in rows) or 1
ts = sum(r[1] for r in rows) or 1
print(f"warp-instr {ti} stall-samples {ts} (per CUDA line, sorted by instructions)")
for n, s, ln, src in sorted(rows, reverse=True)[:N]:
    print(f"{100 * n / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {ln:>16} {src}")

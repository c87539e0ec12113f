"""Per-CUDA-source-line instruction / stall totals of an ncu report (uses the SASS page's
source correlation). usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(out)))
hdr = None
rows = []
fname = ""
for r in rd:
    if r and r[0] == "#":
        hdr = r; continue
    if len(r) == 1 and r[0].startswith("File"): fname = r[0]
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0); n = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        rows.append((n, s, d["#"], d["Source"].strip()[:90]))
ti = sum(r[0] for r in rows) or 1; ts = sum(r[1] for r in rows) or 1
print(f"warp-instr {ti} samples {ts}")
for n, s, ln, src in sorted(rows, reverse=True)[:N]:
    print(f"{100*n/ti:5.1f}% inst {100*s/ts:5.1f}% stall  L{ln:>5} {src}")

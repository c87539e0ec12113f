"""Hot SASS instructions of an ncu report (warp-stall samples, instructions executed).
usage: python tools/ncu_hot.py report.ncu-rep [N]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rd if r and r[0] == "Address")
rows = []
for i, r in enumerate(rd):
    if len(r) == len(hdr) and r[0].startswith("0x"):
        d = dict(zip(hdr, r))
        rows.append((int(d["Warp Stall Sampling (All Samples)"] or 0), int(d["Instructions Executed"] or 0), i, d["Source"].strip()[:70]))
ts = sum(r[0] for r in rows) or 1; ti = sum(r[1] for r in rows) or 1
print(f"samples {ts}  warp-instr {ti}  sass-lines {len(rows)}")
for s, n, i, src in sorted(rows, reverse=True)[:N]:
    print(f"{100*s/ts:5.1f}% stall {100*n/ti:5.2f}% inst  #{i:5d} {src}")

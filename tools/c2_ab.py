"""A/B of the C2 single-query leg under env variants (one subprocess per variant): ms per call via
rtk.bench_topk (C-side loop, engine-recorded call events), n=2^28 U[0,1), k list from KS."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys
sys.path.insert(0, %r)
import torch
from paper_2501_14336_b200 import rtk as R
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.rand(1 << int(os.environ.get("LOGN", "28")), device="cuda", generator=g)
out = []
for k in [int(v) for v in os.environ.get("KS", "256,1048576").split(",")]:
    ms = R.bench_topk(x, k, 30, 3).median_ms
    out.append(f"k={k} {ms*1e3:.1f}us")
print(" | ".join(out))
''' % ROOT

for var in (sys.argv[1:] or [""]):
    env = dict(os.environ)
    for kv in var.split():
        a, b = kv.split("=", 1)
        env[a] = b
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    print(f"[{var or 'default'}]", r.stdout.strip() or r.stderr.strip()[-400:], flush=True)

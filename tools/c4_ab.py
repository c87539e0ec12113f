"""A/B of the C4 leg (n=2^26 U[128.6,128.7) f32, k=2^16, scaled_topk off/always/adaptive) under env
variants, one subprocess per variant, via rtk.bench_scaled (C-side loop)."""
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
xa = (128.6 + 0.1 * torch.rand(1 << 26, device="cuda", generator=g)).float()
out = []
for m in (0, 1, 2):
    pol = R.ScalePolicy(mode=R.ScaleMode(m), trigger_fraction=0.5, seed=31)
    ms = R.bench_scaled(xa, 1 << 16, 20, 3, policy=pol).median_ms
    out.append(f"mode{m} {ms*1e3:.1f}us")
print(" | ".join(out))
''' % ROOT

for var in (sys.argv[1:] or [""]):
    env = dict(os.environ)
    for kv in var.split():
        a, b = kv.split("=", 1)
        env[a] = b
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    print(f"[{var or 'default'}]", r.stdout.strip() or r.stderr.strip()[-400:], flush=True)

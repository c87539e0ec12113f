"""A/B of the C3 batched leg under env variants (one subprocess per variant): ms per batch via
rtk.bench_batch_dense (C-side loop, L2 flushed between steps), fp32 and bf16 logits."""
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
V = int(os.environ.get("V", "128256")); B = int(os.environ.get("B", "256"))
L = torch.randn(B, V, device="cuda", generator=g)
flush = torch.empty(int(os.environ.get("FLUSH_MB", "256")) << 20, dtype=torch.uint8, device="cuda")
out = []
for dt in os.environ.get("DT", "f32").split(","):
    X = L if dt == "f32" else L.to(torch.bfloat16)
    for k in [int(v) for v in os.environ.get("KS", "50,4096").split(",")]:
        ms = R.bench_batch_dense(X, k, 20, 3, flush).median_ms
        out.append(f"{dt} k={k} {ms*1e3:.1f}us")
print(" | ".join(out))
''' % ROOT

for var in (sys.argv[1:] or [""]):
    env = dict(os.environ)
    for kv in var.split():
        a, b = kv.split("=", 1)
        env[a] = b
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    print(f"[{var or 'default'}]", r.stdout.strip() or r.stderr.strip()[-400:], flush=True)

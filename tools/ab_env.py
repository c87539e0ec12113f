"""Device time of one workload under the current RTK_* environment (rtk_bench_* C loops, L2
flushed before each step except C2): python tools/ab_env.py tiny|c1|c2|c3|c3b|c4 k [mode]. RTK_PKG_ROOT
selects another build (tools/build_variant.sh)."""
import os
import sys

sys.path.insert(0, os.environ.get("RTK_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2501_14336_b200 import rtk as R

which, k = sys.argv[1], int(sys.argv[2])
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
if which in ("tiny", "tinynf"):  # the fixed per-call cost: one 1000-element row (one CTA); nf: no L2 flush
    x = torch.from_numpy(np.random.default_rng(1).random(1000, dtype=np.float32)).to(dev)
    b = R.bench_topk(x, k, 20, 5, flush=flush if which == "tiny" else None)
elif which in ("c1", "c2"):
    n = 1 << (20 if which == "c1" else 28)
    x = torch.from_numpy(np.random.default_rng(1).random(n, dtype=np.float32)).to(dev)
    b = R.bench_topk(x, k, 20, 5, flush=flush if which == "c1" else None)  # C2: 1 GiB > L2
elif which in ("c3", "c3b"):
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((256, 128256), dtype=np.float32)).to(dev)
    if which == "c3b":
        x = x.to(torch.bfloat16)
    b = R.bench_batch_dense(x, k, 20, 5, flush)
else:
    n = 1 << 26
    x = torch.from_numpy(np.float32(128.6) + np.float32(0.1) * np.random.default_rng(5).random(n, dtype=np.float32)).to(dev)
    pol = R.ScalePolicy(mode=R.ScaleMode(int(sys.argv[3]) if len(sys.argv) > 3 else 0), trigger_fraction=0.5, seed=31)
    b = R.bench_scaled(x, k, 20, 5, policy=pol, flush=flush)
env = " ".join(f"{a}={v}" for a, v in sorted(os.environ.items()) if a.startswith("RTK_"))
print(f"{which} k={k} {env or '(default)'}: {b.median_ms * 1e3:.1f} us device, {b.median_host_ms * 1e3:.1f} us host")

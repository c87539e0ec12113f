"""Per-phase device times (RTK_PROFILE=1 event marks, printed by the engine to stderr) of one
workload: python tools/prof_marks.py c2|c1|c3|c4|samp [k] — run with RTK_PROFILE=1 (and any other RTK_*
switch) in the environment."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2501_14336_b200 as rtk
from paper_2501_14336_b200 import rtk as R

which = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else None
dev = torch.device("cuda", 0)
if which == "tiny":
    x = torch.from_numpy(np.random.default_rng(1).random(1000, dtype=np.float32)).to(dev)
    for _ in range(3):
        rtk.topk(x, k or 1)
elif which in ("c1", "c2"):
    n = 1 << (20 if which == "c1" else 28)
    x = torch.from_numpy(np.random.default_rng(1).random(n, dtype=np.float32)).to(dev)
    for _ in range(3):
        rtk.topk(x, k or (256 if which == "c1" else 1 << 20))
elif which == "c3":
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((256, 128256), dtype=np.float32)).to(dev)
    if os.environ.get("BF16"):
        x = x.to(torch.bfloat16)
    for _ in range(3):
        rtk.batch_topk_dense(x, k or 50)
elif which == "samp":  # the LLM sampling consumer on the C3 logits (top-k -> softmax -> top-p -> draw)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((256, 128256), dtype=np.float32)).to(dev)
    u = torch.rand(256, device=dev)
    for _ in range(3):
        R.topk_sample(x, k or 50, top_p=0.9, uniform=u)
elif which == "c4":
    n = 1 << 26
    x = torch.from_numpy((np.float32(128.6) + np.float32(0.1) * np.random.default_rng(5).random(n, dtype=np.float32))).to(dev)
    pol = R.ScalePolicy(mode=R.ScaleMode(int(os.environ.get("MODE", "0"))), trigger_fraction=0.5, seed=31)
    for _ in range(3):
        R.scaled_topk(x, k or 1 << 16, policy=pol)
torch.cuda.synchronize()
print(which, "stats", rtk.last_stats(), file=sys.stderr)

"""A/B of the C2 query across library builds: python tools/ab_c2.py <pkg parent dir> — median device
time (torch events around rtk.topk, 20 calls after 5 warm-up) for numpy-PCG64 and torch.rand inputs."""
import os
import statistics
import sys

sys.path.insert(0, sys.argv[1])
import numpy as np
import torch

import paper_2501_14336_b200 as rtk

dev = torch.device("cuda", 0)
xs = {"numpy": torch.from_numpy(np.random.default_rng(1).random(1 << 28, dtype=np.float32)).to(dev)}
g = torch.Generator(device=dev)
g.manual_seed(1)
xs["torch"] = torch.rand(1 << 28, device=dev, generator=g)
for name, x in xs.items():
    for k in (256, 16384, 1 << 20):
        for _ in range(5):
            rtk.topk(x, k)
        ev = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rtk.topk(x, k)
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        print(sys.argv[1][-12:], name, k, round(statistics.median(a.elapsed_time(b) for a, b in ev) * 1000, 1), "us")

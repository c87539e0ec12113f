"""Small driver for ncu: a few rtk.topk calls on the bench workload (n=2^logn, k)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_14336_b200 as rtk

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 28
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.rand(1 << logn, device="cuda", generator=g)
for _ in range(reps):
    r = rtk.topk(x, k)
torch.cuda.synchronize()
print("stats", rtk.last_stats())

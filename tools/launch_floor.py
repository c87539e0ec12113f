"""Fixed per-call costs on this box: events around (a) one tiny torch kernel, (b) a replayed CUDA
graph of one tiny kernel, (c) rtk_topk on 1000 elements (graph replay + host completion wait),
each after a synchronize (GPU idle at the start event, as in the bench loops)."""
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2501_14336_b200 import rtk as R

dev = torch.device("cuda", 0)
x = torch.zeros(1000, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn, n=50):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts[5:])


print(f"torch add_ kernel: {timeit(lambda: x.add_(1.0)):.1f} us")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    x.add_(1.0)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        x.add_(1.0)
print(f"graph replay (1 kernel): {timeit(g.replay):.1f} us")
y = torch.from_numpy(np.random.default_rng(1).random(1000, dtype=np.float32)).to(dev)
print(f"rtk.topk n=1000 k=1 (graph replay + completion wait): {timeit(lambda: R.topk(y, 1)):.1f} us")
b = R.bench_topk(y, 1, 30, 5)
print(f"rtk bench_topk n=1000 k=1: {b.median_ms * 1e3:.1f} us device, {b.median_host_ms * 1e3:.1f} us host")

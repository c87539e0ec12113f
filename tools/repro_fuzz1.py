import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2501_14336_b200 as rtk
from tests.test_gpu_fuzz import _k, _row
from tests.test_gpu_parity import _widen16
case = 100900
rng = np.random.default_rng(case)
dtype = np.float32 if rng.integers(0, 3) else np.uint32
order = int(rng.integers(0, 2))
mode = rng.integers(0, 4)
assert mode == 3
kind = "bf16" if rng.integers(0, 2) else "f16"
n = int(rng.integers(1, 1 << 21))
scale = float(rng.choice([1.0, 1e-3, 100.0]))
xf = torch.from_numpy(rng.standard_normal(n).astype(np.float32) * scale)
t16 = xf.to(torch.bfloat16 if kind == "bf16" else torch.float16)
h = t16.view(torch.int16).numpy().view(np.uint16).copy()
k = _k(rng, n)
print(kind, n, k, order, scale)
x32 = _widen16(h, kind)
wv, wi, wp = O.ref_topk(x32, k, order, grid=8)
print("ref", wi[:5], x32[wi[:5]], h[wi[:5]])
r = rtk.topk(t16.cuda(), k, rtk.SelectionOrder(order))
gi = r.indices.cpu().numpy()
print("gpu", gi[:5], x32[gi[:5].astype(np.int64)], h[gi[:5].astype(np.int64)])
mx = np.nanmax(x32)
print("max", mx, "count", (x32 == mx).sum(), "first idx", np.argmax(x32 == mx), "nan count", np.isnan(x32).sum())

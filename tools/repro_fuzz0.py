import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from tests.test_gpu_fuzz import _row, _k
import paper_2501_14336_b200 as rtk
import oracle as O
from tests.test_gpu_parity import gpu_topk, assert_same
rng = np.random.default_rng(7000)
n = int(rng.choice([rng.integers(1, 1 << 18), rng.integers((1 << 18) + 1, (1 << 21) + 1), rng.integers(1 << 21, 1 << 23)]))
x = _row(rng, n, np.uint32)
k = int(rng.integers(1, 513)) if rng.integers(0, 2) else _k(rng, n)
order = int(rng.integers(0, 2))
print("n", n, "k", k, "order", order, flush=True)
for o in (order, 1 - order):
    for dt in (np.uint32, np.float32):
        xx = x if dt == np.uint32 else x.view(np.float32)
        try:
            r = gpu_topk(xx, k, o, torch.device("cuda", 0))
            assert_same(r, O.ref_topk(xx, k, o, grid=8), "x")
            print("ok", dt.__name__, o, flush=True)
        except Exception as e:
            print("FAIL", dt.__name__, o, str(e)[:200], flush=True)
            raise SystemExit(1)

"""rtk_topk_host end to end (C2: 1 GiB pinned input, k = 2^20): outputs into pageable numpy
arrays vs pinned buffers, against the bare 1 GiB H2D."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2501_14336_b200 import _lib as L
from paper_2501_14336_b200 import rtk as R

n, k = 1 << 28, 1 << 20
hx = torch.from_numpy(np.random.default_rng(1).random(n, dtype=np.float32)).pin_memory()
lib = L.load()
h = R._handle(0)
cfg = R.EngineConfig()._c()


def timed(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


def call(vals, idx, piv):
    st = lib.rtk_topk_host(h, C.c_void_p(hx.data_ptr()), n, k, 0, 0, C.c_void_p(vals), C.c_void_p(idx),
                           C.c_void_p(piv), C.byref(cfg))
    assert st == 0


pv, pi, pp = np.empty(k, np.float32), np.empty(k, np.uint64), np.zeros(1, np.uint32)
t_page = timed(lambda: call(pv.ctypes.data, pi.ctypes.data, pp.ctypes.data))
qv, qi, qp = (torch.empty(k, dtype=torch.float32).pin_memory(), torch.empty(k, dtype=torch.int64).pin_memory(),
              torch.empty(1, dtype=torch.int32).pin_memory())
t_pin = timed(lambda: call(qv.data_ptr(), qi.data_ptr(), qp.data_ptr()))
d = torch.empty(n, dtype=torch.float32, device="cuda")
t_h2d = timed(lambda: (d.copy_(hx, non_blocking=True), torch.cuda.synchronize()))
t_py = timed(lambda: R.topk(hx.numpy(), k))
print(f"rtk_topk_host pageable outputs {t_page:.2f} ms, pinned outputs {t_pin:.2f} ms, bare H2D {t_h2d:.2f} ms, "
      f"python rtk.topk(numpy) {t_py:.2f} ms")

"""Replay fuzz_explore cases (batch mode) with the force switches printed; argv: case ids."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2501_14336_b200 as rtk
from tests.test_gpu_fuzz import _k, _row
from tests.test_gpu_parity import _widen16
dev = torch.device("cuda", 0)
for case in [int(c) for c in sys.argv[1:]]:
    rng = np.random.default_rng(case)
    dtype = np.float32 if rng.integers(0, 3) else np.uint32
    order = int(rng.integers(0, 2))
    mode = rng.integers(0, 6)
    force = rng.integers(0, 8)
    print("case", case, "mode", mode, "force", force, "dtype", dtype.__name__, "order", order)
    if mode == 1:
        B = int(rng.integers(1, 40))
        lens = [int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 200000), rng.integers(200000, 1 << 21)],
                               p=[0.5, 0.4, 0.1])) for _ in range(B)]
        rows = [_row(rng, n, dtype) for n in lens]
        ks = [_k(rng, n) for n in lens]
        offs, parts, pos = [], [], 0
        for t in range(B):
            g = int(rng.integers(0, 9))
            parts.append(np.zeros(g, dtype=dtype)); pos += g; offs.append(pos); parts.append(rows[t]); pos += lens[t]
        data = np.concatenate(parts)
        exp = O.ref_batch_topk(data, offs, lens, ks, order, grid=16)
        td = torch.from_numpy(data.view(np.int32) if dtype == np.uint32 else data).to(dev)
        if dtype == np.uint32:
            td = td.view(torch.uint32)
        for fe, fd in [(0, 0), (1, 0), (0, 1)]:
            rtk.set_option("force_exact", fe); rtk.set_option("force_deep", fd)
            got = rtk.batch_topk(rtk.BatchInput(td, offs, lens, ks), rtk.SelectionOrder(order))
            bad = []
            for t in range(B):
                gi = got[t].indices.cpu().numpy().astype(np.uint64)
                if not np.array_equal(gi, exp[t][1].astype(np.uint64)):
                    bad.append((t, lens[t], ks[t], gi[:3].tolist(), exp[t][1][:3].tolist()))
            print("  force_exact", fe, "force_deep", fd, "bad rows", bad[:4], "| lens", lens[:30], "ks", ks[:30])
        rtk.set_option("force_exact", 0); rtk.set_option("force_deep", 0)

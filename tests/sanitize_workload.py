"""Small workloads covering every kernel of the library, for compute-sanitizer
(tests/test_gpu_sanitizer.py): single queries on the sampled / unsampled / one-CTA paths, a ragged
batch with short, long and dense rows (one-CTA rows, the general pipeline, the LSD sort), 16-bit
keys, all three scale modes, the forced exact path and forced deeper MSD levels, the sampling
consumer and the shard merge. Every result is checked against the C restatement (oracle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2501_14336_b200 as rtk
from paper_2501_14336_b200 import rtk as R


def check(got, x, k, order=0, what=""):
    wv, wi, _ = O.port_topk(x, k, order)
    gi = got.indices.cpu().numpy().astype(np.uint64)
    assert np.array_equal(gi, wi), what


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(17)
    # (1 << 22, 1 << 19): the one-huge-row level-0 MSD over Q co-resident clusters (grid barrier);
    # (1 << 20, 256), (1 << 19 + 5, 512): the single-query cluster kernel (k_row_cluster, DSMEM)
    for n, k in [(3000, 7), (1 << 16, 256), (1 << 17, 50000), (1 << 20, 4096), (1 << 22, 1 << 19),
                 (1 << 20, 256), ((1 << 19) + 5, 512)]:
        x = rng.standard_normal(n).astype(np.float32)
        for order in (0, 1):
            check(rtk.topk(torch.from_numpy(x).to(dev), k, rtk.SelectionOrder(order)), x, k, order, f"topk {n} {k}")
    lens = [5000, 70001, 130000, 9000]
    ks = [50, 4000, 130000, 6000]
    offs = [0]
    for ln in lens[:-1]:
        offs.append(offs[-1] + ln + 3)
    data = rng.standard_normal(offs[-1] + lens[-1]).astype(np.float32)
    got = rtk.batch_topk(rtk.BatchInput(torch.from_numpy(data).to(dev), offs, lens, ks))
    for t in range(4):
        check(got[t], data[offs[t]:offs[t] + lens[t]], ks[t], 0, f"batch {t}")
    lb = torch.from_numpy(rng.standard_normal((4, 20000)).astype(np.float32)).to(dev).to(torch.bfloat16)
    for kb in (50, 20000):
        rtk.batch_topk_dense(lb, kb)
    xa = (np.float32(128.6) + np.float32(0.1) * rng.random(1 << 20, dtype=np.float32)).astype(np.float32)
    for mode in (0, 1, 2):
        r = rtk.scaled_topk(torch.from_numpy(xa).to(dev), 4096, policy=R.ScalePolicy(R.ScaleMode(mode), 0.5, 31))
        wv, wi, _, _ = O.port_scaled_topk(xa, 4096, 0, mode=mode, tau=0.5, seed=31)
        assert np.array_equal(r.indices.cpu().numpy().astype(np.uint64), wi), f"scaled {mode}"
    x = rng.standard_normal(1 << 18).astype(np.float32)
    rtk.set_option("force_exact", 1)
    check(rtk.topk(torch.from_numpy(x).to(dev), 1000), x, 1000, 0, "exact")
    rtk.set_option("force_exact", 0)
    rtk.set_option("force_deep", 1)
    check(rtk.topk(torch.from_numpy(x).to(dev), 100000), x, 100000, 0, "deep")
    rtk.set_option("force_deep", 0)
    lg = torch.from_numpy(rng.standard_normal((8, 4000)).astype(np.float32)).to(dev)
    R.topk_sample(lg, 50, top_p=0.9, uniform=torch.rand(8, device=dev))
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()

"""GPU fuzz parity: seeded random batches that mix every routing decision of one call — one-CTA
short rows (k_rows_fused, both buffer variants), the sampled general pipeline (k_compact ->
MSD -> sort groups), dense rows (k >= n/2: LSD sort), single long queries (k_row_cluster) — with
random distributions (uniform, normal, zipf, heavy ties, sorted runs, NaN/inf sprinkles), orders,
dtypes (f32, u32) and misaligned row offsets. Every row is compared bit-exactly with the
reference engine compiled from the reference (rtk::batch_topk / rtk::topk, batch.hpp:261-367,
engine.hpp:422-443) through oracle/_ref.
"""
import numpy as np
import pytest

import oracle as O
from tests.test_gpu_parity import assert_same

pytestmark = pytest.mark.gpu


def _row(rng, n, dtype):
    kind = rng.integers(0, 6)
    if kind == 0:
        x = rng.random(n, dtype=np.float32)
    elif kind == 1:
        x = rng.standard_normal(n).astype(np.float32)
    elif kind == 2:
        x = (rng.zipf(1.3, n) % 1000).astype(np.float32)
    elif kind == 3:
        x = rng.integers(0, 7, n).astype(np.float32)  # heavy ties
    elif kind == 4:
        x = np.sort(rng.standard_normal(n).astype(np.float32))
        if rng.integers(0, 2):
            x = x[::-1].copy()
    else:
        x = rng.standard_normal(n).astype(np.float32)
        m = max(1, n // 97)
        x[rng.integers(0, n, m)] = np.float32("nan")
        x[rng.integers(0, n, m)] = np.float32("inf")
        x[rng.integers(0, n, m)] = -np.float32("inf")
    if dtype == np.uint32:
        return x.view(np.uint32).copy() if kind != 3 else rng.integers(0, 5, n).astype(np.uint32)
    return x


def _k(rng, n):
    c = rng.integers(0, 5)
    if c == 0:
        return 1
    if c == 1:
        return int(rng.integers(1, min(n, 600) + 1))
    if c == 2:
        return int(rng.integers(1, min(n, 4096) + 1))
    if c == 3:
        return int(rng.integers(max(1, n // 2), n + 1))  # dense
    return int(rng.integers(1, n + 1))


@pytest.mark.parametrize("case", range(24))
def test_fuzz_batches(cuda, case):
    import torch
    import paper_2501_14336_b200 as rtk
    rng = np.random.default_rng(9000 + case)
    dtype = np.float32 if case % 3 else np.uint32
    order = int(case % 2)
    B = int(rng.integers(1, 12))
    lens = [int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 200000), rng.integers(200000, 1 << 20)],
                           p=[0.4, 0.4, 0.2])) for _ in range(B)]
    rows = [_row(rng, n, dtype) for n in lens]
    ks = [_k(rng, n) for n in lens]
    gaps = [int(rng.integers(0, 9)) for _ in range(B)]  # misaligned row starts
    offs, parts, pos = [], [], 0
    for t in range(B):
        parts.append(np.zeros(gaps[t], dtype=dtype))
        pos += gaps[t]
        offs.append(pos)
        parts.append(rows[t])
        pos += lens[t]
    data = np.concatenate(parts)
    exp = O.ref_batch_topk(data, offs, lens, ks, order, grid=8)
    td = torch.from_numpy(data.view(np.int32) if dtype == np.uint32 else data).to(cuda)
    if dtype == np.uint32:
        td = td.view(torch.uint32)
    got = rtk.batch_topk(rtk.BatchInput(td, offs, lens, ks), rtk.SelectionOrder(order))
    for t in range(B):
        gv = got[t].values
        if dtype == np.uint32:
            gv = gv.view(torch.int32).cpu().numpy().view(np.uint32)
        assert_same((gv, got[t].indices, got[t].pivot), exp[t],
                    f"case {case} row {t} n={lens[t]} k={ks[t]} order={order} {dtype.__name__}")


@pytest.mark.parametrize("case", range(12))
def test_fuzz_single_queries(cuda, case):
    # one query per call: the one-CTA path (n <= 2^18), the cluster path (2^18 < n <= 2^21,
    # k <= 512) and the general pipeline, at random n / k / distribution
    import torch
    import paper_2501_14336_b200 as rtk
    from tests.test_gpu_parity import gpu_topk
    rng = np.random.default_rng(7000 + case)
    dtype = np.float32 if case % 4 else np.uint32
    for _ in range(3):
        n = int(rng.choice([rng.integers(1, 1 << 18), rng.integers((1 << 18) + 1, (1 << 21) + 1),
                            rng.integers(1 << 21, 1 << 23)]))
        x = _row(rng, n, dtype)
        k = min(n, int(rng.integers(1, 513))) if rng.integers(0, 2) else _k(rng, n)
        order = int(rng.integers(0, 2))
        assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=8),
                    f"case {case} n={n} k={k} order={order} {dtype.__name__}")

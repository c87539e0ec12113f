"""GPU parity of the single-query cluster kernel (k_row_cluster, rtk_rows.cu): one row with
2^18 < n <= 2^21 and k <= 512 (BASELINE C1 is n = 2^20, k = 256) is selected by ONE 16-CTA
cluster — sampled threshold on CTA 0, slices streamed by all 16 CTAs into CTA 0's candidate
buffer over distributed shared memory, exact k and the sort on CTA 0.

Bit-exact against rtk::topk compiled from the reference (engine.hpp:422-443) on every key mode
the kernel is instantiated for, at the routing boundaries, and on inputs built so that the
kernel's sample misses (m < k) or its candidate buffer overflows (m > 8192): those rows must be
flagged and finished by the exact path (fallback_rows == 1) with the same result.
"""
import numpy as np
import pytest

import oracle as O
from tests.test_gpu_parity import NORMAL, UNIFORM, ZIPF, _check16, _widen16, assert_same, gpu_topk

pytestmark = pytest.mark.gpu


def _sample_positions(n):
    # k_row_cluster's stratified sample: 128 segments of 32 at stride (n - 32) / 127 (16.16 fixed point)
    stride = ((n - 32) << 16) // 127
    seg = (np.arange(128, dtype=np.uint64) * np.uint64(stride)) >> np.uint64(16)
    return (seg[:, None] + np.arange(32, dtype=np.uint64)[None, :]).reshape(-1).astype(np.int64)


@pytest.mark.parametrize("n", [(1 << 18) + 1, 1 << 20, (1 << 20) + 3, 1 << 21])
@pytest.mark.parametrize("kind", [UNIFORM, NORMAL, ZIPF])
@pytest.mark.parametrize("dtype", [np.float32, np.uint32])
def test_row_cluster_parity(cuda, n, kind, dtype):
    import paper_2501_14336_b200 as rtk
    x = O.ref_generate(kind, n, 900 + n % 97 + kind, dtype=dtype, b=1.0)
    for order in (0, 1):
        for k in (1, 7, 256, 512):
            assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=4),
                        f"n={n} kind={kind} {dtype.__name__} order={order} k={k}")


@pytest.mark.parametrize("kind", ["bf16", "f16"])
def test_row_cluster_16bit(cuda, kind):
    import torch
    rng = np.random.default_rng(4242 + (kind == "f16"))
    n = (1 << 20) + 5
    x = torch.from_numpy(rng.standard_normal(n).astype(np.float32))
    t16 = x.to(torch.bfloat16 if kind == "bf16" else torch.float16)
    h = t16.view(torch.int16).numpy().view(np.uint16).copy()
    x32 = _widen16(h, kind)
    for order in (0, 1):
        for k in (1, 256, 512):
            _check16(h, t16, x32, k, order, cuda, f"cluster {kind} order={order} k={k}")


def test_row_cluster_misaligned_view(cuda):
    # a view starting at an odd element: slice bounds and the L2 prefetch round to 16 bytes
    import torch
    import paper_2501_14336_b200 as rtk
    x = O.ref_generate(NORMAL, (1 << 20) + 7, 31, b=1.0)
    t = torch.from_numpy(x).to(cuda)[3:]
    r = rtk.topk(t, 256)
    assert_same((r.values, r.indices, r.pivot), O.ref_topk(x[3:], 256, 0, grid=4), "misaligned view")


def test_row_cluster_ties_and_specials(cuda):
    import paper_2501_14336_b200 as rtk
    n = 1 << 20
    dup = np.full(n, 1.25, dtype=np.float32)
    for k in (1, 300, 512):
        assert_same(gpu_topk(dup, k, 0, cuda), O.ref_topk(dup, k, 0, grid=4), f"all equal k={k}")
    rng = np.random.default_rng(3)
    x = rng.integers(0, 5, n).astype(np.float32)  # five values, ~2^18 copies each
    x[rng.integers(0, n, 64)] = np.float32("nan")
    x[rng.integers(0, n, 64)] = np.float32("inf")
    x[rng.integers(0, n, 64)] = -np.float32("inf")
    x[rng.integers(0, n, 64)] = np.float32(-0.0)
    for order in (0, 1):
        for k in (1, 100, 512):
            assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=4), f"specials o={order} k={k}")


@pytest.mark.parametrize("case", ["sample_miss", "overflow"])
def test_row_cluster_fallback(cuda, case):
    # sample_miss: the sampled positions hold the largest values, so T lands among them and
    # only ~r' elements reach it (m < k). overflow: the sample holds the smallest values, so
    # nearly every element passes T (m > 8192). Both rows must take the exact path.
    import paper_2501_14336_b200 as rtk
    n = 1 << 20
    rng = np.random.default_rng(11 if case == "sample_miss" else 12)
    x = rng.random(n, dtype=np.float32)
    pos = _sample_positions(n)
    if case == "sample_miss":
        x[pos] = 2.0 + rng.random(pos.size, dtype=np.float32)
    else:
        x += 1.0
        x[pos] = 0.0
    for k in (256, 512):
        assert_same(gpu_topk(x, k, 0, cuda), O.ref_topk(x, k, 0, grid=4), f"{case} k={k}")
        assert rtk.last_stats().fallback_rows == 1, case


def test_row_cluster_scaled(cuda):
    # scaled_topk Off / Always / Adaptive(exact trigger) on a C4-like narrow band at n = 2^20
    import torch
    import paper_2501_14336_b200 as rtk
    n, k = 1 << 20, 256
    x = O.ref_generate(UNIFORM, n, 77, a=128.6, b=128.7)
    for mode in (0, 1, 2):
        for order in (0, 1):
            wv, wi, wp, winfo = O.ref_scaled_topk(x, k, order, mode=mode, tau=0.5, seed=9, grid=4)
            info = rtk.ScaleInfo()
            r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), k, rtk.SelectionOrder(order),
                                policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, 9), info=info)
            assert info.scaled == winfo["scaled"]
            assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"scaled mode={mode} order={order}")


def test_row_cluster_replay(cuda):
    # repeated calls (self-cleaning tail, graph-free replay of the same plan) stay exact
    import torch
    import paper_2501_14336_b200 as rtk
    x = O.ref_generate(UNIFORM, 1 << 20, 1)
    t = torch.from_numpy(x).to(cuda)
    want = O.ref_topk(x, 256, 0, grid=4)
    for _ in range(5):
        r = rtk.topk(t, 256)
        assert_same((r.values, r.indices, r.pivot), want, "replay")
    y = x.copy()
    y[12345] = 7.0
    t.copy_(torch.from_numpy(y))
    r = rtk.topk(t, 256)
    assert_same((r.values, r.indices, r.pivot), O.ref_topk(y, 256, 0, grid=4), "rewritten input")


@pytest.mark.parametrize("kind", ["bf16", "f16"])
def test_row_cluster_16bit_every_lane_slot(cuda, kind):
    # each 16-bit step of the stream covers 4 vectors of 8 halves per thread (one 32-bit hit
    # mask); the maxima sit in every slot of a step (found by tools/fuzz_explore.py: with 8
    # vectors per step the upper half of the 64 elements never reached the mask)
    import torch
    import paper_2501_14336_b200 as rtk
    n = (1 << 20) + 6
    rng = np.random.default_rng(5)
    base = torch.from_numpy((rng.random(n, dtype=np.float32) * 0.5).astype(np.float32))
    for pos in (24000, 24000 + 8 * 512 * 5 + 7, n - 3, 3):
        x = base.clone()
        x[pos] = 1000.0
        t16 = x.to(torch.bfloat16 if kind == "bf16" else torch.float16)
        for k in (1, 64):
            r = rtk.topk(t16.to(cuda), k)
            assert int(r.indices[0].item()) == pos, (kind, pos, k)
        h = t16.view(torch.int16).numpy().view(np.uint16).copy()
        _check16(h, t16, _widen16(h, kind), 200, 0, cuda, f"{kind} pos={pos}")

"""CPU: the Philox generator of the n = 2^32 configuration and the streaming verifier.

* The library's host twin (rtk_generate_philox_host) equals the independent plain-C restatement
  in oracle/rtk_verify.c for any index range (unaligned starts, block boundaries, 64-bit indices)
  and for shifted ranges [a, b); the device generator is checked against both on the GPU
  (tests/test_gpu_c5.py).
* A known answer of Philox4x32-10 (Random123's kat_vectors: counter 0, key 0) pins the round
  function itself.
* The streaming verifier accepts the true top-k and rejects every kind of corruption.
"""
import numpy as np
import pytest

import oracle as O
from paper_2501_14336_b200 import rtk as R


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32 10 rounds, counter (0,0,0,0) key (0,0) ->
    # 6627e8d5 e169c58d bc57ac4c 9b00dbd8: elements 0..3 of the seed-0 stream are (w >> 8) * 2^-24
    want = [np.float32((w >> 8) * 2.0 ** -24).view(np.uint32) for w in (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)]
    assert [O.port().rtkv_philox_elem(0, g, 0.0, 1.0) for g in range(4)] == want
    assert list(R.generate_philox_host(4, 0).view(np.uint32)) == want


@pytest.mark.parametrize("seed", [0, 1, 0xDEADBEEF12345678])
@pytest.mark.parametrize("offset,n", [(0, 4096), (3, 1001), ((1 << 32) - 5, 17), ((1 << 35) + 2, 64)])
def test_host_twin_equals_restatement(seed, offset, n):
    got = R.generate_philox_host(n, seed, offset)
    want = O.philox_fill(seed, offset, n)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got = R.generate_philox_host(n, seed, offset, 128.6, 128.7)
    want = O.philox_fill(seed, offset, n, 128.6, 128.7)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.all((want >= np.float32(128.6)) & (want <= np.float32(128.7)))


def test_uniform_range_and_moments():
    x = R.generate_philox_host(1 << 20, 7)
    assert x.min() >= 0.0 and x.max() < 1.0
    assert abs(float(x.mean()) - 0.5) < 2e-3
    assert len(np.unique(x)) > 900000


def _true_topk(x, k, order=0):
    key = x.view(np.uint32).astype(np.uint64)
    key = np.where(key & 0x80000000, ~key & 0xFFFFFFFF, key | 0x80000000)
    if order:
        key = ~key & 0xFFFFFFFF
    idx = np.lexsort((np.arange(x.size), -key.astype(np.int64)))[:k]
    return x[idx], idx.astype(np.uint64)


@pytest.mark.parametrize("order", [0, 1])
def test_streaming_verifier(order):
    n, k, seed = 1 << 20, 5000, 11
    x = O.philox_fill(seed, 0, n, 128.6, 128.7)  # heavy ties: 6.5K distinct values
    v, i = _true_topk(x, k, order)
    ok, msg, st = O.verify_philox_topk(seed, n, k, v, i, order, 128.6, 128.7)
    assert ok, msg
    assert st[0] < k <= st[0] + st[1] and st[1] > 1  # the pivot value is tied
    bad = i.copy()
    bad[-1] = i[-1] + 1 if x[i[-1] + 1] == x[i[-1]] else bad[-1]  # a later tie instead of the lowest
    for name, (vv, ii) in {
        "wrong index": (v, np.where(np.arange(k) == 3, (i[3] + 1) % n, i)),
        "swapped order": (v[[1, 0] + list(range(2, k))], i[[1, 0] + list(range(2, k))]),
        "missing greater": (np.append(v[:-2], v[-1:]), np.append(i[:-2], i[-1:])),
    }.items():
        ok, msg, _ = O.verify_philox_topk(seed, n, len(ii), vv, ii, order, 128.6, 128.7)
        assert not ok, name
    ties = np.nonzero(x == x[i[-1]])[0]
    later = ties[ties > i[-1]]
    if later.size:
        ii = i.copy()
        ii[-1] = later[0]
        ok, msg, _ = O.verify_philox_topk(seed, n, k, v, ii, order, 128.6, 128.7)
        assert not ok and "ties" in msg

"""GPU parity at the BASELINE configurations themselves (the shapes bench.py times).

Every case is bit-exact (value bits, u64 indices, pivot) against the reference compiled in place
(oracle/_ref): rtk::topk (engine.hpp:422-443), rtk::batch_topk (batch.hpp:261-367) and
rtk::scaled_topk (scaling.hpp:42-86), run with grid_size = the host's cores. Inputs come from the
reference's own generators (datagen.hpp:71-141) with the seeds bench.py and SURVEY §8(d) name.

  C2  n = 2^28 U[0,1) seed 1, k in {1, 2^8, 2^14, 2^20}        (BASELINE configs[1])
  C3  256 x 128256 N(0,1) rows (seeds 100 + t), k in {1, 50, 4096, 4097, 20000, 64127, 64128,
      128256}: every routing switch (one-CTA rows <= 4096, sampled general path, dense k >= n/2
      LSD path) on both sides of its boundary                   (BASELINE configs[2])
      + the Peaked rows of SURVEY §8(d) (DistKind::Peaked, mass 0.8, modes 1-2, datagen.hpp:93-104)
  C2  Normal(0, 1) and Zipf(1.1) at n = 2^28, k = 2^20
  C4  n = 2^26 U[128.6, 128.7) seed 5 + n, k = 2^16, scale Off / Always / Adaptive (tau 0.5,
      seed 31)                                                  (BASELINE configs[3])
"""
import os

import numpy as np
import pytest

import oracle as O
from tests.test_gpu_parity import NORMAL, PEAKED, UNIFORM, ZIPF, assert_same

pytestmark = pytest.mark.gpu

CORES = os.cpu_count() or 4


@pytest.fixture(scope="module")
def c2(cuda):
    import torch
    x = O.ref_generate(UNIFORM, 1 << 28, 1)
    t = torch.from_numpy(x).to(cuda)
    yield x, t
    del t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [1, 1 << 8, 1 << 14, 1 << 20])
def test_c2_headline(c2, k):
    import paper_2501_14336_b200 as rtk
    x, t = c2
    r = rtk.topk(t, k)
    assert_same((r.values, r.indices, r.pivot), O.ref_topk(x, k, 0, grid=CORES), f"C2 k={k}")
    assert rtk.last_stats().fallback_rows == 0  # the sampled single-read path, not the exact one


@pytest.fixture(scope="module")
def c3(cuda):
    import torch
    V, B = 128256, 256
    data = np.concatenate([O.ref_generate(NORMAL, V, 100 + t, b=1.0) for t in range(B)])
    t = torch.from_numpy(data).to(cuda).view(B, V)
    yield data, t, B, V
    del t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [1, 50, 4096, 4097, 20000, 64127, 64128, 128256])
def test_c3_headline(c3, k):
    import paper_2501_14336_b200 as rtk
    data, t, B, V = c3
    r = rtk.batch_topk_dense(t, k)
    exp = O.ref_batch_topk(data, [i * V for i in range(B)], [V] * B, [k] * B, 0, grid=CORES)
    gv, gi, gp = r.values.cpu().numpy(), r.indices.cpu().numpy(), r.pivot.cpu().numpy()
    for row in range(B):
        assert_same((gv[row], gi[row], gp[row]), exp[row], f"C3 row {row} k={k}")


@pytest.fixture(scope="module")
def c4(cuda):
    import torch
    n = 1 << 26
    x = O.ref_generate(UNIFORM, n, 5 + n, a=128.6, b=128.7)
    t = torch.from_numpy(x).to(cuda)
    yield x, t
    del t
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_c4_headline(c4, mode):
    import paper_2501_14336_b200 as rtk
    x, t = c4
    k = 1 << 16
    wv, wi, wp, winfo = O.ref_scaled_topk(x, k, 0, mode=mode, tau=0.5, seed=31, grid=CORES)
    info = rtk.ScaleInfo()
    r = rtk.scaled_topk(t, k, policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, 31), info=info)
    assert info.scaled == winfo["scaled"]
    assert info.a_index == (winfo["a_index"] if winfo["scaled"] else 0)
    assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"C4 mode={mode}")
    if mode == 2:  # the sampled trigger guess was verified exact in the selection pass: no extra pass
        assert rtk.last_stats().passes == 0


@pytest.mark.parametrize("k", [50, 4096, 128256])
def test_c3_peaked_rows(cuda, k):
    import torch
    import paper_2501_14336_b200 as rtk
    V, B = 128256, 64
    data = np.concatenate([O.ref_generate(PEAKED, V, 100 + t, mass=0.8, modes=1 + t % 2) for t in range(B)])
    r = rtk.batch_topk_dense(torch.from_numpy(data).to(cuda).view(B, V), k)
    exp = O.ref_batch_topk(data, [i * V for i in range(B)], [V] * B, [k] * B, 0, grid=CORES)
    gv, gi, gp = r.values.cpu().numpy(), r.indices.cpu().numpy(), r.pivot.cpu().numpy()
    for row in range(B):
        assert_same((gv[row], gi[row], gp[row]), exp[row], f"C3 peaked row {row} k={k}")


@pytest.mark.parametrize("kind", [NORMAL, ZIPF])
def test_c2_other_distributions(cuda, kind):
    import torch
    import paper_2501_14336_b200 as rtk
    x = O.ref_generate(kind, 1 << 28, 2 + kind, b=1.0)
    t = torch.from_numpy(x).to(cuda)
    r = rtk.topk(t, 1 << 20)
    assert_same((r.values, r.indices, r.pivot), O.ref_topk(x, 1 << 20, 0, grid=CORES), f"C2 kind={kind}")
    del t
    torch.cuda.empty_cache()

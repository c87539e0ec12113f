"""GPU: the C++ boundary beyond the single-query entry points.

* rtk_topk_sharded over a real NCCL communicator. The box has one GPU, so the
  communicator has one rank (NCCL refuses two ranks on one device); the full path still runs —
  local top-k, ncclAllGather, gap-closing of short shards, final select, global index remap —
  and must equal rtk::topk on the whole query. World > 1 host logic: tests/test_sharded_cpu.py.
* The retargeted acceptance program (tests/cpp/acceptance_b200.cpp) compiled against the drop-in
  header include/rtk/topk.hpp and run: criteria 1, 2, 6, 7, 8 of acceptance_test.cpp.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from tests.test_gpu_parity import UNIFORM, ZIPF, assert_same

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CORES = os.cpu_count() or 4


@pytest.fixture(scope="module")
def comm1(cuda):
    from paper_2501_14336_b200 import sharded as SH
    c = SH.NcclComm(0, 1, 0, uid=SH.unique_id())
    yield c
    c.destroy()


@pytest.mark.parametrize("kind", [UNIFORM, ZIPF])
@pytest.mark.parametrize("k", [1, 4096, 1 << 16])
@pytest.mark.parametrize("order", [0, 1])
def test_topk_sharded_nccl_world1(cuda, comm1, kind, k, order):
    import torch
    from paper_2501_14336_b200 import sharded as SH
    n = (1 << 22) + 5
    x = O.ref_generate(kind, n, 31 + kind + k, b=1.0)
    r = SH.topk_sharded(torch.from_numpy(x).to(cuda), k, [n], comm1, order)
    assert_same((r.values, r.indices, r.pivot.cpu().numpy()[0]), O.ref_topk(x, k, order, grid=CORES),
                f"sharded kind={kind} k={k} order={order}")


def test_topk_sharded_dtypes_and_short_shard(cuda, comm1):
    import torch
    from paper_2501_14336_b200 import sharded as SH
    # u32 keys, and k > shard length is refused like rtk::topk (k outside [1, n])
    u = O.ref_generate(UNIFORM, 100000, 3, dtype=np.uint32)
    t = torch.from_numpy(u.view(np.int32)).to(cuda).view(torch.uint32)
    r = SH.topk_sharded(t, 777, [u.size], comm1, 0)
    wv, wi, wp = O.ref_topk(u, 777, 0, grid=CORES)
    assert np.array_equal(r.values.view(torch.int32).cpu().numpy().view(np.uint32), wv)
    assert np.array_equal(r.indices.cpu().numpy().astype(np.uint64), wi)
    with pytest.raises(IndexError):
        SH.topk_sharded(t, u.size + 1, [u.size], comm1, 0)
    with pytest.raises(ValueError, match="shard holds"):
        SH.topk_sharded(t, 5, [u.size + 1], comm1, 0)


def test_cpp_acceptance_program(cuda, tmp_path):
    exe = tmp_path / "acceptance_b200"
    lib = os.path.join(ROOT, "paper_2501_14336_b200")
    ref = os.path.join(ROOT, "oracle", "_ref")
    b = subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "acceptance_b200.cpp"), "-o", str(exe), "-L", lib,
                        "-lrtk_b200", "-L", ref, "-lrtk_ref", f"-Wl,-rpath,{lib}:{ref}"],
                       capture_output=True, text=True, timeout=300)
    assert b.returncode == 0, b.stderr[-3000:]
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr[-2000:]
    assert "all acceptance criteria passed" in p.stdout

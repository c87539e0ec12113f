"""CPU, world_size 2 over gloo: host logic of the multi-GPU paths.

rtk_topk_sharded (csrc/rtk_sharded.cpp) runs, per rank: local top-k of the shard -> all-gather of
every rank's min(k, shard_n) candidates -> final select with the position in the gathered array
as tie-break index -> remap to global indices. Here the same steps run with the C restatement
(oracle) as the local top-k and the final select, and a real torch.distributed all-gather over
gloo as the exchange; the result must equal the single-device reference on the whole query,
including ties that straddle the shard boundary. The NCCL bootstrap (rank 0's ncclUniqueId
broadcast to every rank, sharded.bootstrap_unique_id) runs over gloo as well.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2501_14336_b200 import sharded as SH


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_gather(vals, idx):
    world = dist.get_world_size()
    n = torch.tensor([len(vals)], dtype=torch.int64)
    lens = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(lens, n)
    lens = [int(t.item()) for t in lens]
    m = max(lens)
    pv = torch.zeros(m, dtype=torch.int64)
    pi = torch.zeros(m, dtype=torch.int64)
    pv[: len(vals)] = torch.from_numpy(np.asarray(vals).view(np.uint32).astype(np.int64))
    pi[: len(idx)] = torch.from_numpy(np.asarray(idx).astype(np.int64))
    gv = [torch.zeros(m, dtype=torch.int64) for _ in range(world)]
    gi = [torch.zeros(m, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gv, pv)
    dist.all_gather(gi, pi)
    vb = [gv[g][: lens[g]].numpy().astype(np.uint32).view(np.float32) for g in range(world)]
    ib = [gi[g][: lens[g]].numpy().astype(np.uint64) for g in range(world)]
    return vb, ib


def _oracle_merge(cv, ci, block_len, shard_base, k):
    # rtk_merge_shards' rule: top-k of the concatenation with the POSITION as tie-break index
    v, pos, piv = O.port_topk(np.ascontiguousarray(cv, dtype=np.float32), k)
    gidx = SH.merge_positions_to_global(pos.tolist(), block_len, ci, shard_base)
    return v, np.array(gidx, dtype=np.uint64), piv


def _sharded_steps(x_local, k, n_total, rank, world):
    # the steps of rtk_topk_sharded with the oracle for the two selects
    start, length = SH.shard_bounds(n_total, world, rank)
    assert length == len(x_local)
    v, i, _ = O.port_topk(x_local, min(k, length))
    vb, ib = _gloo_gather(v, i)
    block_len = [len(b) for b in vb]
    shard_base = [SH.shard_bounds(n_total, world, g)[0] for g in range(world)]
    return _oracle_merge(np.concatenate(vb), np.concatenate(ib), block_len, shard_base, k)


def _worker(rank, world, port, x, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, l = SH.shard_bounds(len(x), world, rank)
        v, i, piv = _sharded_steps(x[s:s + l], k, len(x), rank, world)
        q.put((rank, v.view(np.uint32).tolist(), i.tolist()))
    finally:
        dist.destroy_process_group()


def _run(x, k, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_shard_bounds_cover():
    for n in [1, 7, 100, 2**20 + 3]:
        for w in [1, 2, 3, 8]:
            spans = [SH.shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and sum(l for _, l in spans) == n
            for (s0, l0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + l0 == s1
    assert [SH.row_shard(256, 8, r) for r in (0, 7)] == [(0, 32), (224, 256)]


@pytest.mark.parametrize("k", [1, 100, 5000])
def test_sharded_equals_single_device_gloo(k):
    x = np.random.default_rng(7).random(20001, dtype=np.float32)
    want_v, want_i, _ = O.port_topk(x, k)
    for rank, v, i in _run(x, k):
        assert v == want_v.view(np.uint32).tolist() and i == want_i.tolist(), rank


def test_sharded_ties_across_shard_boundary_gloo():
    # every value appears on both shards: the global tie rule (lowest indices first) must hold
    x = np.tile(np.array([3.0, 1.0, 3.0, 2.0], dtype=np.float32), 501)
    k = 700
    want_v, want_i, _ = O.port_topk(x, k)
    for rank, v, i in _run(x, k):
        assert i == want_i.tolist(), rank


def _boot_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        made = []

        def make_id():
            made.append(rank)
            return bytes((rank * 31 + j) & 0xFF for j in range(128))

        uid = SH.bootstrap_unique_id(rank, make_id=make_id)
        q.put((rank, uid, made))
    finally:
        dist.destroy_process_group()


def test_nccl_bootstrap_broadcasts_rank0_id_gloo():
    # only rank 0 draws the id; every rank ends up with rank 0's 128 bytes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_boot_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = bytes(j & 0xFF for j in range(128))
    assert [o[1] for o in out] == [want, want]
    assert out[0][2] == [0] and out[1][2] == []

"""Multi-GPU partitioning of the top-k path, one process per GPU.

Two strategies, exactly where the path shards naturally:

* ``row_shard``    — batched queries: rank g owns rows [g*B/G, (g+1)*B/G); no collective on the
  hot path (each rank runs rtk_topk_batched on its rows).
* ``topk_sharded`` — one huge query split by contiguous index ranges (``shard_bounds``): the C++
  entry rtk_topk_sharded runs the local top-k of the rank's shard, an ncclAllGather of every
  rank's k (value, local index) candidates and the final select with global indices on every
  rank. The result equals a single-device top-k because the reference's order restricted to
  one shard is that shard's (key desc, index asc) order and shard index ranges increase with
  the rank, so among equal keys the position in the gathered array orders exactly like the
  global index (the tie rule of engine.hpp:387-396).

The NCCL communicator of rtk_topk_sharded is bootstrapped over torch.distributed: rank 0 draws
the ncclUniqueId (rtk_nccl_get_unique_id) and broadcasts it; every rank then calls
rtk_nccl_comm_init_rank on its device.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional, Sequence, Tuple

from . import _lib as L


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous index range [start, start+len) of shard `rank` (remainder to the first ranks)."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def row_shard(B: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [r0, r1) of a batch owned by `rank`."""
    s, l = shard_bounds(B, world, rank)
    return s, s + l


def merge_positions_to_global(pos: Sequence[int], block_len: Sequence[int], cand_idx: Sequence[int],
                              shard_base: Sequence[int]) -> List[int]:
    """Host restatement of the final select's index remap (k_remap_idx): a position in the
    concatenated candidate blocks -> that candidate's shard-local index + its shard's base."""
    starts, acc = [], 0
    for b in block_len:
        starts.append(acc)
        acc += b
    out = []
    for p in pos:
        g = max(i for i, s in enumerate(starts) if s <= p)
        out.append(int(cand_idx[p]) + int(shard_base[g]))
    return out


def _raise(st: int, where: str) -> None:
    from .rtk import _raise as r
    r(st, where)


def unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) from rtk_nccl_get_unique_id."""
    buf = C.create_string_buffer(128)
    _raise(L.load().rtk_nccl_get_unique_id(buf), "rtk_nccl_get_unique_id")
    return buf.raw


def bootstrap_unique_id(rank: int, broadcast: Optional[Callable] = None,
                        make_id: Callable[[], bytes] = unique_id) -> bytes:
    """Rank 0's ncclUniqueId on every rank. broadcast(obj_list) broadcasts a one-element list from
    rank 0 in place (default: torch.distributed.broadcast_object_list on the default group)."""
    if broadcast is None:
        import torch.distributed as dist

        def broadcast(lst):
            dist.broadcast_object_list(lst, src=0)
    box = [make_id() if rank == 0 else None]
    broadcast(box)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad ncclUniqueId received from rank 0")
    return bytes(uid)


class NcclComm:
    """An NCCL communicator of `world` ranks for rtk_topk_sharded (one per process and device)."""

    def __init__(self, rank: int, world: int, device: int, uid: Optional[bytes] = None):
        uid = uid if uid is not None else bootstrap_unique_id(rank)
        self.rank, self.world, self.device = rank, world, device
        self.comm = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        _raise(L.load().rtk_nccl_comm_init_rank(C.byref(self.comm), int(world), buf, int(rank), int(device)),
               "rtk_nccl_comm_init_rank")

    def destroy(self) -> None:
        if self.comm:
            _raise(L.load().rtk_nccl_comm_destroy(self.comm), "rtk_nccl_comm_destroy")
            self.comm = C.c_void_p()


def topk_sharded(x_local, k: int, shard_lens: Sequence[int], comm: NcclComm, order: int = 0):
    """Global top-k of a query whose shard of rank comm.rank is the CUDA tensor x_local
    (shard_lens: every rank's shard length, rank order). Returns rtk.TopKResult with global
    u64 indices, the same on every rank (rtk_topk_sharded)."""
    import torch
    from . import rtk as R
    x = x_local.contiguous()
    if len(shard_lens) != comm.world or int(shard_lens[comm.rank]) != x.numel():
        raise ValueError(f"rank {comm.rank}: shard holds {x.numel()} elements, shard_lens says "
                         f"{list(shard_lens)}")
    code = R._dtype_code(x)
    kk = int(k)
    vals = torch.empty(kk, dtype=x.dtype, device=x.device)
    idx = torch.empty(kk, dtype=torch.int64, device=x.device)
    piv = torch.empty(1, dtype=x.dtype, device=x.device)
    sn, p_sn = R._arr64(shard_lens)
    one = lambda v: (C.c_void_p * 1)(v)  # noqa: E731
    st = L.load().rtk_topk_sharded(
        one(R._handle(x.device.index or 0)), one(comm.comm), 1, one(x.data_ptr()), p_sn, int(comm.world),
        kk, code, int(order), one(vals.data_ptr()), one(idx.data_ptr()), one(piv.data_ptr()),
        one(R._stream_ptr(x)))
    _raise(st, "rtk_topk_sharded")
    return R.TopKResult(vals, idx, piv)

"""Multi-GPU partitioning of the top-k path, one process per GPU.

Two strategies, exactly where the path shards naturally:

* ``row_shard``   — batched queries: rank g owns rows [g*B/G, (g+1)*B/G); no collective on the
  hot path (each rank runs rtk_topk_batched on its rows).
* ``sharded_topk`` — one huge query split by contiguous index ranges: every rank runs the local
  top-k of its shard (rtk_topk, canonical order), the k candidates of every rank are
  all-gathered (NCCL on GPUs, gloo in the CPU tests) and every rank merges them with
  rtk_merge_shards. The result is identical to a single-device top-k because the reference's
  order restricted to one shard is that shard's (key desc, index asc) order and shard index
  ranges are increasing in rank order, so among equal keys the position in the gathered array
  orders exactly like the global index (the tie rule of engine.hpp:387-396).

The local top-k, the gather and the merge are injectable so the host logic can be exercised on
CPU with the oracle (tests/test_sharded_cpu.py); the product path uses the CUDA library.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple


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
    """Host restatement of rtk_merge_shards' index remap (for the CPU tests)."""
    starts, acc = [], 0
    for b in block_len:
        starts.append(acc)
        acc += b
    out = []
    for p in pos:
        g = max(i for i, s in enumerate(starts) if s <= p)
        out.append(int(cand_idx[p]) + int(shard_base[g]))
    return out


def sharded_topk(x_local, k: int, n_total: int, rank: int, world: int,
                 local_topk: Optional[Callable] = None, all_gather: Optional[Callable] = None,
                 merge: Optional[Callable] = None):
    """Global top-k of a query whose shard `rank` is x_local (see module docstring).

    local_topk(x, kk) -> (values, local_indices) in canonical order
    all_gather(values, indices) -> (list of value blocks, list of index blocks) in rank order
    merge(cand_vals, cand_idx, block_len, shard_base, k) -> (values, global indices, pivot)
    Defaults: the CUDA library + torch.distributed (NCCL) on the current device.
    """
    start, length = shard_bounds(n_total, world, rank)
    if length != len(x_local):
        raise ValueError(f"rank {rank}: shard holds {len(x_local)} elements, expected {length}")
    kk = min(k, length)
    if local_topk is None:
        from . import rtk as R

        def local_topk(x, kq):
            r = R.topk(x, kq)
            return r.values, r.indices
    if all_gather is None:
        all_gather = _torch_all_gather
    if merge is None:
        from . import rtk as R

        def merge(cv, ci, bl, sb, kq):
            r = R.merge_shards(cv, ci, bl, sb, kq)
            return r.values, r.indices, r.pivot
    vals, idx = local_topk(x_local, kk)
    vblocks, iblocks = all_gather(vals, idx)
    block_len = [len(v) for v in vblocks]
    shard_base = [shard_bounds(n_total, world, g)[0] for g in range(world)]
    cat_v, cat_i = _concat(vblocks), _concat(iblocks)
    return merge(cat_v, cat_i, block_len, shard_base, k)


def _concat(blocks):
    b0 = blocks[0]
    if hasattr(b0, "is_cuda"):
        import torch
        return torch.cat(list(blocks))
    import numpy as np
    return np.concatenate(list(blocks))


def _torch_all_gather(vals, idx):
    """Variable-length all-gather of (values, indices) blocks over torch.distributed."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    n = torch.tensor([vals.numel()], device=vals.device, dtype=torch.int64)
    lens = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(lens, n)
    lens = [int(t.item()) for t in lens]
    m = max(lens)
    pv = torch.zeros(m, dtype=vals.dtype, device=vals.device)
    pi = torch.zeros(m, dtype=idx.dtype, device=idx.device)
    pv[: vals.numel()] = vals
    pi[: idx.numel()] = idx
    gv = torch.empty(world * m, dtype=vals.dtype, device=vals.device)
    gi = torch.empty(world * m, dtype=idx.dtype, device=idx.device)
    dist.all_gather_into_tensor(gv, pv)
    dist.all_gather_into_tensor(gi, pi)
    return ([gv[g * m: g * m + lens[g]] for g in range(world)],
            [gi[g * m: g * m + lens[g]] for g in range(world)])

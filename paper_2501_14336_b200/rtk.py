"""Python mirror of the reference's top-k interface, backed by the sm_100a C-ABI library.

Same names, argument meaning and error behaviour as /root/reference/proj/include/rtk/:

=====================  =========================================  ==========================
here                   reference                                  C-ABI (include/rtk_c.h)
=====================  =========================================  ==========================
SelectionOrder         keycodec.hpp:19                            RTK_LARGEST / RTK_SMALLEST
EngineConfig           engine.hpp:48-68 (validate :61-67)         rtk_cfg, rtk_cfg_validate
TopKResult             engine.hpp:103-108                         out_vals / out_idx / pivot
topk                   engine.hpp:422-443                         rtk_topk / rtk_topk_host
BatchInput             batch.hpp:27-67 (validate :40-53)          descriptor arrays
BatchOptions           batch.hpp:133-136                          rtk_batch_opts
batch_topk             batch.hpp:261-367                          rtk_topk_batched[_host]
ScaleMode/ScalePolicy  scaling.hpp:20-27                          mode / tau / seed
ScaleInfo              scaling.hpp:29-33                          rtk_scale_info
scaled_topk            scaling.hpp:42-86                          rtk_topk_scaled[_host]
rank_out_of_range      engine.hpp:31-33 (std::out_of_range)       RTK_RANK_OUT_OF_RANGE
invariant_violation    engine.hpp:35-37 (std::logic_error)        RTK_INVARIANT_VIOLATION
empty_input_error      engine.hpp:39-41 (std::invalid_argument)   RTK_EMPTY_INPUT
=====================  =========================================  ==========================

CUDA tensors go through the device-pointer entry points (outputs are CUDA tensors on the same
device); numpy arrays / CPU tensors go through the host entry points (copies included; outputs
are numpy arrays). Values are returned bit-exact, indices as int64 (u64 in the C-ABI).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Any, List, Optional, Sequence

import numpy as np

from . import _lib as L


# ---- exceptions (engine.hpp:31-41) -------------------------------------------------------
class rank_out_of_range(IndexError):
    """std::out_of_range subclass in the reference."""


class invariant_violation(RuntimeError):
    """std::logic_error subclass in the reference."""


class empty_input_error(ValueError):
    """std::invalid_argument subclass in the reference."""


class cuda_error(RuntimeError):
    pass


def _raise(status: int, where: str = "") -> None:
    if status == L.RTK_OK:
        return
    msg = L.last_error() or where
    if status == L.RTK_EMPTY_INPUT:
        raise empty_input_error(msg)
    if status == L.RTK_RANK_OUT_OF_RANGE:
        raise rank_out_of_range(msg)
    if status == L.RTK_INVARIANT_VIOLATION:
        raise invariant_violation(msg)
    if status == L.RTK_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == L.RTK_OUT_OF_MEMORY:
        raise MemoryError(msg)
    if status == L.RTK_IO_ERROR:
        raise RuntimeError(msg)
    raise cuda_error(f"status {status}: {msg}")


# ---- config types ------------------------------------------------------------------------
class SelectionOrder(enum.IntEnum):
    Largest = 0
    Smallest = 1


class BufferPolicy(enum.IntEnum):
    Naive = 0
    FlushEfficient = 1


@dataclass
class EngineConfig:
    d: int = 12
    block_size: int = 1024
    grid_size: int = 4
    buffer_policy: BufferPolicy = BufferPolicy.FlushEfficient
    pack_size: int = 16
    hierarchical_atomics: bool = True
    filter_fixed_ceiling: int = 4096

    def radix(self) -> int:
        return 1 << self.d

    def validate(self) -> None:
        if self.d < 1 or self.d > 16:
            raise ValueError("digit width must be in [1, 16]")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.grid_size < 1:
            raise ValueError("grid_size must be >= 1")
        if self.pack_size < 4 or (self.pack_size & (self.pack_size - 1)) != 0:
            raise ValueError("pack_size must be a power of two >= element width")

    def _c(self) -> L.rtk_cfg:
        return L.rtk_cfg(int(self.d), int(self.block_size), int(self.grid_size),
                         int(self.buffer_policy), int(self.pack_size),
                         int(bool(self.hierarchical_atomics)), int(self.filter_fixed_ceiling))


@dataclass
class BatchOptions:
    rescheduling: bool = True
    padding: bool = True


@dataclass
class BatchRunInfo:
    task_passes: List[int] = field(default_factory=list)
    phase_b_rounds: int = 0


class ScaleMode(enum.IntEnum):
    Off = 0
    Always = 1
    Adaptive = 2


@dataclass
class ScalePolicy:
    mode: ScaleMode = ScaleMode.Off
    trigger_fraction: float = 0.5
    seed: int = 0


@dataclass
class ScaleInfo:
    scaled: bool = False
    a_s: float = 0.0
    a_index: int = 0


@dataclass
class Instrumentation:
    """Work counters of the last call (subset of engine.hpp:74-101 with GPU meaning)."""
    passes: int = 0
    elements_scanned: int = 0
    candidates: int = 0
    fallback_rows: int = 0
    kernel_launches: int = 0
    compact_ms: float = 0.0
    total_ms: float = 0.0
    deep_levels: int = 0


class TopKResult:
    """rtk::TopKResult (engine.hpp:103-108). For device results the pivot stays on the device
    until first read (no host synchronisation inside the call)."""

    __slots__ = ("values", "indices", "_pivot", "_pivot_fn")

    def __init__(self, values, indices, pivot=None, pivot_fn=None):
        self.values, self.indices = values, indices
        self._pivot, self._pivot_fn = pivot, pivot_fn

    @property
    def pivot(self):
        if self._pivot_fn is not None:
            self._pivot, self._pivot_fn = self._pivot_fn(), None
        return self._pivot

    def __iter__(self):
        return iter((self.values, self.indices, self.pivot))

    def __repr__(self):
        return f"TopKResult(values={self.values!r}, indices={self.indices!r}, pivot={self.pivot!r})"


# ---- handle management -------------------------------------------------------------------
_handles: dict = {}


def _handle(device: int) -> C.c_void_p:
    h = _handles.get(device)
    if h is None:
        lib = L.load()
        h = C.c_void_p()
        _raise(lib.rtk_handle_create(C.byref(h), int(device)), "rtk_handle_create")
        _handles[device] = h
    return h


def last_stats(device: int = 0) -> Instrumentation:
    st = L.rtk_stats()
    _raise(L.load().rtk_get_stats(_handle(device), C.byref(st)))
    return Instrumentation(st.passes, st.elements_scanned, st.candidates, st.fallback_rows,
                           st.kernel_launches, st.compact_ms, st.total_ms, st.deep_levels)


def set_option(name: str, value: int, device: int = 0) -> None:
    """rtk_set_option: test switches of the device's handle ("force_exact", "force_deep")."""
    _raise(L.load().rtk_set_option(_handle(device), name.encode(), int(value)), "rtk_set_option")


def set_timing(on: bool, device: int = 0) -> None:
    """Timing mode (rtk_set_timing): no graph replay, CUDA events around k_compact every call."""
    _raise(L.load().rtk_set_timing(_handle(device), int(bool(on))))


@dataclass
class BenchResult:
    """Per-step times of an rtk_bench_* run: device_ms (CUDA events the engine records on the
    launching stream around its device work) and host_ms (wall time of each C entry-point call,
    which returns after the device's completion signal)."""
    device_ms: List[float]
    host_ms: List[float]

    @property
    def median_ms(self) -> float:
        return float(np.median(self.device_ms))

    @property
    def median_host_ms(self) -> float:
        return float(np.median(self.host_ms))


def _steps(steps: int):
    return (C.c_float * int(steps))(), (C.c_float * int(steps))(), C.c_float()


def _flush_args(flush):
    return C.c_void_p(flush.data_ptr() if flush is not None else 0), int(flush.numel() if flush is not None else 0)


def bench_topk(x, k: int, steps: int, warmup: int = 3, order: SelectionOrder = SelectionOrder.Largest,
               cfg: Optional[EngineConfig] = None, flush=None) -> BenchResult:
    """rtk_bench_topk: `steps` back-to-back rtk_topk calls issued from C on x's current stream
    (device-resident input); `flush` (a CUDA byte tensor larger than L2) is overwritten before
    every step outside the clocks."""
    import torch
    cfg = cfg or EngineConfig()
    lib = L.load()
    x = x.contiguous()
    kk = int(k)
    vals = torch.empty(kk, dtype=x.dtype, device=x.device)
    idx = torch.empty(kk, dtype=torch.int64, device=x.device)
    piv = torch.empty(1, dtype=x.dtype, device=x.device)
    per, host, mean = _steps(steps)
    c = cfg._c()
    fp, fb = _flush_args(flush)
    st = lib.rtk_bench_topk(_handle(x.device.index or 0), C.c_void_p(x.data_ptr()), x.numel(), kk,
                            _dtype_code(x), int(order), C.c_void_p(vals.data_ptr()), C.c_void_p(idx.data_ptr()),
                            C.c_void_p(piv.data_ptr()), C.byref(c), _stream_ptr(x), fp, fb, int(warmup), int(steps),
                            per, host, C.byref(mean))
    _raise(st, "rtk_bench_topk")
    return BenchResult([float(v) for v in per], [float(v) for v in host])


def bench_scaled(x, k: int, steps: int, warmup: int = 3, policy: Optional[ScalePolicy] = None,
                 order: SelectionOrder = SelectionOrder.Largest, cfg: Optional[EngineConfig] = None,
                 flush=None) -> BenchResult:
    """rtk_bench_scaled: `steps` back-to-back rtk_topk_scaled calls issued from C on x's current
    stream (device-resident f32 input)."""
    import torch
    cfg = cfg or EngineConfig()
    policy = policy or ScalePolicy()
    lib = L.load()
    x = x.contiguous()
    if x.dtype != torch.float32:
        raise TypeError("scaled_topk is defined for float32 only")
    kk = int(k)
    vals = torch.empty(kk, dtype=x.dtype, device=x.device)
    idx = torch.empty(kk, dtype=torch.int64, device=x.device)
    piv = torch.empty(1, dtype=x.dtype, device=x.device)
    per, host, mean = _steps(steps)
    c = cfg._c()
    fp, fb = _flush_args(flush)
    st = lib.rtk_bench_scaled(_handle(x.device.index or 0), C.c_void_p(x.data_ptr()), x.numel(), kk, int(order),
                              int(policy.mode), float(policy.trigger_fraction),
                              int(policy.seed) & 0xFFFFFFFFFFFFFFFF, C.c_void_p(vals.data_ptr()),
                              C.c_void_p(idx.data_ptr()), C.c_void_p(piv.data_ptr()), C.byref(c), _stream_ptr(x),
                              fp, fb, int(warmup), int(steps), per, host, C.byref(mean))
    _raise(st, "rtk_bench_scaled")
    return BenchResult([float(v) for v in per], [float(v) for v in host])


def bench_batch_dense(x, k: int, steps: int, warmup: int = 3, flush=None,
                      order: SelectionOrder = SelectionOrder.Largest,
                      cfg: Optional[EngineConfig] = None) -> BenchResult:
    """rtk_bench_batched over a dense [B, V] CUDA tensor: `steps` rtk_topk_batched calls issued
    from C; `flush` (a CUDA byte tensor) is overwritten between steps outside the clocks."""
    import torch
    cfg = cfg or EngineConfig()
    lib = L.load()
    x = x.contiguous()
    B, V = x.shape
    offs, p_off = _arr64(np.arange(B, dtype=np.uint64) * V)
    lens, p_len = _arr64(np.full(B, V, dtype=np.uint64))
    kks, p_ks = _arr64(np.full(B, k, dtype=np.uint64))
    oo, p_oo = _arr64(np.arange(B, dtype=np.uint64) * k)
    vals = torch.empty((B, k), dtype=x.dtype, device=x.device)
    idx = torch.empty((B, k), dtype=torch.int64, device=x.device)
    piv = torch.empty(B, dtype=x.dtype, device=x.device)
    per, host, mean = _steps(steps)
    c = cfg._c()
    fp, fb = _flush_args(flush)
    st = lib.rtk_bench_batched(_handle(x.device.index or 0), C.c_void_p(x.data_ptr()), x.numel(), p_off, p_len,
                               p_ks, B, _dtype_code(x), int(order), C.c_void_p(vals.data_ptr()),
                               C.c_void_p(idx.data_ptr()), p_oo, C.c_void_p(piv.data_ptr()), C.byref(c),
                               _stream_ptr(x), fp, fb, int(warmup), int(steps), per, host, C.byref(mean))
    _raise(st, "rtk_bench_batched")
    return BenchResult([float(v) for v in per], [float(v) for v in host])


def _is_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _dtype_code(x) -> int:
    """C-ABI dtype code: 0 f32, 1 u32, 2 f16 (io.hpp:3's code), 3 bf16."""
    if _is_cuda(x) or hasattr(x, "dtype") and "torch" in type(x).__module__:
        import torch
        if x.dtype == torch.float32:
            return 0
        if x.dtype == torch.uint32:
            return 1
        if x.dtype == torch.float16:
            return 2
        if x.dtype == torch.bfloat16:
            return 3
        # the reference defines float and uint32 keys only (keycodec.hpp:55-81): signed int32
        # would rank negative values above positive ones under the u32 codec, so it is refused
        raise TypeError(f"unsupported dtype {x.dtype} (float32, uint32, float16, bfloat16)")
    a = np.asarray(x)
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.uint32:
        return 1
    if a.dtype == np.float16:
        return 2
    raise TypeError(f"unsupported dtype {a.dtype}")


def _stream_ptr(t) -> C.c_void_p:
    import torch
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _np_scalar(bits: int, dtype_code: int):
    if dtype_code == 2:
        return np.array([bits & 0xFFFF], dtype=np.uint16).view(np.float16)[0]
    arr = np.array([bits], dtype=np.uint32)
    return arr.view(np.float32)[0] if dtype_code == 0 else arr[0]


def _arr64(v: Sequence[int]):
    a = np.ascontiguousarray(np.asarray(v, dtype=np.uint64))
    return a, a.ctypes.data_as(L.P64)


# ---- entry points ------------------------------------------------------------------------
def topk(input, k: int, order: SelectionOrder = SelectionOrder.Largest,
         cfg: Optional[EngineConfig] = None) -> TopKResult:
    """rtk::topk (engine.hpp:422-443): k selected elements in (key desc, index asc) order."""
    cfg = cfg or EngineConfig()
    lib = L.load()
    code = _dtype_code(input)
    c = cfg._c()
    if _is_cuda(input):
        import torch
        x = input.contiguous()
        n = x.numel()
        dev = x.device.index or 0
        kk = max(int(k), 0)
        vals = torch.empty(kk, dtype=x.dtype, device=x.device)
        idx = torch.empty(kk, dtype=torch.int64, device=x.device)
        piv = torch.empty(1, dtype=x.dtype, device=x.device)
        st = lib.rtk_topk(_handle(dev), C.c_void_p(x.data_ptr() if n else 0), n, int(k), code,
                          int(order), C.c_void_p(vals.data_ptr()), C.c_void_p(idx.data_ptr()),
                          C.c_void_p(piv.data_ptr()), C.byref(c), _stream_ptr(x))
        _raise(st, "rtk_topk")
        if code in (0, 2, 3):
            return TopKResult(vals, idx, pivot_fn=lambda: piv[0].item())
        return TopKResult(vals, idx, pivot_fn=lambda: int(piv.view(torch.int32)[0].item()) & 0xFFFFFFFF)
    a = np.ascontiguousarray(input.numpy() if hasattr(input, "numpy") else np.asarray(input))
    n = a.size
    kk = max(int(k), 0)
    vals = np.empty(kk, dtype=a.dtype)
    idx = np.empty(kk, dtype=np.uint64)
    piv = np.zeros(1, dtype=np.uint32)
    st = lib.rtk_topk_host(_handle(0), C.c_void_p(a.ctypes.data if n else 0), n, int(k), code,
                           int(order), C.c_void_p(vals.ctypes.data), C.c_void_p(idx.ctypes.data),
                           C.c_void_p(piv.ctypes.data), C.byref(c))
    _raise(st, "rtk_topk_host")
    return TopKResult(vals, idx, _np_scalar(int(piv[0]), code))


@dataclass
class BatchInput:
    """rtk::BatchInput (batch.hpp:27-67): concatenated payload + per-task descriptors."""
    data: Any
    offsets: List[int]
    lengths: List[int]
    ks: List[int]

    def task_count(self) -> int:
        return len(self.lengths)

    def task_view(self, i: int):
        return self.data[self.offsets[i]:self.offsets[i] + self.lengths[i]]

    def validate(self) -> None:
        if not self.lengths:
            raise ValueError("batch: no tasks")
        if len(self.offsets) != len(self.lengths) or len(self.ks) != len(self.lengths):
            raise ValueError("batch: descriptor arrays disagree")
        size = len(self.data)
        for i in range(len(self.lengths)):
            nxt = self.offsets[i + 1] if i + 1 < len(self.offsets) else size
            if self.offsets[i] + self.lengths[i] > nxt:
                raise ValueError(f"batch: task {i} overlaps its successor")
            if self.ks[i] == 0 or self.ks[i] > self.lengths[i]:
                raise ValueError(f"batch: task {i} has k outside [1, n]")

    @staticmethod
    def concatenate(tasks: Sequence[Any], ks: Sequence[int]) -> "BatchInput":
        offsets, lengths, at = [], [], 0
        for t in tasks:
            offsets.append(at)
            lengths.append(len(t))
            at += len(t)
        if tasks and _is_cuda(tasks[0]):
            import torch
            data = torch.cat([t.reshape(-1) for t in tasks])
        else:
            data = np.concatenate([np.asarray(t).reshape(-1) for t in tasks]) if tasks else np.zeros(0, np.float32)
        b = BatchInput(data, offsets, lengths, list(ks))
        b.validate()
        return b


def batch_topk(batch: BatchInput, order: SelectionOrder = SelectionOrder.Largest,
               cfg: Optional[EngineConfig] = None, opts: Optional[BatchOptions] = None,
               info: Optional[BatchRunInfo] = None) -> List[TopKResult]:
    """rtk::batch_topk (batch.hpp:261-367): one TopKResult per task, each equal to topk."""
    cfg = cfg or EngineConfig()
    opts = opts or BatchOptions()
    lib = L.load()
    B = len(batch.lengths)
    offs, p_off = _arr64(batch.offsets)
    lens, p_len = _arr64(batch.lengths)
    ks, p_ks = _arr64(batch.ks)
    oo = np.zeros(max(B, 1), dtype=np.uint64)
    if B:
        oo[1:B] = np.cumsum(ks[:-1])
    p_oo = oo.ctypes.data_as(L.P64)
    total = int(ks.sum()) if B else 0
    c = cfg._c()
    o = L.rtk_batch_opts(int(opts.rescheduling), int(opts.padding))
    code = _dtype_code(batch.data)
    if _is_cuda(batch.data):
        import torch
        x = batch.data.contiguous()
        vals = torch.empty(total, dtype=x.dtype, device=x.device)
        idx = torch.empty(total, dtype=torch.int64, device=x.device)
        piv = torch.empty(max(B, 1), dtype=x.dtype, device=x.device)
        st = lib.rtk_topk_batched(_handle(x.device.index or 0), C.c_void_p(x.data_ptr()), x.numel(),
                                  p_off, p_len, p_ks, B, code, int(order),
                                  C.c_void_p(vals.data_ptr()), C.c_void_p(idx.data_ptr()), p_oo,
                                  C.c_void_p(piv.data_ptr()), C.byref(c), C.byref(o), _stream_ptr(x))
        _raise(st, "rtk_topk_batched")
        pivs = piv.cpu()
    else:
        a = np.ascontiguousarray(batch.data.numpy() if hasattr(batch.data, "numpy") else np.asarray(batch.data))
        vals = np.empty(total, dtype=a.dtype)
        idx = np.empty(total, dtype=np.uint64)
        pivs = np.empty(max(B, 1), dtype=a.dtype)
        st = lib.rtk_topk_batched_host(_handle(0), C.c_void_p(a.ctypes.data), a.size, p_off, p_len,
                                       p_ks, B, code, int(order), C.c_void_p(vals.ctypes.data),
                                       C.c_void_p(idx.ctypes.data), p_oo, C.c_void_p(pivs.ctypes.data),
                                       C.byref(c), C.byref(o))
        _raise(st, "rtk_topk_batched_host")
    kl = [int(v) for v in ks]
    if hasattr(vals, "split"):
        vs, ix = vals.split(kl), idx.split(kl)
        pl = pivs.tolist()
    else:
        cut = np.cumsum(kl)[:-1] if B else []
        vs, ix = np.split(vals, cut), np.split(idx, cut)
        pl = list(pivs[:B])
    out = [TopKResult(vs[t], ix[t], pl[t]) for t in range(B)]
    if info is not None:  # BatchRunInfo (batch.hpp:138-141) as measured by the engine
        dev = (batch.data.device.index or 0) if _is_cuda(batch.data) else 0
        tp, p_tp = _arr64(np.zeros(max(B, 1), dtype=np.uint64))
        rounds = C.c_uint64()
        _raise(lib.rtk_get_batch_info(_handle(dev), p_tp, B, C.byref(rounds)), "rtk_get_batch_info")
        info.task_passes = [int(v) for v in tp[:B]]
        info.phase_b_rounds = int(rounds.value)
    return out


def batch_topk_dense(x, k: int, order: SelectionOrder = SelectionOrder.Largest,
                     cfg: Optional[EngineConfig] = None) -> TopKResult:
    """Dense fast path of batch_topk for a [B, V] CUDA tensor (e.g. LLM logits): every row
    gets the same k; returns values [B, k], indices [B, k] (row-local) and pivots [B]."""
    import torch
    cfg = cfg or EngineConfig()
    lib = L.load()
    x = x.contiguous()
    B, V = x.shape
    offs, p_off = _arr64(np.arange(B, dtype=np.uint64) * V)
    lens, p_len = _arr64(np.full(B, V, dtype=np.uint64))
    kks, p_ks = _arr64(np.full(B, k, dtype=np.uint64))
    oo, p_oo = _arr64(np.arange(B, dtype=np.uint64) * k)
    vals = torch.empty((B, k), dtype=x.dtype, device=x.device)
    idx = torch.empty((B, k), dtype=torch.int64, device=x.device)
    piv = torch.empty(B, dtype=x.dtype, device=x.device)
    c = cfg._c()
    o = L.rtk_batch_opts(1, 1)
    st = lib.rtk_topk_batched(_handle(x.device.index or 0), C.c_void_p(x.data_ptr()), x.numel(), p_off, p_len,
                              p_ks, B, _dtype_code(x), int(order), C.c_void_p(vals.data_ptr()),
                              C.c_void_p(idx.data_ptr()), p_oo, C.c_void_p(piv.data_ptr()), C.byref(c),
                              C.byref(o), _stream_ptr(x))
    _raise(st, "rtk_topk_batched")
    return TopKResult(vals, idx, piv)


def scaled_topk(input, k: int, order: SelectionOrder = SelectionOrder.Largest,
                cfg: Optional[EngineConfig] = None, policy: Optional[ScalePolicy] = None,
                info: Optional[ScaleInfo] = None) -> TopKResult:
    """rtk::scaled_topk (scaling.hpp:42-86): selection on y = x - a_s, values re-read from x."""
    cfg = cfg or EngineConfig()
    policy = policy or ScalePolicy()
    lib = L.load()
    c = cfg._c()
    si = L.rtk_scale_info()
    if _is_cuda(input):
        import torch
        x = input.contiguous()
        if x.dtype != torch.float32:
            raise TypeError("scaled_topk is defined for float32 only")
        n = x.numel()
        kk = max(int(k), 0)
        vals = torch.empty(kk, dtype=x.dtype, device=x.device)
        idx = torch.empty(kk, dtype=torch.int64, device=x.device)
        piv = torch.empty(1, dtype=x.dtype, device=x.device)
        st = lib.rtk_topk_scaled(_handle(x.device.index or 0), C.c_void_p(x.data_ptr() if n else 0), n,
                                 int(k), int(order), int(policy.mode), float(policy.trigger_fraction),
                                 int(policy.seed) & 0xFFFFFFFFFFFFFFFF, C.c_void_p(vals.data_ptr()),
                                 C.c_void_p(idx.data_ptr()), C.c_void_p(piv.data_ptr()),
                                 C.byref(si), C.byref(c), _stream_ptr(x))
        _raise(st, "rtk_topk_scaled")
        res = TopKResult(vals, idx, pivot_fn=lambda: piv[0].item())
    else:
        a = np.ascontiguousarray(input.numpy() if hasattr(input, "numpy") else np.asarray(input))
        if a.dtype != np.float32:
            raise TypeError("scaled_topk is defined for float32 only")
        n = a.size
        kk = max(int(k), 0)
        vals = np.empty(kk, dtype=np.float32)
        idx = np.empty(kk, dtype=np.uint64)
        piv = np.zeros(1, dtype=np.float32)
        st = lib.rtk_topk_scaled_host(_handle(0), C.c_void_p(a.ctypes.data if n else 0), n, int(k),
                                      int(order), int(policy.mode), float(policy.trigger_fraction),
                                      int(policy.seed) & 0xFFFFFFFFFFFFFFFF, C.c_void_p(vals.ctypes.data),
                                      C.c_void_p(idx.ctypes.data), C.c_void_p(piv.ctypes.data),
                                      C.byref(si), C.byref(c))
        _raise(st, "rtk_topk_scaled_host")
        res = TopKResult(vals, idx, piv[0])
    if info is not None:
        info.scaled = bool(si.scaled)
        info.a_s = float(si.a_s)
        info.a_index = int(si.a_index)
    return res


def generate_philox(n: int, seed: int, offset: int = 0, a: float = 0.0, b: float = 1.0, device=None):
    """rtk_generate_philox: elements [offset, offset + n) of the Philox uniform f32 stream written
    straight into a new CUDA tensor (the per-shard generator of the n = 2^32 configuration)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    out = torch.empty(int(n), dtype=torch.float32, device=dev)
    _raise(L.load().rtk_generate_philox(C.c_void_p(out.data_ptr()), int(n), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                        int(offset), float(a), float(b), _stream_ptr(out)), "rtk_generate_philox")
    return out


def generate_philox_host(n: int, seed: int, offset: int = 0, a: float = 0.0, b: float = 1.0) -> np.ndarray:
    """rtk_generate_philox_host: the bit-identical host twin of generate_philox."""
    out = np.empty(int(n), dtype=np.float32)
    _raise(L.load().rtk_generate_philox_host(C.c_void_p(out.ctypes.data), int(n), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                             int(offset), float(a), float(b)), "rtk_generate_philox_host")
    return out


def merge_shards(cand_vals, cand_idx, block_len: Sequence[int], shard_base: Sequence[int], k: int,
                 order: SelectionOrder = SelectionOrder.Largest) -> TopKResult:
    """Final select of an n-sharded query: G canonical per-shard results (concatenated in
    shard order, shard-local indices) -> the global top-k with global indices."""
    import torch
    lib = L.load()
    code = _dtype_code(cand_vals)
    bl, p_bl = _arr64(block_len)
    sb, p_sb = _arr64(shard_base)
    vals = torch.empty(int(k), dtype=cand_vals.dtype, device=cand_vals.device)
    idx = torch.empty(int(k), dtype=torch.int64, device=cand_vals.device)
    piv = torch.empty(1, dtype=cand_vals.dtype, device=cand_vals.device)
    cv = cand_vals.contiguous()
    ci = cand_idx.contiguous()
    st = lib.rtk_merge_shards(_handle(cv.device.index or 0), C.c_void_p(cv.data_ptr()),
                              C.c_void_p(ci.data_ptr()), p_bl, p_sb, len(bl), int(k), code, int(order),
                              C.c_void_p(vals.data_ptr()), C.c_void_p(idx.data_ptr()),
                              C.c_void_p(piv.data_ptr()), _stream_ptr(cv))
    _raise(st, "rtk_merge_shards")
    return TopKResult(vals, idx, pivot_fn=lambda: piv[0].item())


# ---- LLM sampling consumer --------------------------------------------------
def topk_sample(logits, k: int, top_p: float = 1.0, temperature: float = 1.0, uniform=None, generator=None,
                return_probs: bool = False):
    """Top-k -> softmax -> top-p -> one draw per row, on the device (rtk_topk_sample, rtk_c.h).

    ``logits``: CUDA tensor [B, V] (float32 / float16 / bfloat16, unit stride along V). ``uniform``:
    [B] float32 CUDA tensor of draws in [0, 1) (``torch.rand`` with ``generator`` if None).
    Returns the sampled row-local token ids (int64 [B]); with ``return_probs`` also the renormalised
    top-k/top-p probabilities [B, k] (0 past the nucleus) and the top-k indices [B, k], whose
    order is the reference's canonical top-k order.
    """
    import torch
    if not _is_cuda(logits) or logits.dim() != 2 or logits.stride(1) != 1:
        raise ValueError("topk_sample: logits must be a 2-D CUDA tensor with unit stride along V")
    B, V = logits.shape
    dev = logits.device
    if uniform is None:
        uniform = torch.rand(B, device=dev, generator=generator, dtype=torch.float32)
    uniform = uniform.to(device=dev, dtype=torch.float32).contiguous()
    token = torch.empty(B, dtype=torch.int64, device=dev)
    probs = torch.empty((B, k), dtype=torch.float32, device=dev) if return_probs else None
    tv = torch.empty((B, k), dtype=logits.dtype, device=dev) if return_probs else None
    ti = torch.empty((B, k), dtype=torch.int64, device=dev) if return_probs else None
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    st = L.load().rtk_topk_sample(_handle(dev.index or 0), ptr(logits), B, V, logits.stride(0),
                                  _dtype_code(logits), int(k), float(top_p), float(temperature), ptr(uniform),
                                  ptr(token), ptr(probs), ptr(tv), ptr(ti), _stream_ptr(logits))
    _raise(st, "rtk_topk_sample")
    return (token, probs, ti) if return_probs else token

"""RTK1 / RTKB dataset containers — mirror of rtk/io.hpp.

``write_dataset`` / ``read_dataset`` <- rtk::write_dataset / read_dataset (io.cpp:38-80): magic
"RTK1", u8 dtype code (0 f32, 1 u32, 2 f16; 3 bf16 is this build's extension), u64 count, raw
little-endian payload. ``write_batch`` / ``read_batch`` <- io.cpp:82-110: magic "RTKB", u32 task
count, u64 lengths, concatenated payloads (offsets derived from the lengths, misalignment kept).
Errors are ``RuntimeError`` with the reference's messages (std::runtime_error there). The byte
work is done by librtk_b200.so (rtk_host.cpp); these are host utilities, not the GPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _lib as L
from .rtk import _raise


class DType(enum.IntEnum):  # io.hpp:19 (+ BF16, this build)
    F32 = 0
    U32 = 1
    F16 = 2
    BF16 = 3


_NP = {DType.F32: np.float32, DType.U32: np.uint32, DType.F16: np.float16, DType.BF16: np.uint16}


def _code(a: np.ndarray, dtype) -> DType:
    if dtype is not None:
        return DType(dtype)
    return {np.dtype(np.float32): DType.F32, np.dtype(np.uint32): DType.U32,
            np.dtype(np.float16): DType.F16}[a.dtype]


@dataclass
class Dataset:
    dtype: DType
    values: np.ndarray  # bf16 payloads are returned as their uint16 bit patterns

    def size(self) -> int:
        return int(self.values.size)


@dataclass
class BatchFile:
    lengths: List[int] = field(default_factory=list)
    payload: bytes = b""

    def derived_offsets(self) -> List[int]:  # io.hpp:33-41
        out, at = [], 0
        for n in self.lengths:
            out.append(at)
            at += n
        return out


def write_dataset(path: str, values, dtype=None) -> None:
    a = np.ascontiguousarray(values)
    code = _code(a, dtype)
    _raise(L.load().rtk_write_dataset(str(path).encode(), int(code), a.ctypes.data_as(C.c_void_p), a.size),
           "write_dataset")


def read_dataset(path: str) -> Dataset:
    lib = L.load()
    code, n = C.c_int(0), C.c_uint64(0)
    _raise(lib.rtk_read_dataset(str(path).encode(), C.byref(code), C.byref(n), None, 0), "read_dataset")
    out = np.empty(n.value, dtype=_NP[DType(code.value)])
    _raise(lib.rtk_read_dataset(str(path).encode(), C.byref(code), C.byref(n), out.ctypes.data_as(C.c_void_p),
                                out.size), "read_dataset")
    return Dataset(DType(code.value), out)


def write_batch(path: str, lengths, payload) -> None:
    ln = np.ascontiguousarray(np.asarray(lengths, dtype=np.uint64))
    pb = np.frombuffer(bytes(payload), dtype=np.uint8) if not isinstance(payload, np.ndarray) \
        else np.ascontiguousarray(payload).view(np.uint8).reshape(-1)
    _raise(L.load().rtk_write_batch(str(path).encode(), ln.ctypes.data_as(L.P64), len(ln),
                                    pb.ctypes.data_as(C.c_void_p), pb.size), "write_batch")


def read_batch(path: str) -> BatchFile:
    lib = L.load()
    t, nb = C.c_uint32(0), C.c_uint64(0)
    _raise(lib.rtk_read_batch(str(path).encode(), C.byref(t), C.byref(nb), None, None), "read_batch")
    ln = np.empty(t.value, dtype=np.uint64)
    pb = np.empty(nb.value, dtype=np.uint8)
    _raise(lib.rtk_read_batch(str(path).encode(), C.byref(t), C.byref(nb), ln.ctypes.data_as(L.P64),
                              pb.ctypes.data_as(C.c_void_p)), "read_batch")
    return BatchFile([int(v) for v in ln], pb.tobytes())


def find_nan(values) -> int:
    """Index of the first NaN, or -1 (io.hpp:56)."""
    a = np.asarray(values)
    hit = np.flatnonzero(np.isnan(a))
    return int(hit[0]) if hit.size else -1

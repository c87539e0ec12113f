"""Parity oracle (TEST INFRASTRUCTURE — never imported by the product package).

Two CPU checkers, both loaded through ctypes:

* ``port``: oracle/liboracle.so, the plain-C restatement of the reference algorithm
  (oracle/rtk_oracle.c, each function citing the reference file:line it follows).
* ``ref``:  oracle/_ref/librtk_ref.so, the reference's own headers
  (/root/reference/proj/include/rtk/*.hpp) compiled in place through oracle/ref_shim.cpp.
  Built here by oracle/Makefile; travels prebuilt to the GPU box (the reference tree does not).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
use this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "librtk_ref.so")

u64, u32, vp = C.c_uint64, C.c_uint32, C.c_void_p
P64 = C.POINTER(C.c_uint64)

STATUS = {0: "ok", 1: "empty_input_error", 2: "rank_out_of_range", 3: "invariant_violation",
          4: "invalid_argument", 6: "nomem", 7: "other"}


class OracleError(Exception):
    def __init__(self, code: int):
        super().__init__(STATUS.get(code, str(code)))
        self.code = code
        self.kind = STATUS.get(code, str(code))


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    return C.CDLL(path)


_port = None
_ref = None


def port() -> C.CDLL:
    global _port
    if _port is None:
        lib = _load(PORT_PATH)
        lib.rtko_topk.argtypes = [vp, u64, u64, C.c_int, C.c_int, C.c_uint, vp, vp, vp, vp]
        lib.rtko_oracle_topk.argtypes = [vp, u64, u64, C.c_int, C.c_int, vp, vp, vp]
        lib.rtko_scaled_topk.argtypes = [vp, u64, u64, C.c_int, C.c_uint, C.c_int, C.c_double, u64,
                                         vp, vp, vp, vp]
        lib.rtko_batch_topk.argtypes = [vp, u64, P64, P64, P64, u64, C.c_int, C.c_int, C.c_uint, vp,
                                        vp, P64, vp, vp]
        lib.rtko_count_bins.argtypes = [vp, u64, C.c_uint, C.c_uint, vp]
        lib.rtko_count_bins.restype = None
        lib.rtko_select_bin.argtypes = [vp, u64, u64, vp, vp]
        lib.rtko_encode_f32_bits.argtypes = [u32, C.c_int]
        lib.rtko_encode_f32_bits.restype = u32
        lib.rtko_decode_f32_bits.argtypes = [u32, C.c_int]
        lib.rtko_decode_f32_bits.restype = u32
        lib.rtko_extract_digit.argtypes = [u32, C.c_uint, C.c_uint]
        lib.rtko_extract_digit.restype = u32
        lib.rtko_mt19937_64_first.argtypes = [u64]
        lib.rtko_mt19937_64_first.restype = u64
        lib.rtkv_philox_elem.argtypes = [u64, u64, C.c_float, C.c_float]
        lib.rtkv_philox_elem.restype = u32
        lib.rtkv_philox_fill.argtypes = [u64, u64, u64, C.c_float, C.c_float, vp]
        lib.rtkv_philox_fill.restype = None
        lib.rtkv_verify_philox_topk.argtypes = [u64, u64, C.c_float, C.c_float, C.c_int, u64, vp, vp, C.c_int,
                                                vp, C.c_char_p, C.c_int]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_PATH) or os.path.isdir("/root/reference/proj/include/rtk")


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = _load(REF_PATH)
        lib.ref_topk.argtypes = [vp, u64, u64, C.c_int, C.c_int, C.c_uint, C.c_uint, vp, vp, vp, vp]
        lib.ref_oracle_topk.argtypes = [vp, u64, u64, C.c_int, C.c_int, vp, vp, vp]
        lib.ref_batch_topk.argtypes = [vp, u64, P64, P64, P64, u64, C.c_int, C.c_int, C.c_uint,
                                       C.c_uint, C.c_int, C.c_int, vp, vp, P64, vp]
        lib.ref_scaled_topk.argtypes = [vp, u64, u64, C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_double,
                                        u64, vp, vp, vp, vp]
        lib.ref_generate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint,
                                     u64, u64, C.c_int, vp]
        lib.ref_count_bins.argtypes = [vp, u64, C.c_uint, C.c_uint, C.c_uint, vp]
        lib.ref_select_bin.argtypes = [vp, u64, u64, vp, vp]
        lib.ref_encode_f32.argtypes = [C.c_float, C.c_int]
        lib.ref_encode_f32.restype = u32
        lib.ref_io_error.restype = C.c_char_p
        lib.ref_write_dataset.argtypes = [C.c_char_p, C.c_int, vp, u64]
        lib.ref_read_dataset.argtypes = [C.c_char_p, C.POINTER(C.c_int), P64, vp]
        lib.ref_write_batch.argtypes = [C.c_char_p, P64, u32, vp, u64]
        lib.ref_read_batch.argtypes = [C.c_char_p, C.POINTER(u32), P64, P64, vp]
        _ref = lib
    return _ref


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.uint32:
        return 1
    raise TypeError(a.dtype)


def _ck(code: int) -> None:
    if code:
        raise OracleError(code)


Result = Tuple[np.ndarray, np.ndarray, object]


# ---- C restatement ("port") --------------------------------------------------------------
def port_topk(x: np.ndarray, k: int, order: int = 0, d: int = 12) -> Result:
    x = np.ascontiguousarray(x)
    kk = max(int(k), 1)
    vals = np.empty(kk, dtype=x.dtype)
    idx = np.empty(kk, dtype=np.uint64)
    piv = np.zeros(1, dtype=np.uint32)
    _ck(port().rtko_topk(x.ctypes.data if x.size else None, x.size, int(k), _dt(x), order, d,
                         vals.ctypes.data, idx.ctypes.data, piv.ctypes.data, None))
    return vals[:k], idx[:k], piv.view(x.dtype)[0]


def port_oracle_topk(x: np.ndarray, k: int, order: int = 0) -> Result:
    x = np.ascontiguousarray(x)
    kk = max(int(k), 1)
    vals = np.empty(kk, dtype=x.dtype)
    idx = np.empty(kk, dtype=np.uint64)
    piv = np.zeros(1, dtype=np.uint32)
    _ck(port().rtko_oracle_topk(x.ctypes.data if x.size else None, x.size, int(k), _dt(x), order,
                                vals.ctypes.data, idx.ctypes.data, piv.ctypes.data))
    return vals[:k], idx[:k], piv.view(x.dtype)[0]


def port_scaled_topk(x: np.ndarray, k: int, order: int = 0, d: int = 12, mode: int = 0,
                     tau: float = 0.5, seed: int = 0) -> Tuple[np.ndarray, np.ndarray, object, dict]:
    x = np.ascontiguousarray(x, dtype=np.float32)
    kk = max(int(k), 1)
    vals = np.empty(kk, dtype=np.float32)
    idx = np.empty(kk, dtype=np.uint64)
    piv = np.zeros(1, dtype=np.uint32)
    info = np.zeros(3, dtype=np.uint64)
    _ck(port().rtko_scaled_topk(x.ctypes.data if x.size else None, x.size, int(k), order, d, mode,
                                tau, seed, vals.ctypes.data, idx.ctypes.data, piv.ctypes.data,
                                info.ctypes.data))
    a_s = np.array([info[1]], dtype=np.uint64).astype(np.uint32).view(np.float32)[0]
    return vals[:k], idx[:k], piv.view(np.float32)[0], {"scaled": bool(info[0]), "a_s": a_s,
                                                          "a_index": int(info[2])}


def port_batch_topk(data: np.ndarray, offsets, lengths, ks, order: int = 0, d: int = 12):
    data = np.ascontiguousarray(data)
    B = len(lengths)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    ln = np.ascontiguousarray(lengths, dtype=np.uint64)
    kk = np.ascontiguousarray(ks, dtype=np.uint64)
    oo = np.zeros(B, dtype=np.uint64)
    if B:
        oo[1:] = np.cumsum(kk[:-1])
    tot = int(kk.sum()) if B else 0
    vals = np.empty(max(tot, 1), dtype=data.dtype)
    idx = np.empty(max(tot, 1), dtype=np.uint64)
    piv = np.empty(max(B, 1), dtype=np.uint32)
    bad = np.zeros(1, dtype=np.uint64)
    _ck(port().rtko_batch_topk(data.ctypes.data, data.size, off.ctypes.data_as(P64),
                               ln.ctypes.data_as(P64), kk.ctypes.data_as(P64), B, _dt(data), order, d,
                               vals.ctypes.data, idx.ctypes.data, oo.ctypes.data_as(P64),
                               piv.ctypes.data, bad.ctypes.data))
    return [(vals[int(oo[t]):int(oo[t]) + int(kk[t])], idx[int(oo[t]):int(oo[t]) + int(kk[t])],
             piv.view(data.dtype)[t]) for t in range(B)]


def encode(x: np.ndarray, order: int = 0) -> np.ndarray:
    """Vectorised KeyCodec encode (keycodec.hpp:55-81) for fixture checks."""
    x = np.asarray(x)
    raw = x.view(np.uint32) if x.dtype == np.float32 else x.astype(np.uint32)
    if x.dtype == np.float32:
        bits = np.where(raw & np.uint32(0x80000000), ~raw, raw | np.uint32(0x80000000)).astype(np.uint32)
    else:
        bits = raw.copy()
    return (~bits).astype(np.uint32) if order == 1 else bits


# ---- the reference itself ("ref") --------------------------------------------------------
def ref_generate(kind: int, n: int, seed: int, dtype=np.float32, a: float = 0.0, b: float = 1.0,
                 s: float = 1.1, mass: float = 0.8, modes: int = 1) -> np.ndarray:
    out = np.empty(n, dtype=dtype)
    _ck(ref().ref_generate(kind, a, b, s, mass, modes, seed, n, _dt(out), out.ctypes.data))
    return out


def _io_ck(code: int) -> None:
    if code:
        raise RuntimeError(ref().ref_io_error().decode())


def ref_write_dataset(path: str, x: np.ndarray) -> None:  # rtk::write_dataset (io.cpp:38-44)
    x = np.ascontiguousarray(x)
    _io_ck(ref().ref_write_dataset(str(path).encode(), _dt(x), x.ctypes.data, x.size))


def ref_read_dataset(path: str):  # rtk::read_dataset (io.cpp:46-80) -> (dtype code, array)
    dt, n = C.c_int(0), C.c_uint64(0)
    _io_ck(ref().ref_read_dataset(str(path).encode(), C.byref(dt), C.byref(n), None))
    out = np.empty(n.value, dtype=np.float32 if dt.value == 0 else np.uint32)
    _io_ck(ref().ref_read_dataset(str(path).encode(), C.byref(dt), C.byref(n), out.ctypes.data))
    return dt.value, out


def ref_write_batch(path: str, lengths, payload: bytes) -> None:  # io.cpp:82-92
    ln = np.ascontiguousarray(np.asarray(lengths, dtype=np.uint64))
    pb = np.frombuffer(payload, dtype=np.uint8)
    _io_ck(ref().ref_write_batch(str(path).encode(), ln.ctypes.data_as(P64), len(ln), pb.ctypes.data, pb.size))


def ref_read_batch(path: str):  # io.cpp:94-110 -> (lengths, payload bytes)
    t, nb = C.c_uint32(0), C.c_uint64(0)
    _io_ck(ref().ref_read_batch(str(path).encode(), C.byref(t), C.byref(nb), None, None))
    ln = np.empty(t.value, dtype=np.uint64)
    pb = np.empty(nb.value, dtype=np.uint8)
    _io_ck(ref().ref_read_batch(str(path).encode(), C.byref(t), C.byref(nb), ln.ctypes.data_as(P64), pb.ctypes.data))
    return [int(v) for v in ln], pb.tobytes()


def ref_topk(x: np.ndarray, k: int, order: int = 0, d: int = 12, grid: int = 1) -> Result:
    x = np.ascontiguousarray(x)
    kk = max(int(k), 1)
    vals = np.empty(kk, dtype=x.dtype)
    idx = np.empty(kk, dtype=np.uint64)
    piv = np.zeros(1, dtype=np.uint32)
    _ck(ref().ref_topk(x.ctypes.data if x.size else None, x.size, int(k), _dt(x), order, d, grid,
                       vals.ctypes.data, idx.ctypes.data, piv.ctypes.data, None))
    return vals[:k], idx[:k], piv.view(x.dtype)[0]


def ref_oracle_topk(x: np.ndarray, k: int, order: int = 0) -> Result:
    x = np.ascontiguousarray(x)
    kk = max(int(k), 1)
    vals = np.empty(kk, dtype=x.dtype)
    idx = np.empty(kk, dtype=np.uint64)
    piv = np.zeros(1, dtype=np.uint32)
    _ck(ref().ref_oracle_topk(x.ctypes.data if x.size else None, x.size, int(k), _dt(x), order,
                              vals.ctypes.data, idx.ctypes.data, piv.ctypes.data))
    return vals[:k], idx[:k], piv.view(x.dtype)[0]


def ref_scaled_topk(x: np.ndarray, k: int, order: int = 0, d: int = 12, mode: int = 0,
                    tau: float = 0.5, seed: int = 0, grid: int = 1):
    x = np.ascontiguousarray(x, dtype=np.float32)
    kk = max(int(k), 1)
    vals = np.empty(kk, dtype=np.float32)
    idx = np.empty(kk, dtype=np.uint64)
    piv = np.zeros(1, dtype=np.float32)
    info = np.zeros(3, dtype=np.uint64)
    _ck(ref().ref_scaled_topk(x.ctypes.data, x.size, int(k), order, d, grid, mode, tau, seed,
                              vals.ctypes.data, idx.ctypes.data, piv.ctypes.data, info.ctypes.data))
    a_s = np.array([info[1]], dtype=np.uint64).astype(np.uint32).view(np.float32)[0]
    return vals[:k], idx[:k], piv[0], {"scaled": bool(info[0]), "a_s": a_s, "a_index": int(info[2])}


def ref_batch_topk(data: np.ndarray, offsets, lengths, ks, order: int = 0, d: int = 12,
                   grid: int = 1, rescheduling: bool = True, padding: bool = True):
    data = np.ascontiguousarray(data)
    B = len(lengths)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    ln = np.ascontiguousarray(lengths, dtype=np.uint64)
    kk = np.ascontiguousarray(ks, dtype=np.uint64)
    oo = np.zeros(B, dtype=np.uint64)
    if B:
        oo[1:] = np.cumsum(kk[:-1])
    tot = int(kk.sum()) if B else 0
    vals = np.empty(max(tot, 1), dtype=data.dtype)
    idx = np.empty(max(tot, 1), dtype=np.uint64)
    piv = np.empty(max(B, 1), dtype=data.dtype)
    _ck(ref().ref_batch_topk(data.ctypes.data, data.size, off.ctypes.data_as(P64),
                             ln.ctypes.data_as(P64), kk.ctypes.data_as(P64), B, _dt(data), order, d,
                             grid, int(rescheduling), int(padding), vals.ctypes.data, idx.ctypes.data,
                             oo.ctypes.data_as(P64), piv.ctypes.data))
    return [(vals[int(oo[t]):int(oo[t]) + int(kk[t])], idx[int(oo[t]):int(oo[t]) + int(kk[t])], piv[t])
            for t in range(B)]


# ---- Philox stream (rtk_verify.c: an independent restatement of rtk_generate_philox) ---------
def philox_fill(seed: int, offset: int, n: int, a: float = 0.0, b: float = 1.0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    port().rtkv_philox_fill(seed, offset, n, a, b, out.ctypes.data)
    return out.view(np.float32)


def verify_philox_topk(seed: int, n: int, k: int, values, indices, order: int = 0, a: float = 0.0,
                       b: float = 1.0, threads: int = 0):
    """Streaming O(k)-memory check of a top-k of the Philox query (rtk_verify.c). Returns
    (ok, message, [#{key > P}, #{key == P}, #{key == P, index <= last returned index}])."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float32).view(np.uint32))
    i = np.ascontiguousarray(np.asarray(indices).astype(np.uint64))
    stats = np.zeros(3, dtype=np.uint64)
    msg = C.create_string_buffer(256)
    rc = port().rtkv_verify_philox_topk(seed, n, a, b, order, k, v.ctypes.data, i.ctypes.data,
                                        threads or (os.cpu_count() or 1), stats.ctypes.data, msg, 256)
    return rc == 0, msg.value.decode(), [int(x) for x in stats]

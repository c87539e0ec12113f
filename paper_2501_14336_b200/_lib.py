"""ctypes binding of the in-tree C-ABI library ``librtk_b200.so`` (include/rtk_c.h).

The product path has no fallback: if the CUDA library is missing or cannot be loaded, every
call raises. Build it with ``python -c "import __graft_entry__ as g; g.build()"`` or
``make -C paper_2501_14336_b200``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librtk_b200.so")

u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int32
vp = C.c_void_p
P64 = C.POINTER(C.c_uint64)

# status codes (rtk_c.h)
RTK_OK = 0
RTK_EMPTY_INPUT = 1
RTK_RANK_OUT_OF_RANGE = 2
RTK_INVARIANT_VIOLATION = 3
RTK_INVALID_ARGUMENT = 4
RTK_CUDA_ERROR = 5
RTK_OUT_OF_MEMORY = 6
RTK_INTERNAL = 7
RTK_IO_ERROR = 8


class rtk_cfg(C.Structure):
    _fields_ = [("d", u32), ("block_size", u64), ("grid_size", u32), ("buffer_policy", i32),
                ("pack_size", u64), ("hierarchical_atomics", i32), ("filter_fixed_ceiling", u64)]


class rtk_batch_opts(C.Structure):
    _fields_ = [("rescheduling", i32), ("padding", i32)]


class rtk_scale_info(C.Structure):
    _fields_ = [("scaled", i32), ("a_s", C.c_float), ("a_index", u64)]


class rtk_stats(C.Structure):
    _fields_ = [("passes", u64), ("elements_scanned", u64), ("candidates", u64),
                ("fallback_rows", u64), ("kernel_launches", u64), ("compact_ms", C.c_float),
                ("total_ms", C.c_float), ("deep_levels", u64)]


class rtk_dist(C.Structure):
    _fields_ = [("kind", i32), ("a", C.c_double), ("b", C.c_double), ("s", C.c_double),
                ("mass", C.c_double), ("modes", u32), ("seed", u64), ("n", u64)]


# name -> (restype, argtypes); exactly the entry points include/rtk_c.h declares
SIGNATURES = {
    "rtk_version": (C.c_char_p, []),
    "rtk_last_error": (C.c_char_p, []),
    "rtk_handle_create": (C.c_int, [C.POINTER(vp), C.c_int]),
    "rtk_handle_destroy": (C.c_int, [vp]),
    "rtk_get_stats": (C.c_int, [vp, C.POINTER(rtk_stats)]),
    "rtk_set_timing": (C.c_int, [vp, C.c_int]),
    "rtk_set_option": (C.c_int, [vp, C.c_char_p, C.c_int64]),
    "rtk_nccl_get_unique_id": (C.c_int, [vp]),
    "rtk_nccl_comm_init_rank": (C.c_int, [C.POINTER(vp), C.c_int, vp, C.c_int, C.c_int]),
    "rtk_nccl_comm_destroy": (C.c_int, [vp]),
    "rtk_topk_sharded": (C.c_int, [C.POINTER(vp), C.POINTER(vp), C.c_int, C.POINTER(vp), P64, C.c_int, u64,
                                   C.c_int, C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    "rtk_get_batch_info": (C.c_int, [vp, P64, u64, P64]),
    "rtk_bench_batched": (C.c_int, [vp, vp, u64, P64, P64, P64, u64, C.c_int, C.c_int, vp, vp, P64, vp,
                                    C.POINTER(rtk_cfg), vp, vp, u64, C.c_int, C.c_int,
                                    C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "rtk_bench_topk": (C.c_int, [vp, vp, u64, u64, C.c_int, C.c_int, vp, vp, vp, C.POINTER(rtk_cfg), vp, vp, u64,
                                 C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                 C.POINTER(C.c_float)]),
    "rtk_bench_scaled": (C.c_int, [vp, vp, u64, u64, C.c_int, C.c_int, C.c_double, u64, vp, vp, vp,
                                   C.POINTER(rtk_cfg), vp, vp, u64, C.c_int, C.c_int, C.POINTER(C.c_float),
                                   C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "rtk_cfg_default": (None, [C.POINTER(rtk_cfg)]),
    "rtk_cfg_validate": (C.c_int, [C.POINTER(rtk_cfg)]),
    "rtk_topk": (C.c_int, [vp, vp, u64, u64, C.c_int, C.c_int, vp, vp, vp, C.POINTER(rtk_cfg), vp]),
    "rtk_topk_batched": (C.c_int, [vp, vp, u64, P64, P64, P64, u64, C.c_int, C.c_int, vp, vp, P64,
                                   vp, C.POINTER(rtk_cfg), C.POINTER(rtk_batch_opts), vp]),
    "rtk_topk_scaled": (C.c_int, [vp, vp, u64, u64, C.c_int, C.c_int, C.c_double, u64, vp, vp, vp,
                                  C.POINTER(rtk_scale_info), C.POINTER(rtk_cfg), vp]),
    "rtk_topk_host": (C.c_int, [vp, vp, u64, u64, C.c_int, C.c_int, vp, vp, vp, C.POINTER(rtk_cfg)]),
    "rtk_topk_batched_host": (C.c_int, [vp, vp, u64, P64, P64, P64, u64, C.c_int, C.c_int, vp, vp,
                                        P64, vp, C.POINTER(rtk_cfg), C.POINTER(rtk_batch_opts)]),
    "rtk_topk_scaled_host": (C.c_int, [vp, vp, u64, u64, C.c_int, C.c_int, C.c_double, u64, vp, vp,
                                       vp, C.POINTER(rtk_scale_info), C.POINTER(rtk_cfg)]),
    "rtk_merge_shards": (C.c_int, [vp, vp, vp, P64, P64, u32, u64, C.c_int, C.c_int, vp, vp, vp, vp]),
    "rtk_topk_sample": (C.c_int, [vp, vp, u64, u64, u64, C.c_int, u64, C.c_float, C.c_float, vp, vp, vp, vp,
                                  vp, vp]),
    "rtk_generate": (C.c_int, [C.POINTER(rtk_dist), C.c_int, vp]),
    "rtk_generate_philox": (C.c_int, [vp, u64, u64, u64, C.c_float, C.c_float, vp]),
    "rtk_generate_philox_host": (C.c_int, [vp, u64, u64, u64, C.c_float, C.c_float]),
    "rtk_result_checksum": (u64, [vp, C.c_int, P64, u64]),
    "rtk_write_dataset": (C.c_int, [C.c_char_p, C.c_int, vp, u64]),
    "rtk_read_dataset": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), P64, vp, u64]),
    "rtk_write_batch": (C.c_int, [C.c_char_p, P64, u32, vp, u64]),
    "rtk_read_batch": (C.c_int, [C.c_char_p, C.POINTER(u32), P64, P64, vp]),
}

_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load librtk_b200.so (raises if it is absent — there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the CUDA library first "
                    "(python -c 'import __graft_entry__ as g; g.build()')")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def last_error() -> str:
    msg = load().rtk_last_error()
    return msg.decode() if msg else ""

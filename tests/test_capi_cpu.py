"""CPU: the C-ABI library loads without a GPU and exports exactly what include/rtk_c.h declares.

No compute calls here (there is no GPU in the build container); host-only entry points
(config defaults/validation, error reporting) are exercised.
"""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rtk_c.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rtk_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2501_14336_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2501_14336_b200")], check=True)
    return _lib.load()


def test_header_declares_the_reference_entry_points():
    fns = header_functions()
    for name in ["rtk_topk", "rtk_topk_batched", "rtk_topk_scaled", "rtk_topk_host", "rtk_topk_batched_host",
                 "rtk_topk_scaled_host", "rtk_merge_shards", "rtk_handle_create", "rtk_handle_destroy",
                 "rtk_cfg_default", "rtk_cfg_validate", "rtk_last_error", "rtk_get_stats", "rtk_set_timing", "rtk_bench_topk", "rtk_bench_batched", "rtk_bench_scaled", "rtk_version"]:
        assert name in fns


def test_library_exports_every_declared_symbol(lib):
    from paper_2501_14336_b200 import _lib
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rtk_[a-z_]+)$", nm, flags=re.M))
    declared = set(header_functions())
    assert declared <= exported, declared - exported
    assert declared == set(_lib.SIGNATURES), "ctypes signatures must cover the header exactly"
    for name in declared:
        assert getattr(lib, name) is not None


def test_library_is_sm100a_only():
    from paper_2501_14336_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_cfg_defaults_and_validation(lib):
    from paper_2501_14336_b200 import _lib
    c = _lib.rtk_cfg()
    lib.rtk_cfg_default(C.byref(c))
    # EngineConfig defaults (engine.hpp:48-57)
    assert (c.d, c.block_size, c.grid_size, c.buffer_policy, c.pack_size, c.hierarchical_atomics,
            c.filter_fixed_ceiling) == (12, 1024, 4, 1, 16, 1, 4096)
    assert lib.rtk_cfg_validate(C.byref(c)) == _lib.RTK_OK
    # EngineConfig::validate (engine.hpp:61-67) / engine_test.cpp config validation
    for field, bad in [("d", 0), ("d", 17), ("block_size", 0), ("grid_size", 0), ("pack_size", 12)]:
        lib.rtk_cfg_default(C.byref(c))
        setattr(c, field, bad)
        assert lib.rtk_cfg_validate(C.byref(c)) == _lib.RTK_INVALID_ARGUMENT
        assert _lib.last_error()


def test_python_mirror_validation():
    import paper_2501_14336_b200 as rtk
    rtk.EngineConfig().validate()
    for kw in [dict(d=0), dict(d=17), dict(pack_size=12), dict(block_size=0), dict(grid_size=0)]:
        with pytest.raises(ValueError):
            rtk.EngineConfig(**kw).validate()
    b = rtk.BatchInput([1.0, 2.0, 3.0], [0, 2], [2, 1], [1, 2])
    with pytest.raises(ValueError, match="task 1"):
        b.validate()
    with pytest.raises(ValueError, match="overlaps"):
        rtk.BatchInput([1.0, 2.0, 3.0], [0, 1], [3, 1], [1, 1]).validate()


def test_handle_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2501_14336_b200 import _lib
    h = C.c_void_p()
    st = lib.rtk_handle_create(C.byref(h), 0)
    assert st != _lib.RTK_OK and _lib.last_error()
    import numpy as np
    import paper_2501_14336_b200 as rtk
    with pytest.raises(Exception):
        rtk.topk(np.ones(16, dtype=np.float32), 4)  # no silent CPU fallback


def test_cpp_header_compiles_against_the_library(tmp_path):
    # the drop-in C++ front end (include/rtk/topk.hpp) and the retargeted acceptance program
    # compile and link against librtk_b200.so (run on the GPU in tests/test_gpu_sharded.py)
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("no g++")
    ref = os.path.join(ROOT, "oracle", "_ref")
    out = tmp_path / "acc"
    p = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "acceptance_b200.cpp"), "-o", str(out),
                        "-L", os.path.join(ROOT, "paper_2501_14336_b200"), "-lrtk_b200", "-L", ref, "-lrtk_ref"],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]


def test_bench_reference_arm_contract():
    # bench.py --impl reference: one JSON line with the contract's keys (tiny workload on CPU)
    import json
    import sys
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--logn", "16",
                        "--k", "256", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["n"] == 1 << 16

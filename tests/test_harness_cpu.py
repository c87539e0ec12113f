"""Harness rows of SURVEY §8f (host only, no GPU): the reference's generators, the `rtk bench`
checksum and the RTK1/RTKB containers, each checked against the reference compiled in place
(oracle/_ref: datagen.hpp, rtk_cli.cpp's FNV-1a restated below, io.cpp)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2501_14336_b200 import io as rio
from paper_2501_14336_b200 import report

ref = pytest.mark.skipif(not O.ref_available(), reason="reference build (oracle/_ref) absent")


@ref
@pytest.mark.parametrize("kind,dtype,extra", [
    ("uniform", np.float32, {}), ("uniform", np.float32, {"a": 128.6, "b": 128.7}),
    ("normal", np.float32, {"b": 2.5}), ("zipf", np.float32, {"s": 1.3}), ("peaked", np.float32, {"modes": 2}),
    ("uniform", np.uint32, {}), ("normal", np.uint32, {}), ("zipf", np.uint32, {}),
])
def test_generate_matches_reference(kind, dtype, extra):
    # datagen.hpp:68-140: same mt19937_64 stream and libstdc++ distributions -> identical bits
    for n, seed in [(1, 3), (1000, 7), (100003, 600)]:
        if kind == "peaked" and n <= extra.get("modes", 1):
            continue
        spec = report.DistributionSpec(kind=kind, seed=seed, n=n, **extra)
        got = report.generate(spec, dtype)
        want = O.ref_generate(report.KINDS[kind], n, seed, dtype, a=spec.a, b=spec.b, s=spec.s,
                              mass=spec.mass, modes=spec.modes)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (kind, n)


def test_generate_validation_messages():
    # DistributionSpec::validate (datagen.hpp:27-48)
    with pytest.raises(ValueError, match="n must be positive"):
        report.generate(report.DistributionSpec(n=0))
    with pytest.raises(ValueError, match="uniform: requires a < b"):
        report.generate(report.DistributionSpec(a=1.0, b=1.0, n=4))
    with pytest.raises(ValueError, match="normal: requires sigma > 0"):
        report.generate(report.DistributionSpec(kind="normal", b=0.0, n=4))
    with pytest.raises(ValueError, match="zipf: requires s > 1"):
        report.generate(report.DistributionSpec(kind="zipf", s=1.0, n=4))
    with pytest.raises(ValueError, match="peaked: modes must be in"):
        report.generate(report.DistributionSpec(kind="peaked", modes=4, n=4))
    with pytest.raises(ValueError, match="defined for f32 only"):
        report.generate(report.DistributionSpec(kind="peaked", n=4), np.uint32)


def _fnv(values: np.ndarray, indices: np.ndarray) -> int:
    # rtk_cli.cpp:100-115 restated: FNV-1a 64 over value bytes then u64 index bytes, per element
    h = 14695981039346656037
    if len(values) == 0:
        return h
    vb = values.view(np.uint8).reshape(len(values), -1)
    ib = indices.astype(np.uint64).view(np.uint8).reshape(len(indices), 8)
    for i in range(len(values)):
        for c in list(vb[i]) + list(ib[i]):
            h = ((h ^ int(c)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_result_checksum_is_fnv1a():
    rng = np.random.default_rng(5)
    for k in (0, 1, 17, 300):
        v = rng.standard_normal(k).astype(np.float32)
        i = rng.integers(0, 1 << 40, k).astype(np.uint64)
        assert report.result_checksum(v, i) == _fnv(v, i)
    h = rng.integers(0, 1 << 16, 33).astype(np.uint16).view(np.float16)
    i = np.arange(33, dtype=np.uint64)
    assert report.result_checksum(h, i) == _fnv(h, i)


@ref
def test_checksum_of_reference_result():
    # the checksum a CPU `rtk bench` cell reports for a task equals ours on the same result
    x = O.ref_generate(0, 5000, 11)
    v, i, _ = O.ref_topk(x, 64)
    assert report.result_checksum(v, i) == _fnv(v, i)


@ref
@pytest.mark.parametrize("dtype", [np.float32, np.uint32])
def test_rtk1_roundtrip_with_reference(tmp_path, dtype):
    # io_test.cpp:28-70: write/read round trip, both directions against io.cpp
    x = O.ref_generate(1, 1003, 9, dtype)
    if dtype == np.float32:
        x[[3, 700]] = [np.nan, -0.0]
    p1, p2 = str(tmp_path / "ours.rtk1"), str(tmp_path / "ref.rtk1")
    rio.write_dataset(p1, x)
    O.ref_write_dataset(p2, x)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    code, back = O.ref_read_dataset(p1)
    assert code == (0 if dtype == np.float32 else 1) and np.array_equal(back.view(np.uint32), x.view(np.uint32))
    ds = rio.read_dataset(p2)
    assert int(ds.dtype) == code and np.array_equal(ds.values.view(np.uint32), x.view(np.uint32))
    if dtype == np.float32:
        assert rio.find_nan(ds.values) == 3


def test_rtk1_16bit_and_errors(tmp_path):
    h = np.arange(-8, 8, dtype=np.float16)
    p = str(tmp_path / "h.rtk1")
    rio.write_dataset(p, h)
    ds = rio.read_dataset(p)
    assert ds.dtype == rio.DType.F16 and np.array_equal(ds.values.view(np.uint16), h.view(np.uint16))
    bf = np.arange(10, dtype=np.uint16)
    rio.write_dataset(p, bf, dtype=rio.DType.BF16)
    assert rio.read_dataset(p).dtype == rio.DType.BF16
    # io.cpp error messages (std::runtime_error)
    with pytest.raises(RuntimeError, match="cannot open"):
        rio.read_dataset(str(tmp_path / "missing.rtk1"))
    open(p, "wb").write(b"NOPE" + bytes(9))
    with pytest.raises(RuntimeError, match="bad magic, not an RTK1 dataset"):
        rio.read_dataset(p)
    open(p, "wb").write(b"RTK1" + bytes([0]) + (100).to_bytes(8, "little") + bytes(12))
    with pytest.raises(RuntimeError, match="truncated file"):
        rio.read_dataset(p)
    open(p, "wb").write(b"RTK1" + bytes([9]) + (0).to_bytes(8, "little"))
    with pytest.raises(RuntimeError, match="unknown dtype code 9"):
        rio.read_dataset(p)


@ref
def test_rtkb_roundtrip_with_reference(tmp_path):
    # io_test.cpp:100-150: misaligned task lengths survive; offsets derive from the lengths
    tasks = [O.ref_generate(0, n, 600 + t) for t, n in enumerate([5, 1, 77, 3])]
    lengths = [len(t) for t in tasks]
    payload = np.concatenate(tasks).tobytes()
    p1, p2 = str(tmp_path / "ours.rtkb"), str(tmp_path / "ref.rtkb")
    rio.write_batch(p1, lengths, payload)
    O.ref_write_batch(p2, lengths, payload)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    ln, pb = O.ref_read_batch(p1)
    assert ln == lengths and pb == payload
    b = rio.read_batch(p2)
    assert b.lengths == lengths and b.payload == payload
    assert b.derived_offsets() == [0, 5, 6, 83]
    open(p1, "wb").write(b"RTK1" + bytes(8))
    with pytest.raises(RuntimeError, match="bad magic, not an RTKB batch"):
        rio.read_batch(p1)


def test_report_csv_layout():
    rep = {"cells": [{"variant": "configured", "n": 10, "k": 2, "batch": 1, "median_ms": 0.5, "checksum": 7,
                      "verified": True, "instrumentation": {"passes": 0, "flushes": 0, "global_merges": 0,
                                                            "elements_scanned": 10, "modeled_transactions": 0}},
                     {"variant": "configured", "n": 10, "k": 20, "batch": 1, "error": "boom"}]}
    lines = report.to_csv(rep).splitlines()
    assert lines[0].startswith("variant,n,k,batch,median_ms,checksum,verified")
    assert lines[1] == "configured,10,2,1,0.5,7,1,0,0,0,10,0,"
    assert lines[2] == 'configured,10,20,1,,,,,,,,,"boom"'

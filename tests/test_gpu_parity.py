"""GPU parity: the sm_100a path (through the C-ABI) against the reference CPU engine.

Every comparison is bit-exact on values (as u32 bit patterns), indices and pivot, in the
reference's canonical order (engine.hpp:402-420). Inputs come from the reference's own seeded
generators (datagen.hpp:71-141) through oracle/_ref; expected outputs from rtk::topk /
rtk::batch_topk / rtk::scaled_topk compiled from the reference headers (oracle/_ref) — the
configurations follow the reference tests cited on each case.
"""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

UNIFORM, NORMAL, ZIPF, PEAKED = 0, 1, 2, 3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rtk():
    import paper_2501_14336_b200 as rtk
    return rtk


def _bits(v):
    v = np.asarray(v)
    return v.view(np.uint32) if v.dtype == np.float32 else v.astype(np.uint32)


def assert_same(got, want, what=""):
    gv, gi, gp = got
    wv, wi, wp = want
    gv = gv.cpu().numpy() if hasattr(gv, "cpu") else np.asarray(gv)
    gi = gi.cpu().numpy() if hasattr(gi, "cpu") else np.asarray(gi)
    assert gv.shape == wv.shape, what
    bad = np.nonzero((_bits(gv) != _bits(wv)) | (gi.astype(np.uint64) != wi.astype(np.uint64)))[0]
    assert bad.size == 0, f"{what}: first mismatch at rank {bad[:5]}: got {gv[bad[:3]]}/{gi[bad[:3]]} want {wv[bad[:3]]}/{wi[bad[:3]]}"
    gp_bits = np.array([gp], dtype=wv.dtype).view(np.uint32)[0] if wv.dtype == np.float32 else np.uint32(gp)
    assert int(gp_bits) == int(_bits(np.array([wp], dtype=wv.dtype))[0]), f"{what}: pivot"


def gpu_topk(x, k, order, cuda):
    import torch
    rtk = _rtk()
    t = torch.from_numpy(x.view(np.int32) if x.dtype == np.uint32 else x).to(cuda)
    if x.dtype == np.uint32:
        t = t.view(torch.uint32)
    r = rtk.topk(t, k, rtk.SelectionOrder(order))
    vals = r.values.view(torch.int32).cpu().numpy().view(np.uint32) if x.dtype == np.uint32 else r.values.cpu().numpy()
    return vals, r.indices.cpu().numpy(), r.pivot


@pytest.mark.parametrize("k", [256, 1, 4096, 1 << 19])
def test_c1_uniform_largest(cuda, k):
    # BASELINE C1: single query fp32 uniform n=2^20, largest (acceptance_test.cpp:48-94 sizes)
    x = O.ref_generate(UNIFORM, 1 << 20, 1)
    assert_same(gpu_topk(x, k, 0, cuda), O.ref_topk(x, k, 0, grid=4), f"C1 k={k}")


@pytest.mark.parametrize("n", [10, 1000, 3001, 1 << 16, (1 << 20) + 3])
@pytest.mark.parametrize("kind", [UNIFORM, NORMAL, ZIPF])
@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("dtype", [np.float32, np.uint32])
def test_randomized_suite(cuda, n, kind, order, dtype):
    # acceptance criterion 1 (acceptance_test.cpp:48-94): n x dist x order x k in {1,7,512,n/2,n}
    seed = 10000 + n * 7 + kind * 3 + order
    x = O.ref_generate(kind, n, seed, dtype=dtype, b=1.0)
    for k in sorted({1, 7, 512, n // 2, n}):
        if k < 1 or k > n:
            continue
        assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=4),
                    f"n={n} kind={kind} order={order} dtype={dtype.__name__} k={k}")


def test_ties_all_duplicates(cuda):
    # engine_test.cpp:188-198: duplicate-only input; ties fill by ascending index (:219-230)
    x = np.full(1000, 2.5, dtype=np.float32)
    for k in [1, 123, 999, 1000]:
        assert_same(gpu_topk(x, k, 0, cuda), O.ref_topk(x, k, 0), f"dupes k={k}")
    big = np.full((1 << 20) + 5, -7.0, dtype=np.float32)
    assert_same(gpu_topk(big, 40000, 0, cuda), O.ref_topk(big, 40000, 0, grid=4), "big dupes")


def test_two_value_input(cuda):
    # acceptance criterion 2 (acceptance_test.cpp:117-126): two values, k=40000 of 2^16
    x = np.ones(1 << 16, dtype=np.float32)
    x[::2] = 2.0
    assert_same(gpu_topk(x, 40000, 0, cuda), O.ref_topk(x, 40000, 0), "two values")


def test_special_values(cuda):
    # NaN / inf / signed zero by bit order
    x = np.array([0.0, -0.0, 1.0, float("nan"), -float("nan"), -1.0, 0.0, float("inf"), -float("inf")],
                 dtype=np.float32)
    x[4] = np.array([0xFFC00000], dtype=np.uint32).view(np.float32)[0]
    for order in [0, 1]:
        for k in range(1, 10):
            assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order), f"special order={order} k={k}")


def test_adversarial_narrow_band(cuda):
    # C4-like: U[128.6,128.7] (one first-pass bin, heavy ties), scaling_test.cpp:16-26
    x = O.ref_generate(UNIFORM, 1 << 22, 5 + (1 << 22), a=128.6, b=128.7)
    for k in [512, 1 << 16]:
        assert_same(gpu_topk(x, k, 0, cuda), O.ref_topk(x, k, 0, grid=8), f"narrow k={k}")


@pytest.mark.parametrize("shift", [0, 7, 12, 20])
def test_strided_tie_heavy_keys(cuda, shift):
    # keys that are all congruent modulo 2^shift and heavily tied (the scaled C4 shape: x - a_s
    # keeps the 2^-16 spacing of x inside much finer floats): the level-0 MSD digit squeezes the
    # common trailing zeros out of the key range (SegSlot::tz) and must keep the exact order
    rng = np.random.default_rng(shift)
    n = 1 << 22
    x = ((rng.integers(0, 4096, n, dtype=np.uint64) << np.uint64(shift)) + np.uint64(12345)).astype(np.uint32)
    for order in (0, 1):
        for k in (700, 1 << 15):
            assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=8), f"stride {shift} k={k}")


def test_scaled_c4_shape(cuda):
    # C4 at 1/16 size through scaled_topk Always: candidates are 9-ish distinct scaled keys 2^12
    # float-ulps apart with ~10K copies each
    import torch
    rtk = _rtk()
    n = 1 << 22
    x = O.ref_generate(UNIFORM, n, 31, a=128.6, b=128.7)
    for mode in (1, 2):
        wv, wi, wp, winfo = O.ref_scaled_topk(x, 1 << 12, 0, mode=mode, seed=31, grid=8)
        info = rtk.ScaleInfo()
        r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), 1 << 12, policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, 31),
                            info=info)
        assert info.scaled == winfo["scaled"]
        assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"scaled C4 shape mode={mode}")


def test_integer_ramp(cuda):
    # engine_test.cpp:292-303
    x = np.arange(1 << 20, dtype=np.uint32)
    v, i, _ = gpu_topk(x, 4, 0, cuda)
    assert list(v) == [(1 << 20) - 1, (1 << 20) - 2, (1 << 20) - 3, (1 << 20) - 4]
    v, i, _ = gpu_topk(x, 3, 1, cuda)
    assert list(v) == [0, 1, 2]


def test_sorted_inputs(cuda):
    # adversarial orderings for the stratified sample: ascending and descending runs
    x = np.sort(O.ref_generate(NORMAL, 1 << 21, 77, b=1.0))
    for arr in (x, x[::-1].copy()):
        for k in [100, 1 << 15]:
            assert_same(gpu_topk(arr, k, 0, cuda), O.ref_topk(arr, k, 0, grid=8), f"sorted k={k}")


def test_errors(cuda):
    import torch
    rtk = _rtk()
    one = torch.tensor([3.5], device=cuda)
    with pytest.raises(rtk.empty_input_error):
        rtk.topk(torch.empty(0, device=cuda), 1)
    with pytest.raises(rtk.rank_out_of_range):
        rtk.topk(one, 2)
    with pytest.raises(rtk.rank_out_of_range):
        rtk.topk(one, 0)
    with pytest.raises(ValueError):
        rtk.topk(one, 1, cfg=rtk.EngineConfig(d=17))
    r = rtk.topk(one, 1)
    assert r.values.cpu().tolist() == [3.5] and r.indices.cpu().tolist() == [0]


def test_grid_config_invariance(cuda):
    # engine_test.cpp:305-322: results independent of grid/block/d hints
    rtk = _rtk()
    import torch
    x = O.ref_generate(NORMAL, 50000, 21, b=2.0)
    t = torch.from_numpy(x).to(cuda)
    base = rtk.topk(t, 777)
    for cfg in [rtk.EngineConfig(grid_size=1), rtk.EngineConfig(grid_size=8, d=8, block_size=512)]:
        r = rtk.topk(t, 777, cfg=cfg)
        assert torch.equal(r.values, base.values) and torch.equal(r.indices, base.indices)


# ---- batch -------------------------------------------------------------------------------
def _batch_expect(data, offsets, lengths, ks, order):
    return O.ref_batch_topk(data, offsets, lengths, ks, order, grid=8)


def test_batch_ragged_misaligned(cuda):
    # batch_test.cpp:145-165 / acceptance criterion 8: first task one element short
    import torch
    rtk = _rtk()
    tasks = [O.ref_generate(UNIFORM, (1 << 16) - (1 if t == 0 else 0), 600 + t) for t in range(16)]
    b = rtk.BatchInput.concatenate(tasks, [256] * 16)
    exp = _batch_expect(b.data, b.offsets, b.lengths, b.ks, 0)
    bd = rtk.BatchInput(torch.from_numpy(b.data).to(cuda), b.offsets, b.lengths, b.ks)
    got = rtk.batch_topk(bd, rtk.SelectionOrder.Largest)
    for t in range(16):
        assert_same((got[t].values, got[t].indices, got[t].pivot), exp[t], f"task {t}")


def test_batch_heterogeneous_k(cuda):
    # batch_test.cpp:122-143: Normal rows of varying n, k = 1 + 100 t, smallest
    import torch
    rtk = _rtk()
    tasks = [O.ref_generate(NORMAL, 3000 + 17 * t, 50 + t, b=1.0) for t in range(5)]
    ks = [1 + 100 * t for t in range(5)]
    b = rtk.BatchInput.concatenate(tasks, ks)
    exp = _batch_expect(b.data, b.offsets, b.lengths, b.ks, 1)
    got = rtk.batch_topk(rtk.BatchInput(torch.from_numpy(b.data).to(cuda), b.offsets, b.lengths, b.ks),
                         rtk.SelectionOrder.Smallest)
    for t in range(5):
        assert_same((got[t].values, got[t].indices, got[t].pivot), exp[t], f"task {t}")


@pytest.mark.parametrize("k", [50, 4096, 128256])
def test_batch_llm_vocab_rows(cuda, k):
    # BASELINE C3 shape (batch x 128256 logits), 16 rows here; bench runs 256
    import torch
    rtk = _rtk()
    V, B = 128256, 16
    tasks = [O.ref_generate(NORMAL, V, 100 + t, b=1.0) for t in range(B)]
    b = rtk.BatchInput.concatenate(tasks, [k] * B)
    exp = _batch_expect(b.data, b.offsets, b.lengths, b.ks, 0)
    got = rtk.batch_topk(rtk.BatchInput(torch.from_numpy(b.data).to(cuda), b.offsets, b.lengths, b.ks))
    for t in range(B):
        assert_same((got[t].values, got[t].indices, got[t].pivot), exp[t], f"row {t} k={k}")


def test_batch_errors(cuda):
    import torch
    rtk = _rtk()
    d = torch.tensor([1.0, 2.0, 3.0], device=cuda)
    with pytest.raises(ValueError, match="task 1"):
        rtk.batch_topk(rtk.BatchInput(d, [0, 2], [2, 1], [1, 2]))
    with pytest.raises(ValueError, match="overlaps"):
        rtk.batch_topk(rtk.BatchInput(d, [0, 1], [3, 1], [1, 1]))


# ---- scaling -----------------------------------------------------------------------------
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_scaled_matches_reference(cuda, mode):
    # scaling_test.cpp:106-139 and acceptance criterion 6 (acceptance_test.cpp:215-265)
    import torch
    rtk = _rtk()
    for n, seed in [(1 << 16, 1), (1 << 20, 5 + (1 << 20))]:
        x = O.ref_generate(UNIFORM, n, seed, a=128.6, b=128.7)
        wv, wi, wp, winfo = O.ref_scaled_topk(x, 512, 0, mode=mode, seed=31 + n, grid=4)
        info = rtk.ScaleInfo()
        r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), 512, rtk.SelectionOrder.Largest,
                            policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, 31 + n), info=info)
        assert info.scaled == winfo["scaled"] and info.a_index == (winfo["a_index"] if winfo["scaled"] else 0)
        assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"scaled mode={mode} n={n}")


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("n,k", [(3000, 700), (1 << 18, 1 << 17), (1 << 21, 4096)])
def test_scaled_smallest_and_shapes(cuda, mode, n, k):
    # the device-decided scale flag must reach every path: fused short rows, dense k >= n/2 rows,
    # the sampled-threshold pipeline; smallest order subtracts the same a_s (scaling.hpp:70-72)
    import torch
    rtk = _rtk()
    x = O.ref_generate(UNIFORM, n, 77 + n, a=128.6, b=128.7)
    for order in (0, 1):
        wv, wi, wp, winfo = O.ref_scaled_topk(x, k, order, mode=mode, seed=5 + k, grid=4)
        info = rtk.ScaleInfo()
        r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), k, rtk.SelectionOrder(order),
                            policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, 5 + k), info=info)
        assert info.scaled == winfo["scaled"]
        assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"scaled mode={mode} n={n} order={order}")


def test_adaptive_benign_does_not_scale(cuda):
    # scaling_test.cpp:173-196
    import torch
    rtk = _rtk()
    x = O.ref_generate(UNIFORM, 1 << 14, 43)
    info = rtk.ScaleInfo()
    r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), 128, policy=rtk.ScalePolicy(rtk.ScaleMode.Adaptive, 0.5, 13),
                        info=info)
    assert not info.scaled
    assert_same((r.values, r.indices, r.pivot), O.ref_topk(x, 128, 0), "benign adaptive")


# ---- host entry points (numpy in / numpy out) --------------------------------------------
def test_host_entry_points(cuda):
    rtk = _rtk()
    x = O.ref_generate(UNIFORM, 1 << 20, 3)
    r = rtk.topk(x, 1000)
    assert_same((r.values, r.indices, r.pivot), O.ref_topk(x, 1000, 0, grid=4), "host topk")
    tasks = [O.ref_generate(NORMAL, 5000 + t, 9 + t, b=1.0) for t in range(7)]
    b = rtk.BatchInput.concatenate(tasks, [100 * (t + 1) for t in range(7)])
    got = rtk.batch_topk(b)
    exp = _batch_expect(b.data, b.offsets, b.lengths, b.ks, 0)
    for t in range(7):
        assert_same((got[t].values, got[t].indices, got[t].pivot), exp[t], f"host task {t}")
    y = O.ref_generate(UNIFORM, 1 << 16, 2, a=128.6, b=128.7)
    wv, wi, wp, _ = O.ref_scaled_topk(y, 512, 0, mode=1, seed=2)
    r = rtk.scaled_topk(y, 512, policy=rtk.ScalePolicy(rtk.ScaleMode.Always, 0.5, 2))
    assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), "host scaled")


# ---- 16-bit floats ---------------------------------------------------
# The reference declares f16 (io.hpp:3, dtype code 2) but does not build it (io.cpp:71-72). Both f16
# and bf16 widen EXACTLY and order-preservingly to f32 (NaN payloads, +-0 and +-inf included), so
# the reference engine on the widened input is the oracle: identical indices, and the returned
# 16-bit words must be the inputs at those indices (bit-exact widening: tests/test_oracle.py).
def _widen16(h, kind):
    from tests.test_oracle import widen16_exact
    return widen16_exact(h, kind).view(np.float32)


def _gpu_topk16(t16, k, order, cuda):
    import torch
    rtk = _rtk()
    r = rtk.topk(t16.to(cuda), k, rtk.SelectionOrder(order))
    return r.values.view(torch.int16).cpu().numpy().view(np.uint16), r.indices.cpu().numpy(), r


def _check16(h, t16, x32, k, order, cuda, what):
    gv, gi, r = _gpu_topk16(t16, k, order, cuda)
    _, wi, _ = O.ref_topk(x32, k, order, grid=4)
    bad = np.nonzero(gi.astype(np.uint64) != wi.astype(np.uint64))[0]
    assert bad.size == 0, f"{what}: index mismatch at ranks {bad[:5]}"
    assert np.array_equal(gv, h[wi.astype(np.int64)]), f"{what}: value bits"
    # pivot = k-th value (engine.hpp:333): compare through the widened f32 value
    pv = np.float32(r.pivot)
    assert pv.view(np.uint32) == x32[wi[-1]].view(np.uint32) or (np.isnan(pv) and np.isnan(x32[wi[-1]])), f"{what}: pivot"


@pytest.mark.parametrize("kind", ["bf16", "f16"])
@pytest.mark.parametrize("n", [1000, 1 << 16, (1 << 20) + 3])
@pytest.mark.parametrize("order", [0, 1])
def test_16bit_topk(cuda, kind, n, order):
    rng = np.random.default_rng(7000 + n + (kind == "f16") * 3 + order)
    import torch
    x = torch.from_numpy(rng.standard_normal(n).astype(np.float32))
    t16 = x.to(torch.bfloat16 if kind == "bf16" else torch.float16)
    h = t16.view(torch.int16).numpy().view(np.uint16).copy()
    x32 = _widen16(h, kind)
    for k in sorted({1, 50, 512, n // 2, n}):
        _check16(h, t16, x32, k, order, cuda, f"{kind} n={n} order={order} k={k}")


@pytest.mark.parametrize("kind", ["bf16", "f16"])
def test_16bit_special_values_and_ties(cuda, kind):
    import torch
    dt = torch.bfloat16 if kind == "bf16" else torch.float16
    base = torch.tensor([float("nan"), float("inf"), 1.0, 0.0, -0.0, -1.0, float("-inf"), -float("nan"), 1.0, 0.0],
                        dtype=torch.float32).to(dt)
    t16 = base.repeat(4000)  # heavy ties: every value 4000 times
    h = t16.view(torch.int16).numpy().view(np.uint16).copy()
    h[::997] = 0x7C01 if kind == "f16" else 0x7F81  # signalling-NaN payloads too
    t16 = torch.from_numpy(h.view(np.int16)).view(dt)
    x32 = _widen16(h, kind)
    for order in (0, 1):
        for k in (1, 7, 3999, 12345, t16.numel()):
            _check16(h, t16, x32, k, order, cuda, f"{kind} special order={order} k={k}")


@pytest.mark.parametrize("k", [50, 4096, 32000])
def test_16bit_batch_llm_rows(cuda, k):
    # C3-like bf16 logits: 8 rows of a 32000 vocabulary, batch == per-row topk (batch_test.cpp:90-107)
    import torch
    rtk = _rtk()
    B, V = 8, 32000
    g = torch.Generator().manual_seed(11)
    logits = torch.randn(B, V, generator=g).to(torch.bfloat16)
    r = rtk.batch_topk_dense(logits.to(cuda), k)
    gv = r.values.view(torch.int16).cpu().numpy().view(np.uint16)
    gi = r.indices.cpu().numpy()
    h = logits.view(torch.int16).numpy().view(np.uint16)
    x32 = _widen16(h.reshape(-1), "bf16").reshape(B, V)
    for t in range(B):
        _, wi, _ = O.ref_topk(np.ascontiguousarray(x32[t]), k, 0, grid=4)
        assert np.array_equal(gi[t].astype(np.uint64), wi.astype(np.uint64)), f"row {t}"
        assert np.array_equal(gv[t], h[t][wi.astype(np.int64)]), f"row {t} values"


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("kind", [UNIFORM, ZIPF])
def test_sharded_query_merge_on_device(cuda, G, kind):
    # SURVEY §8e / C5 on one device: per-shard rtk_topk (contiguous index ranges), the shard
    # blocks concatenated in shard order (the NCCL all-gather's layout), rtk_merge_shards; must
    # equal rtk::topk on the whole query — ties across shard boundaries included (Zipf).
    import torch
    rtk = _rtk()
    from paper_2501_14336_b200 import sharded as SH
    n, k = (1 << 20) + 13, 4096
    x = O.ref_generate(kind, n, 4242 + G, dtype=np.float32, b=1.0)
    t = torch.from_numpy(x).to(cuda)
    vals, idx, bases = [], [], []
    for g in range(G):
        s0, ln = SH.shard_bounds(n, G, g)
        r = rtk.topk(t[s0:s0 + ln], k)
        vals.append(r.values)
        idx.append(r.indices)
        bases.append(s0)
    m = rtk.merge_shards(torch.cat(vals), torch.cat(idx), [k] * G, bases, k)
    assert_same((m.values, m.indices, m.pivot), O.ref_topk(x, k, 0, grid=4), f"G={G} kind={kind}")


# ---- bench/report harness ------------------------------------------------
def test_report_bench_checksum_matches_reference(cuda):
    # `rtk bench` cell semantics (rtk_cli.cpp:372-420): tasks seeded seed + 100 t + n + k, the first
    # one n - 1 long, checksum = XOR of per-task FNV-1a; the reference's batch_topk on the same
    # inputs must give the same checksum
    from paper_2501_14336_b200 import report
    n, k, B, seed = 1 << 16, 100, 3, 4
    rep = report.bench([n], [k], batch=B, repeats=2, seed=seed, verify=True)
    cell = rep["cells"][0]
    assert cell["verified"] and "error" not in cell
    want = 0
    for t in range(B):
        x = O.ref_generate(0, n - 1 if t == 0 else n, seed + 100 * t + n + k)
        v, i, _ = O.ref_topk(x, k, 0, grid=4)
        want ^= report.result_checksum(v, i)
    assert cell["checksum"] == want
    q = report.bench([4096], [], batch=1, repeats=1, quantile=True)
    assert [c["k"] for c in q["cells"]] == [40, 1024, 2048]


# ---- LLM sampling consumer --------------------------------------------------
def _sample_ref(v: np.ndarray, idx: np.ndarray, top_p: float, T: float, u: float):
    """fp64 restatement of rtk_topk_sample's definition (rtk_c.h) on one row's canonical top-k."""
    e = np.exp((v.astype(np.float64) - float(v[0])) / T)
    c = np.cumsum(e)
    m = len(e) if top_p >= 1.0 else int(np.searchsorted(c, top_p * c[-1], side="left")) + 1
    m = min(m, len(e))
    q = e[:m] / c[m - 1]
    cq = np.cumsum(q)
    j = min(int(np.searchsorted(cq, u, side="right")), m - 1)
    return int(idx[j]), q, m, cq


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("k,top_p,T", [(50, 0.9, 1.0), (1, 1.0, 1.0), (4096, 0.95, 0.7), (128256, 0.5, 1.3),
                                       (200, 1.0, 2.0)])
def test_topk_sample(cuda, dtype, k, top_p, T):
    import torch
    rtk = _rtk()
    B, V = 24, 128256
    g = torch.Generator(device="cuda")
    g.manual_seed(7 + k)
    logits = (torch.randn(B, V, device=cuda, generator=g) * 3).to(
        {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dtype])
    u = torch.rand(B, device=cuda, generator=g)
    tok, probs, ti = rtk.topk_sample(logits, k, top_p=top_p, temperature=T, uniform=u, return_probs=True)
    plain = rtk.topk_sample(logits, k, top_p=top_p, temperature=T, uniform=u)
    assert torch.equal(tok, plain)
    L = logits.float().cpu().numpy()
    tok, probs, ti, u = tok.cpu().numpy(), probs.cpu().numpy(), ti.cpu().numpy(), u.cpu().numpy()
    for b in range(B):
        # the top-k indices are the exact canonical top-k (checked bit-exactly elsewhere); values
        # are the logits at those indices
        v = L[b, ti[b]]
        assert np.all(v[:-1] >= v[1:])
        want, q, m, cq = _sample_ref(v, ti[b], top_p, T, float(u[b]))
        assert np.allclose(probs[b, :m], q, rtol=1e-4, atol=2e-6), f"row {b} probs"
        margin = np.min(np.abs(cq - u[b])) if m > 0 else 1.0
        if margin > 1e-5:  # u not within fp32 rounding of a CDF step
            assert tok[b] == want, f"row {b}: token {tok[b]} != {want} (u={u[b]}, margin {margin})"
        assert np.all(probs[b, m + 2:] == 0)


def test_topk_sample_errors(cuda):
    import torch
    rtk = _rtk()
    x = torch.randn(2, 100, device=cuda)
    with pytest.raises(ValueError, match="top_p"):
        rtk.topk_sample(x, 5, top_p=0.0)
    with pytest.raises(ValueError, match="temperature"):
        rtk.topk_sample(x, 5, temperature=0.0)
    with pytest.raises(IndexError):
        rtk.topk_sample(x, 101)


@pytest.mark.parametrize("mode", ["all", "off", "16"])
def test_dense_rows_lsd_forced(cuda, mode):
    # dense rows (k >= n/2): the segmented one-sweep LSD sort (default, RTK_LSD=all), the MSD +
    # bucket-sort path (off) and LSD for 16-bit keys only (16), each in a fresh process; all must
    # equal the reference per row, ragged rows, both orders, u32 ties and heavy f32 ties included
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle as O, paper_2501_14336_b200 as rtk
rng = np.random.default_rng(3)
lens = [5000, 4096, 12289, 70001]
offs = [0]
for n in lens[:-1]: offs.append(offs[-1] + n + 3)
data = rng.standard_normal(offs[-1] + lens[-1]).astype(np.float32)
data[offs[2]:offs[2] + lens[2]:3] = 0.5
ks = [5000, 2048, 12289, 40000]
for order in (0, 1):
    b = rtk.BatchInput(torch.from_numpy(data).cuda(), offs, lens, ks)
    got = rtk.batch_topk(b, rtk.SelectionOrder(order))
    for t in range(4):
        x = data[offs[t]:offs[t] + lens[t]]
        wv, wi, _ = O.port_topk(x, ks[t], order)
        assert np.array_equal(got[t].values.cpu().numpy().view(np.uint32), wv.view(np.uint32)), (order, t)
        assert np.array_equal(got[t].indices.cpu().numpy().astype(np.uint64), wi), (order, t)
u = rng.integers(0, 50, 3 * 9000, dtype=np.uint32)
b = rtk.BatchInput(torch.from_numpy(u.view(np.int32)).cuda().view(torch.uint32), [0, 9000, 18000], [9000] * 3, [9000, 6000, 4500])
got = rtk.batch_topk(b)
for t in range(3):
    wv, wi, _ = O.port_topk(u[9000 * t:9000 * (t + 1)], [9000, 6000, 4500][t], 0)
    assert np.array_equal(got[t].indices.cpu().numpy().astype(np.uint64), wi), ("u32", t)
print("ok")
''' % ROOT
    env = dict(os.environ, RTK_LSD=mode)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr


def test_bench_helpers_time_the_same_call(cuda):
    # rtk_bench_topk / rtk_bench_scaled time back-to-back calls with engine-recorded events; the
    # outputs of the timed calls are the same as one plain call's (checked on the scaled path)
    import torch
    from paper_2501_14336_b200 import rtk as R
    x = torch.from_numpy(O.ref_generate(UNIFORM, 1 << 22, 5, a=128.6, b=128.7)).to(cuda)
    b = R.bench_topk(x, 4096, 4, 1)
    assert b.median_ms > 0 and len(b.device_ms) == 4 and all(p > 0 for p in b.device_ms)
    assert all(h >= d * 0.5 for h, d in zip(b.host_ms, b.device_ms))
    pol = R.ScalePolicy(mode=R.ScaleMode(2), trigger_fraction=0.5, seed=31)
    b = R.bench_scaled(x, 4096, 4, 1, policy=pol)
    assert b.median_ms > 0 and all(p > 0 for p in b.device_ms)
    got = R.scaled_topk(x, 4096, policy=pol)
    want = O.ref_scaled_topk(x.cpu().numpy(), 4096, 0, mode=2, tau=0.5, seed=31)
    assert np.array_equal(got.indices.cpu().numpy().astype(np.uint64), np.asarray(want[1], dtype=np.uint64))


@pytest.mark.parametrize("n", [6911791, 3 * (1 << 20) + 5, (1 << 22) + (1 << 21) - 3])
def test_sample_cluster_sizes(cuda, n):
    # huge rows whose stratified sample (n/128 elements) is not a power of two: the sample
    # kernel's cluster must still be a power of two (its 2048 bins split into equal slices);
    # found by tests/test_gpu_fuzz.py (n = 6911791: 13 CTAs before the fix, misaligned DSMEM)
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n).astype(np.float32)
    for k, order in [(398, 1), (1000, 0), (70000, 0)]:
        assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=8), f"n={n} k={k}")
        u = x.view(np.uint32)
        assert_same(gpu_topk(u, k, order, cuda), O.ref_topk(u, k, order, grid=8), f"u32 n={n} k={k}")


def test_batch_tiny_misaligned_rows(cuda):
    # rows shorter than their distance to 16-byte alignment (n = 1..7 at every misalignment,
    # f32 / u32 / f16 / bf16): k_rows_fused's scalar head must stop at the row's end (found by
    # tools/fuzz_explore.py: a 1-element row read its neighbours)
    import torch
    rtk = _rtk()
    rng = np.random.default_rng(77)
    lens = [n for n in range(1, 8) for _ in range(8)] + [3000]
    offs, pos = [], 0
    for t, n in enumerate(lens):
        pos += t % 5
        offs.append(pos)
        pos += n
    data = rng.standard_normal(pos).astype(np.float32)
    ks = [1 + (t % n) for t, n in enumerate(lens)]
    for order in (0, 1):
        exp = _batch_expect(data, offs, lens, ks, order)
        got = rtk.batch_topk(rtk.BatchInput(torch.from_numpy(data).to(cuda), offs, lens, ks), rtk.SelectionOrder(order))
        for t in range(len(lens)):
            assert_same((got[t].values, got[t].indices, got[t].pivot), exp[t], f"f32 row {t} n={lens[t]}")
    for kind in ("bf16", "f16"):
        t16 = torch.from_numpy(data).to(torch.bfloat16 if kind == "bf16" else torch.float16)
        h = t16.view(torch.int16).numpy().view(np.uint16).copy()
        x32 = _widen16(h, kind)
        exp = _batch_expect(x32, offs, lens, ks, 0)
        got = rtk.batch_topk(rtk.BatchInput(t16.to(cuda), offs, lens, ks))
        for t in range(len(lens)):
            gi = got[t].indices.cpu().numpy().astype(np.uint64)
            assert np.array_equal(gi, exp[t][1].astype(np.uint64)), f"{kind} row {t} n={lens[t]}"

"""GPU parity of the rare paths, forced, plus the crafted and lifecycle cases.

* "force_exact" (rtk_set_option): every row takes the exact path — radix_select's digit passes
  with the early stop (engine.hpp:293-312), then the re-compaction and the ordering — as if its
  sampled threshold had missed. Each call must report fallback_rows == rows.
* "force_deep": the level-0 MSD digit is cut to 6 bits so buckets exceed one CTA sort and the
  host-driven deeper levels run (rtk_stats.deep_levels >= 1).
* k_compact's dense-hit branch must feed the per-row key OR that sets the MSD digit's trailing
  zero squeeze (plan_row's tz): a tile-aligned run of fine-grained keys next to sparse "round"
  keys sharing the threshold's low zero bits.
* scaled_topk NaN propagation as on x86 (x NaN, a_s NaN, inf - inf).
* graph replay with the input rewritten in place between calls; concurrent callers of one
  handle.
All expectations come from the reference compiled in place (oracle/_ref).
"""
import os
import threading

import numpy as np
import pytest

import oracle as O
from tests.test_gpu_parity import NORMAL, UNIFORM, ZIPF, assert_same, gpu_topk

pytestmark = pytest.mark.gpu
CORES = os.cpu_count() or 4


def _rtk():
    import paper_2501_14336_b200 as rtk
    return rtk


@pytest.fixture
def force_exact(cuda):
    rtk = _rtk()
    rtk.set_option("force_exact", 1)
    yield
    rtk.set_option("force_exact", 0)


@pytest.fixture
def force_deep(cuda):
    rtk = _rtk()
    rtk.set_option("force_deep", 1)
    yield
    rtk.set_option("force_deep", 0)


def test_unknown_option(cuda):
    with pytest.raises(ValueError, match="unknown option"):
        _rtk().set_option("no_such_switch", 1)


# ---- exact path ------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [10, 3001, 1 << 16, (1 << 20) + 3])
@pytest.mark.parametrize("kind", [UNIFORM, ZIPF])
@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("dtype", [np.float32, np.uint32])
def test_exact_path_randomized(force_exact, cuda, n, kind, order, dtype):
    # acceptance criterion 1's grid (acceptance_test.cpp:48-94) through the exact path
    rtk = _rtk()
    x = O.ref_generate(kind, n, 20000 + n + kind * 3 + order, dtype=dtype, b=1.0)
    for k in sorted({1, 7, 512, n // 2, n}):
        if k < 1 or k > n:
            continue
        assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=CORES), f"exact n={n} k={k}")
        st = rtk.last_stats()
        assert st.fallback_rows == 1 and st.passes >= 1, st


def test_exact_path_ties(force_exact, cuda):
    # engine_test.cpp:188-198 (duplicates: window exhaustion) and acceptance criterion 2
    x = np.full((1 << 20) + 5, -7.0, dtype=np.float32)
    for k in (1, 40000, x.size):
        assert_same(gpu_topk(x, k, 0, cuda), O.ref_topk(x, k, 0, grid=CORES), f"dupes k={k}")
    y = np.ones(1 << 16, dtype=np.float32)
    y[::2] = 2.0
    assert_same(gpu_topk(y, 40000, 0, cuda), O.ref_topk(y, 40000, 0), "two values")
    z = O.ref_generate(UNIFORM, 1 << 22, 5 + (1 << 22), a=128.6, b=128.7)
    assert_same(gpu_topk(z, 1 << 16, 0, cuda), O.ref_topk(z, 1 << 16, 0, grid=CORES), "narrow band")


def test_exact_path_batch(force_exact, cuda):
    # batch_test.cpp:90-165 shapes through the exact path; BatchRunInfo counts the extra passes
    import torch
    rtk = _rtk()
    tasks = [O.ref_generate(NORMAL, 3000 + 4099 * t, 50 + t, b=1.0) for t in range(6)]
    tasks.append(O.ref_generate(NORMAL, 128256, 106, b=1.0))
    ks = [1, 100, 4096, 5000, 2, 20000, 128256]
    b = rtk.BatchInput.concatenate(tasks, ks)
    exp = O.ref_batch_topk(b.data, b.offsets, b.lengths, b.ks, 1, grid=CORES)
    info = rtk.BatchRunInfo()
    got = rtk.batch_topk(rtk.BatchInput(torch.from_numpy(b.data).to(cuda), b.offsets, b.lengths, b.ks),
                         rtk.SelectionOrder.Smallest, info=info)
    for t in range(len(ks)):
        assert_same((got[t].values, got[t].indices, got[t].pivot), exp[t], f"task {t}")
    assert rtk.last_stats().fallback_rows == len(ks)
    assert len(info.task_passes) == len(ks) and all(p >= 3 for p in info.task_passes), info


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_exact_path_scaled(force_exact, cuda, mode):
    import torch
    rtk = _rtk()
    n = 1 << 20
    x = O.ref_generate(UNIFORM, n, 5 + n, a=128.6, b=128.7)
    wv, wi, wp, winfo = O.ref_scaled_topk(x, 4096, 0, mode=mode, seed=31, grid=CORES)
    info = rtk.ScaleInfo()
    r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), 4096, policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, 31),
                        info=info)
    assert info.scaled == winfo["scaled"]
    assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"exact scaled mode={mode}")
    assert rtk.last_stats().fallback_rows == 1


@pytest.mark.parametrize("kind", ["bf16", "f16"])
def test_exact_path_16bit(force_exact, cuda, kind):
    import torch
    from tests.test_gpu_parity import _check16, _widen16
    rng = np.random.default_rng(99)
    t16 = torch.from_numpy(rng.standard_normal((1 << 18) + 7).astype(np.float32)).to(
        torch.bfloat16 if kind == "bf16" else torch.float16)
    h = t16.view(torch.int16).numpy().view(np.uint16).copy()
    x32 = _widen16(h, kind)
    for order in (0, 1):
        for k in (1, 50, 5000, t16.numel() // 2):
            _check16(h, t16, x32, k, order, cuda, f"exact {kind} order={order} k={k}")


# ---- deeper MSD levels -------------------------------------------------------------------------
@pytest.mark.parametrize("kind", [UNIFORM, NORMAL, ZIPF])
@pytest.mark.parametrize("k", [1 << 17, 1 << 19])
def test_deep_levels(force_deep, cuda, kind, k):
    rtk = _rtk()
    x = O.ref_generate(kind, 1 << 22, 300 + kind, b=1.0)
    for order in (0, 1):
        assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=CORES), f"deep kind={kind} k={k}")
        assert rtk.last_stats().deep_levels >= 1


def test_deep_levels_ties_and_scaled(force_deep, cuda):
    import torch
    rtk = _rtk()
    n = 1 << 22
    x = O.ref_generate(UNIFORM, n, 5 + n, a=128.6, b=128.7)
    assert_same(gpu_topk(x, 1 << 18, 0, cuda), O.ref_topk(x, 1 << 18, 0, grid=CORES), "deep narrow band")
    assert rtk.last_stats().deep_levels >= 1
    for mode in (1, 2):
        wv, wi, wp, _ = O.ref_scaled_topk(x, 1 << 18, 0, mode=mode, seed=31, grid=CORES)
        r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), 1 << 18, policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, 31))
        assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"deep scaled mode={mode}")


def test_deep_levels_batch(force_deep, cuda):
    import torch
    rtk = _rtk()
    V, B = 1 << 20, 3
    data = np.concatenate([O.ref_generate(NORMAL, V, 700 + t, b=1.0) for t in range(B)])
    ks = [300000, 1 << 18, 150000]
    offs = [t * V for t in range(B)]
    exp = O.ref_batch_topk(data, offs, [V] * B, ks, 0, grid=CORES)
    info = rtk.BatchRunInfo()
    got = rtk.batch_topk(rtk.BatchInput(torch.from_numpy(data).to(cuda), offs, [V] * B, ks), info=info)
    for t in range(B):
        assert_same((got[t].values, got[t].indices, got[t].pivot), exp[t], f"deep batch row {t}")
    assert info.phase_b_rounds >= 1


# ---- k_compact dense-hit branch and the MSD digit's trailing-zero squeeze ------------------------
def _round_and_run(n, run_len, ascending, rng):
    """u32 keys: background < 2^20; 'round' keys 0x40000000 + j * 2^16 (j < 4) at ~2 % density
    (sparse, staged hits); one tile-aligned run of run_len consecutive keys 0x40040001 + i above
    them (dense hits, > 512 per warp-tile), in ascending or descending index order."""
    x = rng.integers(0, 1 << 20, n, dtype=np.uint32)
    pos = np.nonzero(rng.random(n) < 0.02)[0]
    x[pos] = (0x40000000 + (rng.integers(0, 4, pos.size, dtype=np.uint32) << 16)).astype(np.uint32)
    start = 8192 * 37
    run = (0x40040001 + np.arange(run_len, dtype=np.uint32)).astype(np.uint32)
    x[start:start + run_len] = run if ascending else run[::-1]
    return x


@pytest.mark.parametrize("ascending", [True, False])
@pytest.mark.parametrize("dtype", ["u32", "f32"])
@pytest.mark.parametrize("order", [0, 1])
def test_dense_hits_keep_key_or(cuda, ascending, dtype, order):
    rng = np.random.default_rng(1234 + ascending)
    n, run_len = 1 << 22, 32768
    x = _round_and_run(n, run_len, ascending, rng)
    if order == 1:  # the same key structure under Smallest: complemented keys
        x = ~x if dtype == "u32" else x | np.uint32(0x80000000)
    if dtype == "f32":
        x = x.view(np.float32)
    # k: the whole run plus part of the top round key's copies, so T lands on a round key
    for k in (run_len + 30000, run_len + 50000):
        assert_same(gpu_topk(x, k, order, cuda), O.ref_topk(x, k, order, grid=CORES),
                    f"dense+round {dtype} asc={ascending} order={order} k={k}")


# ---- scaled_topk NaN propagation (x86 subss rules, scaling.hpp:69-70) ---------------------------
@pytest.mark.parametrize("mode", [1, 2])
def test_scaled_nan_propagation(cuda, mode):
    import torch
    rtk = _rtk()
    n, k, seed = 1 << 20, 4096, 77
    base = O.ref_generate(UNIFORM, n, 9, a=128.6, b=128.7)
    a_index = O.ref_scaled_topk(base, k, 0, mode=1, seed=seed)[3]["a_index"]

    def nan(bits):
        return np.array([bits], dtype=np.uint32).view(np.float32)[0]

    cases = {}
    x = base.copy()
    x[::1001] = nan(0x7FC01234)   # +qNaN with payload
    x[5::1003] = nan(0xFFA00007)  # -sNaN with payload (quieted by the subtraction)
    cases["x NaN"] = x
    x = base.copy()
    x[::4097] = nan(0x7F800001)
    x[a_index] = nan(0xFF812345)  # a_s is a negative sNaN: every y = a_s quieted
    cases["a_s NaN"] = x
    x = base.copy()
    x[::777] = np.float32(np.inf)  # inf - inf = x86 default NaN 0xFFC00000
    x[3::999] = -np.float32(np.inf)
    x[a_index] = np.float32(np.inf)
    cases["inf - inf"] = x
    for name, x in cases.items():
        for order in (0, 1):
            wv, wi, _, winfo = O.ref_scaled_topk(x, k, order, mode=mode, seed=seed, grid=CORES)
            r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), k, rtk.SelectionOrder(order),
                                policy=rtk.ScalePolicy(rtk.ScaleMode(mode), 0.5, seed))
            gv = r.values.cpu().numpy().view(np.uint32)
            gi = r.indices.cpu().numpy().astype(np.uint64)
            assert np.array_equal(gi, wi.astype(np.uint64)), f"{name} mode={mode} order={order}: indices"
            assert np.array_equal(gv, wv.view(np.uint32)), f"{name} mode={mode} order={order}: values"


# ---- graph replay with in-place rewrites ----------------------------------------------------------
def test_replay_with_inplace_rewrites(cuda):
    # repeated identical calls replay one CUDA graph from the third call on (same pointers, shape,
    # k): the input rewritten in place between calls must be re-read every time — the LLM decode
    # loop usage. Tie-heavy and sorted contents mid-sequence change the candidate structure.
    import torch
    rtk = _rtk()
    n, k = 1 << 22, 4096
    t = torch.empty(n, dtype=torch.float32, device=cuda)
    contents = [O.ref_generate(UNIFORM, n, 1000 + i) for i in range(3)]
    contents.insert(1, O.ref_generate(UNIFORM, n, 5 + n, a=128.6, b=128.7))
    contents.insert(3, np.sort(O.ref_generate(NORMAL, n, 3, b=1.0)))
    contents.append(np.full(n, 1.5, dtype=np.float32))
    for i, x in enumerate(contents * 2):
        t.copy_(torch.from_numpy(x))
        r = rtk.topk(t, k)
        assert_same((r.values, r.indices, r.pivot), O.ref_topk(x, k, 0, grid=CORES), f"topk call {i}")
    B, V, kb = 32, 128256, 50
    tb = torch.empty(B, V, dtype=torch.float32, device=cuda)
    for i in range(5):
        d = np.concatenate([O.ref_generate(NORMAL, V, 40 * i + t, b=1.0) for t in range(B)])
        if i == 2:
            d[:] = np.round(d, 1)  # heavy ties
        tb.copy_(torch.from_numpy(d).view(B, V))
        r = rtk.batch_topk_dense(tb, kb)
        exp = O.ref_batch_topk(d, [j * V for j in range(B)], [V] * B, [kb] * B, 0, grid=CORES)
        gv, gi, gp = r.values.cpu().numpy(), r.indices.cpu().numpy(), r.pivot.cpu().numpy()
        for row in range(B):
            assert_same((gv[row], gi[row], gp[row]), exp[row], f"batch call {i} row {row}")
    ts = torch.empty(n, dtype=torch.float32, device=cuda)
    pol = rtk.ScalePolicy(rtk.ScaleMode.Adaptive, 0.5, 31)
    for i in range(5):
        x = O.ref_generate(UNIFORM, n, 60 + i, a=128.6 if i % 2 == 0 else 0.0, b=128.7 if i % 2 == 0 else 1.0)
        ts.copy_(torch.from_numpy(x))
        r = rtk.scaled_topk(ts, k, policy=pol)
        wv, wi, wp, _ = O.ref_scaled_topk(x, k, 0, mode=2, seed=31, grid=CORES)
        assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"scaled call {i}")


def test_replay_with_forced_exact(force_exact, cuda):
    # the exact path runs on the host after a replayed graph as well
    import torch
    rtk = _rtk()
    n, k = 1 << 21, 1000
    t = torch.empty(n, dtype=torch.float32, device=cuda)
    for i in range(5):
        x = O.ref_generate(UNIFORM, n, 500 + i)
        t.copy_(torch.from_numpy(x))
        r = rtk.topk(t, k)
        assert_same((r.values, r.indices, r.pivot), O.ref_topk(x, k, 0, grid=CORES), f"call {i}")
        assert rtk.last_stats().fallback_rows == 1


# ---- one handle, several threads ------------------------------------------------------------------
def test_concurrent_callers_share_one_handle(cuda):
    import torch
    rtk = _rtk()
    xs = [O.ref_generate(UNIFORM if i % 2 else NORMAL, (1 << 20) + 17 * i, 900 + i, b=1.0) for i in range(6)]
    want = [O.ref_topk(x, 1000 + i, 0, grid=CORES) for i, x in enumerate(xs)]
    errors = []
    rtk.topk(torch.from_numpy(xs[0]).to(cuda), 10)  # the device's handle exists before the threads

    def worker(i):
        try:
            torch.cuda.set_device(cuda)
            s = torch.cuda.Stream(device=cuda)
            t = torch.from_numpy(xs[i]).to(cuda)
            for _ in range(4):
                with torch.cuda.stream(s):
                    r = rtk.topk(t, 1000 + i)
                    got = (r.values.cpu(), r.indices.cpu(), r.pivot)
                assert_same(got, want[i], f"thread {i}")
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors


# ---- Adaptive scaling: the sampled trigger guess and its exact verification ------------------------
@pytest.mark.parametrize("order", [0, 1])
def test_adaptive_guess_accepted_and_rejected(cuda, order):
    # scaling.hpp:47-58 decides on the EXACT first-window histogram. The library guesses from a
    # sample (k_scale_guess) and verifies with exact counts taken in the same streaming pass; a
    # wrong guess reruns with the exact trigger pass (stats.passes == 1). Both must equal the
    # reference bit for bit.
    import torch
    rtk = _rtk()
    n, k = 1 << 22, 400
    narrow = O.ref_generate(UNIFORM, n, 77, a=128.6, b=128.7)  # one fat bin: guess "scale", accepted
    hidden = O.ref_generate(UNIFORM, n, 78)                     # top-k hidden between sample segments
    stride = (n - 32) // 511
    pos = np.array([s * stride + 4000 + j for s in range(511) for j in range(2)])
    hidden[pos] = -1000.0 if order else 1000.0
    balanced = O.ref_generate(UNIFORM, n, 79)                   # the k-th bin holds ~half the row
    balanced[: n // 2 + 1] = np.float32(1.5) if order == 0 else np.float32(-1.5)
    for name, x, want_passes in (("narrow", narrow, 0), ("hidden", hidden, 1), ("balanced", balanced, None)):
        for tau in (0.5, 0.3):
            wv, wi, wp, winfo = O.ref_scaled_topk(x, k, order, mode=2, tau=tau, seed=31, grid=CORES)
            info = rtk.ScaleInfo()
            r = rtk.scaled_topk(torch.from_numpy(x).to(cuda), k, rtk.SelectionOrder(order),
                                policy=rtk.ScalePolicy(rtk.ScaleMode.Adaptive, tau, 31), info=info)
            assert info.scaled == winfo["scaled"], (name, tau)
            assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), f"adaptive {name} tau={tau}")
            if want_passes is not None:
                assert rtk.last_stats().passes == want_passes, (name, rtk.last_stats())

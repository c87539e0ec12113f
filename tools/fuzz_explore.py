"""Long fuzz exploration (not part of the suite): tests/test_gpu_fuzz.py's generators over many
seeds, batches and single queries, plus scaled_topk and 16-bit rows; prints failures and goes on.
python tools/fuzz_explore.py SEED0 COUNT"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2501_14336_b200 as rtk
from tests.test_gpu_fuzz import _k, _row
from tests.test_gpu_parity import assert_same, gpu_topk

dev = torch.device("cuda", 0)
s0, cnt = int(sys.argv[1]), int(sys.argv[2])
fails = 0
t_end = time.time() + float(os.environ.get("FUZZ_SECONDS", "1e9"))
for case in range(s0, s0 + cnt):
    if time.time() > t_end:
        break
    rng = np.random.default_rng(case)
    dtype = np.float32 if rng.integers(0, 3) else np.uint32
    order = int(rng.integers(0, 2))
    what = ""
    try:
        mode = rng.integers(0, 8)
        force = rng.integers(0, 8)  # 1/8 of the cases on a forced rare path
        rtk.set_option("force_exact", 1 if force == 0 else 0)
        rtk.set_option("force_deep", 1 if force == 1 else 0)
        if mode == 0:  # single query
            n = int(rng.choice([rng.integers(1, 1 << 18), rng.integers((1 << 18) + 1, (1 << 21) + 1),
                                rng.integers(1 << 21, 1 << 24)]))
            x = _row(rng, n, dtype)
            k = min(n, int(rng.integers(1, 513))) if rng.integers(0, 2) else _k(rng, n)
            what = f"single n={n} k={k} order={order} {dtype.__name__}"
            assert_same(gpu_topk(x, k, order, dev), O.ref_topk(x, k, order, grid=16), what)
        elif mode == 1:  # batch
            B = int(rng.integers(1, 40))
            lens = [int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 200000), rng.integers(200000, 1 << 21)],
                                   p=[0.5, 0.4, 0.1])) for _ in range(B)]
            rows = [_row(rng, n, dtype) for n in lens]
            ks = [_k(rng, n) for n in lens]
            offs, parts, pos = [], [], 0
            for t in range(B):
                g = int(rng.integers(0, 9))
                parts.append(np.zeros(g, dtype=dtype))
                pos += g
                offs.append(pos)
                parts.append(rows[t])
                pos += lens[t]
            data = np.concatenate(parts)
            what = f"batch B={B} order={order} {dtype.__name__}"
            exp = O.ref_batch_topk(data, offs, lens, ks, order, grid=16)
            td = torch.from_numpy(data.view(np.int32) if dtype == np.uint32 else data).to(dev)
            if dtype == np.uint32:
                td = td.view(torch.uint32)
            got = rtk.batch_topk(rtk.BatchInput(td, offs, lens, ks), rtk.SelectionOrder(order))
            for t in range(B):
                gv = got[t].values
                if dtype == np.uint32:
                    gv = gv.view(torch.int32).cpu().numpy().view(np.uint32)
                assert_same((gv, got[t].indices, got[t].pivot), exp[t], what + f" row {t} n={lens[t]} k={ks[t]}")
        elif mode == 2:  # scaled_topk
            n = int(rng.choice([rng.integers(1, 1 << 16), rng.integers(1 << 16, 1 << 22)]))
            lo = float(rng.choice([0.0, 128.6, -3.0, 1e6]))
            x = (np.float32(lo) + np.float32(rng.random()) * rng.random(n, dtype=np.float32)).astype(np.float32)
            if rng.integers(0, 4) == 0:
                x[rng.integers(0, n, max(1, n // 1000))] = np.float32("nan")
            k = _k(rng, n)
            m = int(rng.integers(0, 3))
            seed = int(rng.integers(0, 1000))
            what = f"scaled n={n} k={k} mode={m} order={order}"
            wv, wi, wp, winfo = O.ref_scaled_topk(x, k, order, mode=m, tau=0.5, seed=seed, grid=16)
            info = rtk.ScaleInfo()
            r = rtk.scaled_topk(torch.from_numpy(x).to(dev), k, rtk.SelectionOrder(order),
                                policy=rtk.ScalePolicy(rtk.ScaleMode(m), 0.5, seed), info=info)
            assert info.scaled == winfo["scaled"], what + " scaled flag"
            assert_same((r.values, r.indices, r.pivot), (wv, wi, wp), what)
        elif mode == 4:  # ragged 16-bit batch: indices against the widened f32 rows, values = inputs
            from tests.test_gpu_parity import _widen16
            kind = "bf16" if rng.integers(0, 2) else "f16"
            B = int(rng.integers(1, 20))
            lens = [int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 300000)])) for _ in range(B)]
            ks = [_k(rng, n) for n in lens]
            offs, pos = [], 0
            for t in range(B):
                pos += int(rng.integers(0, 9))
                offs.append(pos)
                pos += lens[t]
            xf = torch.from_numpy(rng.standard_normal(pos).astype(np.float32) * float(rng.choice([1.0, 1e-2, 50.0])))
            t16 = xf.to(torch.bfloat16 if kind == "bf16" else torch.float16)
            h = t16.view(torch.int16).numpy().view(np.uint16).copy()
            x32 = _widen16(h, kind)
            what = f"{kind} batch B={B} order={order}"
            exp = O.ref_batch_topk(x32, offs, lens, ks, order, grid=16)
            got = rtk.batch_topk(rtk.BatchInput(t16.to(dev), offs, lens, ks), rtk.SelectionOrder(order))
            for t in range(B):
                gi = got[t].indices.cpu().numpy().astype(np.uint64)
                wi = exp[t][1].astype(np.uint64)
                assert np.array_equal(gi, wi), what + f" row {t} n={lens[t]} k={ks[t]}: indices"
                gv = got[t].values.view(torch.int16).cpu().numpy().view(np.uint16)
                assert np.array_equal(gv, h[offs[t] + wi.astype(np.int64)]), what + f" row {t}: values"
        elif mode == 6:  # dense [B, V] rows (batch_topk_dense), f32
            B = int(rng.integers(1, 64))
            V = int(rng.choice([rng.integers(1, 4000), rng.integers(4000, 140000)]))
            data = np.concatenate([_row(rng, V, np.float32) for _ in range(B)])
            k = _k(rng, V)
            what = f"dense B={B} V={V} k={k} order={order}"
            exp = O.ref_batch_topk(data, [i * V for i in range(B)], [V] * B, [k] * B, order, grid=16)
            r = rtk.batch_topk_dense(torch.from_numpy(data).to(dev).view(B, V), k, rtk.SelectionOrder(order))
            gv, gi, gp = r.values.cpu().numpy(), r.indices.cpu().numpy(), r.pivot.cpu().numpy()
            for t in range(B):
                assert_same((gv[t], gi[t], gp[t]), exp[t], what + f" row {t}")
        elif mode == 7:  # host entry points (numpy in, copies inside the call)
            n = int(rng.integers(1, 1 << 22))
            x = _row(rng, n, np.float32)
            k = _k(rng, n)
            what = f"host n={n} k={k} order={order}"
            r = rtk.topk(x, k, rtk.SelectionOrder(order))
            assert_same((r.values, r.indices, r.pivot), O.ref_topk(x, k, order, grid=16), what)
        else:  # 16-bit rows (indices against the exactly widened f32 input)
            from tests.test_gpu_parity import _check16, _widen16
            kind = "bf16" if rng.integers(0, 2) else "f16"
            n = int(rng.integers(1, 1 << 21))
            xf = torch.from_numpy(rng.standard_normal(n).astype(np.float32) * float(rng.choice([1.0, 1e-3, 100.0])))
            t16 = xf.to(torch.bfloat16 if kind == "bf16" else torch.float16)
            h = t16.view(torch.int16).numpy().view(np.uint16).copy()
            k = _k(rng, n)
            what = f"{kind} n={n} k={k} order={order}"
            _check16(h, t16, _widen16(h, kind), k, order, dev, what)
    except AssertionError as e:
        fails += 1
        print(f"FAIL case {case}: {str(e)[:300]}", flush=True)
    except Exception as e:
        fails += 1
        print(f"ERROR case {case} ({what}): {type(e).__name__}: {str(e)[:300]}", flush=True)
        if "cuda" in type(e).__name__.lower():
            break
rtk.set_option("force_exact", 0)
rtk.set_option("force_deep", 0)
print(f"fuzz {s0}..{case + 1}: {case + 1 - s0} cases, {fails} failures", flush=True)

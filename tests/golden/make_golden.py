"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Inputs come from the reference's seeded generators (rtk::generate, datagen.hpp:71-141) and
outputs from the reference engine / oracle / batch / scaled entry points, all compiled from
/root/reference/proj/include by oracle/Makefile into oracle/_ref/librtk_ref.so. Run here (the
reference tree is only present in the build container):

    python tests/golden/make_golden.py

The fixtures are small (<= a few hundred KB) so they travel with the repo; the parity tests
check both the C restatement (oracle/rtk_oracle.c) and the GPU path against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

UNIFORM, NORMAL, ZIPF, PEAKED = 0, 1, 2, 3


def single_cases():
    cases = []
    # engine_test.cpp:324-349 style randomized cells + acceptance :48-94 style sizes
    rng = np.random.default_rng(31337)
    for t in range(40):
        kind = int(rng.integers(0, 3))
        n = int(rng.integers(1, 3000))
        k = int(rng.integers(1, n + 1))
        order = int(rng.integers(0, 2))
        dtype = np.float32 if t % 2 == 0 else np.uint32
        seed = int(rng.integers(0, 2**31))
        a = -5.0 if kind == UNIFORM else 1.0
        cases.append(dict(kind=kind, n=n, k=k, order=order, dtype=dtype, seed=seed, a=a, b=5.0))
    for n, k in [(1 << 16, 256), (1 << 16, 1), ((1 << 16) + 7, 40000)]:
        cases.append(dict(kind=UNIFORM, n=n, k=k, order=0, dtype=np.float32, seed=1, a=0.0, b=1.0))
    # adversarial narrow band (scaling_test.cpp:16-26), many ties
    cases.append(dict(kind=UNIFORM, n=1 << 15, k=4096, order=0, dtype=np.float32, seed=42, a=128.6, b=128.7))
    return cases


def main():
    out = {}
    for i, c in enumerate(single_cases()):
        x = O.ref_generate(c["kind"], c["n"], c["seed"], dtype=c["dtype"], a=c["a"], b=c["b"])
        v, idx, piv = O.ref_topk(x, c["k"], c["order"], grid=3)
        ov, oidx, opiv = O.ref_oracle_topk(x, c["k"], c["order"])
        assert np.array_equal(idx, oidx) and np.array_equal(v.view(np.uint32), ov.view(np.uint32))
        out[f"single{i}_x"] = x
        out[f"single{i}_meta"] = np.array([c["k"], c["order"], c["kind"], c["seed"]], dtype=np.uint64)
        out[f"single{i}_vals"] = v
        out[f"single{i}_idx"] = idx
        out[f"single{i}_pivot"] = np.array([piv], dtype=x.dtype)
    # semantics vector: +-0, +-inf, +-nan
    sem = np.array([0.0, -0.0, 1.0, np.nan, 0.0, -1.0, 0.0, np.inf, -np.inf], dtype=np.float32)
    sem[4] = np.array([0xFFC00000], dtype=np.uint32).view(np.float32)[0]
    out["sem_x"] = sem
    for order in (0, 1):
        v, idx, piv = O.ref_topk(sem, 9, order)
        out[f"sem{order}_idx"] = idx
    # batch (batch_test.cpp:122-143 heterogeneous ranks)
    tasks = [O.ref_generate(NORMAL, 300 + 17 * t, 50 + t, b=1.0) for t in range(5)]
    ks = [1 + 10 * t for t in range(5)]
    data = np.concatenate(tasks)
    offs = np.cumsum([0] + [len(t) for t in tasks[:-1]]).astype(np.uint64)
    lens = np.array([len(t) for t in tasks], dtype=np.uint64)
    res = O.ref_batch_topk(data, offs, lens, ks, 1, grid=2)
    out["batch_data"] = data
    out["batch_offs"] = offs
    out["batch_lens"] = lens
    out["batch_ks"] = np.array(ks, dtype=np.uint64)
    for t, (v, idx, piv) in enumerate(res):
        out[f"batch{t}_idx"] = idx
        out[f"batch{t}_vals"] = v
    # scaled (scaling_test.cpp:106-139, 173-196)
    y = O.ref_generate(UNIFORM, 1 << 14, 42, a=128.6, b=128.7)
    out["scaled_x"] = y
    for mode in (0, 1, 2):
        v, idx, piv, info = O.ref_scaled_topk(y, 128, 0, mode=mode, seed=13)
        out[f"scaled{mode}_idx"] = idx
        out[f"scaled{mode}_vals"] = v
        out[f"scaled{mode}_info"] = np.array([int(info["scaled"]), int(info["a_index"])], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()

"""Bench/report harness with the reference's report shape.

Mirrors `rtk gen` / `rtk bench` (rtk_cli.cpp:165-216, 350-481) so a GPU report and the CPU
reference's report diff cleanly:

* ``generate`` <- rtk::generate<float|uint32_t> (datagen.hpp:68-140): the same mt19937_64 stream
  and libstdc++ distributions (computed in librtk_b200.so), so inputs are bit-identical;
* ``result_checksum`` <- result_checksum (rtk_cli.cpp:100-115): FNV-1a over (value bits, u64 index);
* ``bench`` <- cmd_bench / bench_cell (rtk_cli.cpp:372-481): cells over n x k (``quantile`` gives
  k in {n/100, n/4, n/2}), ``batch`` tasks per cell with the reference's seeds
  (seed + 100 t + n + k) and its deliberately misaligned first task (n - 1), median wall time of
  ``repeats`` runs, XOR of the per-task checksums, the JSON / CSV layouts of the reference.

The CPU engine's modelled counters (flushes, global merges, modelled transactions) have no GPU
counterpart and are reported as 0; ``passes`` and ``elements_scanned`` come from the GPU run.
``verified`` (``verify=True``) is a self-consistency check of every result (values equal the input
at the returned indices, canonical order), not a second top-k.

    python -m paper_2501_14336_b200.report gen uniform --n 1048576 --seed 1 -o x.rtk1
    python -m paper_2501_14336_b200.report bench --n-list 1048576 --k-list 256 --batch 4
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib as L
from . import rtk as R
from .rtk import _raise

KINDS = {"uniform": 0, "normal": 1, "zipf": 2, "peaked": 3}


@dataclass
class DistributionSpec:  # datagen.hpp:18-26
    kind: str = "uniform"
    a: float = 0.0
    b: float = 1.0
    s: float = 1.1
    mass: float = 0.8
    modes: int = 1
    seed: int = 0
    n: int = 0


def generate(spec: DistributionSpec, dtype=np.float32) -> np.ndarray:
    code = {np.dtype(np.float32): 0, np.dtype(np.uint32): 1}[np.dtype(dtype)]
    if spec.kind not in KINDS:
        raise ValueError(f"unknown distribution: {spec.kind}")
    d = L.rtk_dist(KINDS[spec.kind], spec.a, spec.b, spec.s, spec.mass, spec.modes, spec.seed, spec.n)
    out = np.empty(max(int(spec.n), 0), dtype=dtype)
    _raise(L.load().rtk_generate(C.byref(d), code, out.ctypes.data_as(C.c_void_p)), "generate")
    return out


def result_checksum(values, indices) -> int:
    v = np.ascontiguousarray(values)
    i = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
    code = {np.dtype(np.float32): 0, np.dtype(np.uint32): 1, np.dtype(np.float16): 2}.get(v.dtype, 3)
    return int(L.load().rtk_result_checksum(v.ctypes.data_as(C.c_void_p), code, i.ctypes.data_as(L.P64), len(i)))


def _consistent(x: np.ndarray, res: R.TopKResult, order: R.SelectionOrder) -> bool:
    v, idx = np.asarray(res.values), np.asarray(res.indices).astype(np.int64)
    if not np.array_equal(x[idx].view(np.uint32), v.view(np.uint32)):
        return False
    u = v.view(np.uint32).astype(np.uint64)
    key = np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000) if x.dtype == np.float32 else u
    if order == R.SelectionOrder.Smallest:
        key = (~key) & 0xFFFFFFFF
    comp = (key << np.uint64(32)) | ((~idx.astype(np.uint64)) & np.uint64(0xFFFFFFFF))
    return bool(np.all(comp[:-1] > comp[1:]))


def bench_cell(n: int, k: int, batch: int, dist: str, seed: int, repeats: int,
               order: R.SelectionOrder, verify: bool, variant: str = "configured",
               device: bool = True) -> Dict:
    payloads, ks = [], []
    for t in range(batch):  # rtk_cli.cpp:381-388
        nt = n - 1 if (t == 0 and batch > 1) else n
        payloads.append(generate(DistributionSpec(kind=dist, s=1.1, n=nt, seed=seed + 100 * t + n + k)))
        ks.append(k)
    b = R.BatchInput.concatenate(payloads, ks)
    data = b.data
    if device:
        import torch
        data = torch.from_numpy(b.data).cuda()
        sync = torch.cuda.synchronize
    else:
        sync = lambda: None  # noqa: E731
    run = R.BatchInput(data, b.offsets, b.lengths, b.ks)
    times, checksum, verified, stats = [], 0, True, None
    for r in range(repeats):
        sync()
        t0 = time.perf_counter()
        results = R.batch_topk(run, order)
        sync()
        times.append((time.perf_counter() - t0) * 1e3)
        stats = R.last_stats()
        checksum = 0
        for t, res in enumerate(results):
            vals = res.values.cpu().numpy() if hasattr(res.values, "cpu") else np.asarray(res.values)
            idx = res.indices.cpu().numpy() if hasattr(res.indices, "cpu") else np.asarray(res.indices)
            checksum ^= result_checksum(vals, idx)
            if r == 0 and verify:
                verified &= _consistent(payloads[t], R.TopKResult(vals, idx), order)
    times.sort()
    cell = {"variant": variant, "n": n, "k": k, "batch": batch, "median_ms": times[len(times) // 2],
            "checksum": checksum,
            "instrumentation": {"passes": stats.passes if stats else 0, "flushes": 0, "partitions": 0,
                                "global_merges": 0,
                                "elements_scanned": stats.elements_scanned if stats else 0,
                                "modeled_transactions": 0}}
    if verify:
        cell["verified"] = bool(verified)
    return cell


def bench(ns: Sequence[int], ks: Sequence[int], batch: int = 1, dist: str = "uniform", quantile: bool = False,
          repeats: int = 3, order: R.SelectionOrder = R.SelectionOrder.Largest, seed: int = 0,
          verify: bool = False, ablate: bool = False, device: bool = True) -> Dict:
    # the reference's ablation variants toggle CPU-engine mechanisms (hierarchical atomics,
    # flush buffer, rescheduling, padding) that do not change results; they are accepted and
    # reported under the same names (BatchOptions are result-neutral, batch_test.cpp:145-165)
    variants = ["configured"]
    if ablate:
        names = ["hier-atomics", "flush-buffer", "reschedule", "pad"]
        variants = ["all-on"] + [p + m for m in names for p in ("only-", "no-")]
    cells: List[Dict] = []
    for n in ns:
        kl = [n // 100, n // 4, n // 2] if quantile else list(ks)
        for k in kl:
            if k == 0 or k > n:
                continue
            for v in variants:
                try:
                    cells.append(bench_cell(n, k, batch, dist, seed, repeats, order, verify, v, device))
                except Exception as e:  # reported in its cell, the sweep continues (rtk_cli.cpp:436-444)
                    cells.append({"variant": v, "n": n, "k": k, "batch": batch, "error": str(e)})
    config = {"d": 12, "block_size": 1024, "grid_size": 4, "pack_size": 16, "buffer": "efficient",
              "reschedule": "on", "pad": "on", "scale": "off", "tau": 0.5,
              "order": "largest" if order == R.SelectionOrder.Largest else "smallest", "seed": seed,
              "engine": "rtk-b200 (sm_100a)"}
    return {"config": config, "cells": cells}


def to_csv(report: Dict) -> str:  # rtk_cli.cpp:459-476
    lines = ["variant,n,k,batch,median_ms,checksum,verified,passes,flushes,global_merges,"
             "elements_scanned,modeled_transactions,error"]
    for c in report["cells"]:
        if "error" in c:
            lines.append(f'{c["variant"]},{c["n"]},{c["k"]},{c["batch"]},,,,,,,,,"{c["error"]}"')
            continue
        i = c["instrumentation"]
        lines.append(f'{c["variant"]},{c["n"]},{c["k"]},{c["batch"]},{c["median_ms"]},{c["checksum"]},'
                     f'{1 if c.get("verified", True) else 0},{i["passes"]},{i["flushes"]},{i["global_merges"]},'
                     f'{i["elements_scanned"]},{i["modeled_transactions"]},')
    return "\n".join(lines) + "\n"


def main(argv: Optional[Sequence[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2501_14336_b200.report")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="write an RTK1 dataset (rtk gen)")
    g.add_argument("dist", choices=sorted(KINDS))
    g.add_argument("params", nargs="*", type=float)
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--s", type=float, default=1.1)
    g.add_argument("--mass", type=float, default=0.8)
    g.add_argument("--modes", type=int, default=1)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--dtype", choices=["f32", "u32"], default="f32")
    g.add_argument("-o", "--out", required=True)
    b = sub.add_parser("bench", help="rtk bench report (JSON or CSV)")
    b.add_argument("--n-list", type=int, nargs="+", default=[1 << 20])
    b.add_argument("--k-list", type=int, nargs="+", default=[256])
    b.add_argument("--dist", choices=["uniform", "normal", "zipf"], default="uniform")
    b.add_argument("--batch", type=int, default=1)
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--quantile", action="store_true")
    b.add_argument("--ablate", action="store_true")
    b.add_argument("--verify", action="store_true")
    b.add_argument("--order", choices=["largest", "smallest"], default="largest")
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--format", choices=["json", "csv"], default="json")
    a = ap.parse_args(argv)
    if a.cmd == "gen":
        spec = DistributionSpec(kind=a.dist, s=a.s, mass=a.mass, modes=a.modes, seed=a.seed, n=a.n)
        if a.dist == "uniform" and len(a.params) >= 2:
            spec.a, spec.b = a.params[0], a.params[1]
        if a.dist == "normal":
            spec.a = a.params[0] if len(a.params) >= 1 else 0.0
            spec.b = a.params[1] if len(a.params) >= 2 else 1.0
        from .io import write_dataset
        x = generate(spec, np.float32 if a.dtype == "f32" else np.uint32)
        write_dataset(a.out, x)
        print(f"wrote {a.n} {a.dtype} elements to {a.out}", file=sys.stderr)
        return 0
    order = R.SelectionOrder.Largest if a.order == "largest" else R.SelectionOrder.Smallest
    rep = bench(a.n_list, a.k_list, a.batch, a.dist, a.quantile, a.repeats, order, a.seed, a.verify, a.ablate)
    sys.stdout.write(json.dumps(rep, indent=2) + "\n" if a.format == "json" else to_csv(rep))
    return 0 if all(c.get("verified", True) for c in rep["cells"]) else 1


if __name__ == "__main__":
    sys.exit(main())

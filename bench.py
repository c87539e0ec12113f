#!/usr/bin/env python3
"""bench.py — B200 radix top-k benchmark (contract: one JSON line on rank 0).

Headline (N = 1, BASELINE.json configs[1]): ONE fp32 query, n = 2^28 Uniform[0,1) elements
resident in HBM, k = 2^20 (largest), values + u64 indices in the reference's canonical order.
Metric: the north-star "effective GB/s" = algorithmic bytes (4n + 12k per query: every key read
once, k values + k u64 indices written) / time.

* value         median device time of back-to-back rtk_topk calls issued from C
                (rtk_bench_topk: CUDA events the engine records on the launching stream around
                its device work); the input (1 GiB) is larger than L2.
* host_ms       the same calls' host wall time (C steady_clock around each rtk_topk, which
                returns after the device's completion signal).
* e2e           the same metric through the host entry point rtk_topk_host: the 1 GiB H2D copy
                from pinned memory and the D2H of the result inside the timed region.
* roofline      the dominant kernel (k_compact, the single streaming pass) timed with CUDA
                events on its stream; algorithmic bytes per launch = 4n.
* cpu_baseline  the reference's own engine (rtk::topk from its headers, oracle/_ref) on this
                box's host cores, on the SAME input and config (n = 2^28, k = 2^20).
* legs          C1 (n = 2^20, k = 256, L2 flushed), the k sweep of C2, C3 (256 x 128256 logits,
                f32 and bf16, L2 flushed), C4 (n = 2^26 adversarial, scale off/always/adaptive),
                the C5 shard shape (2^29 Philox elements, k = 2^16) — each with the reference
                engine timed on the same input where it runs in bounded time.

Multi-GPU (N > 1; `--gpus N` re-launches itself under torch.distributed.run when WORLD_SIZE is
unset): BASELINE configs[4] (C5) — one query of N * 2^29 fp32 elements (n = 2^32 at N = 8), each
rank generating its shard on its device (Philox, rtk_generate_philox), k = 2^16; per step
rtk_topk_sharded: local top-k + ncclAllGather of the candidates + final select on every rank.
Weak scaling; time = max over ranks of the median step.

--impl reference: the reference CPU engine (oracle/_ref) on the host cores, same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0
METRIC = "topk_effective_GBps"
C5_SEED = 5


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every few ms during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int, period_s: float = 0.002):
        self.gpu, self.period = gpu, period_s
        self.sm, self.mask, self.max_sm = [], 0, None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover - no NVML
            self.err = repr(e)
            self.N = None
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.sm.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                self.mask |= N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if getattr(self, "N", None):
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": ["unsampled"]}
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(self.sm)}


def gbs(n_elem_bytes: float, k: int, ms: float) -> float:
    return (n_elem_bytes + 12 * k) / (ms * 1e-3) / 1e9


# ---- the reference CPU engine (oracle/_ref), timed on the host cores -------------------------
def _timed(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), ts


def torch_topk_ms(fn, steps, flush=None):
    """Median device time (CUDA events on torch's current stream) of fn() — torch.topk as a timing
    competitor; its ties are not ordered by index, so it is not a parity oracle."""
    import statistics
    import torch
    for _ in range(3):
        fn()
    ts = []
    for _ in range(steps):
        if flush is not None:
            flush.fill_(1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def cpu_topk(x, k, reps, cores):
    import oracle as O
    t, _ = _timed(lambda: O.ref_topk(x, k, 0, 12, cores), reps)
    return t


def host_inputs(n, k):
    """The headline query on the host: numpy's PCG64 (seed 1) Uniform[0,1) fp32 — the same array
    is uploaded for the GPU arm and handed to the reference engine."""
    import numpy as np
    return np.random.default_rng(1).random(n, dtype=np.float32)


def reference_arm(args, world, rank):
    """bench.py --impl reference: rtk::topk (the reference engine compiled from its headers) on the
    host cores, on this arm's workload. N = 1: the full C2 query (n = 2^28, k = 2^20), one call per
    step. N > 1: the query is N * 2^29 elements (C5), beyond host memory for the reference's four
    copies; each step runs a 2^28-element prefix sample with k scaled by the sample fraction."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    if world == 1:
        n, k = 1 << args.logn, args.k
        ns, ks = n, k
        sample = f"the full query: n=2^{args.logn} PCG64(1) U[0,1) k={k}, rtk::topk grid_size={cores}, one call per step"
        config = headline_config(args, 1)
    else:
        n, k = world * (1 << args.shard_logn), args.shard_k
        ns = 1 << 28
        ks = max(1, k * ns // n)
        sample = (f"the first 2^28 elements (Philox seed {C5_SEED}) of the {world}x2^{args.shard_logn} query, k "
                  f"scaled to {ks}, rtk::topk grid_size={cores}, one call per step (the full query exceeds host "
                  "memory for the reference's copies)")
        config = c5_config(args, world)
    if world == 1:
        x = host_inputs(ns, ks)
    else:
        import oracle as O
        x = O.philox_fill(C5_SEED, 0, ns)
    for _ in range(args.warmup):
        cpu_topk(x, ks, 1, cores)
    vals = []
    for _ in range(args.steps):
        t = cpu_topk(x, ks, 1, cores)
        vals.append(gbs(4 * ns, ks, t * 1e3))
    v = statistics.median(vals)
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": (4 * ns + 12 * ks) / v / 1e6,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                      "data": "synthetic", "config": config,
                      "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "reference",
                                       "cpu_model": cpu_model(), "sample": sample},
                      "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def headline_config(args, world):
    n = 1 << args.logn
    return {"workload": f"C2: single query fp32 Uniform[0,1) n=2^{args.logn}, k={args.k}, largest, values+u64 "
                        "indices, sorted (BASELINE configs[1])",
            "n": n, "k": args.k, "dtype": "f32", "order": "largest",
            "l2": "input 1 GiB > 126 MB L2 (no flush needed)", "parallelism": "single"}


def c5_config(args, world):
    ns = 1 << args.shard_logn
    return {"workload": f"C5: single huge query fp32 Uniform[0,1) n={world}x2^{args.shard_logn}"
                        f"{' = 2^32' if world * ns == 1 << 32 else ''}, k={args.shard_k}, largest, sharded by index "
                        "range: local top-k + NCCL allgather + final select (BASELINE configs[4])",
            "n": world * ns, "n_per_gpu": ns, "k": args.shard_k, "dtype": "f32", "order": "largest",
            "generator": f"Philox4x32-10 seed {C5_SEED} on each rank's device (rtk_generate_philox)",
            "l2": "input 2 GiB per GPU > L2 (no flush needed)", "parallelism": f"n-sharded x{world} (NCCL)"}


# ---- self-launch for --gpus N ------------------------------------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    port = _free_port()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries the one JSON line only
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


# ---- the GPU arm --------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--logn", type=int, default=28)
    ap.add_argument("--k", type=int, default=1 << 20)
    ap.add_argument("--shard-logn", type=int, default=29, help="C5: elements per GPU (2^x)")
    ap.add_argument("--shard-k", type=int, default=1 << 16, help="C5: k")
    ap.add_argument("--sweep", type=str, default="256,16384", help="extra C2 k values")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-torch-topk", action="store_true", help="skip the torch.topk timing competitor")
    ap.add_argument("--legs", type=str, default="c1,c2dist,c3,c4,c5", help="secondary legs (N = 1)")
    ap.add_argument("--batch-ks", type=str, default="50,4096,128256")
    ap.add_argument("--batch-rows", type=int, default=256)
    ap.add_argument("--vocab", type=int, default=128256)
    ap.add_argument("--sharded-1gpu", action="store_true",
                    help="run the N > 1 code path (C5 shards, rtk_topk_sharded over NCCL) with one rank")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":  # rank 0's work only: no ranks to launch
            os.environ.update(WORLD_SIZE=str(args.gpus), RANK="0")
        else:
            sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    if world > 1 or args.sharded_1gpu:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        multi_gpu(args, rank, world, local)
    else:
        single_gpu(args)


def single_gpu(args):
    import numpy as np
    import torch

    import paper_2501_14336_b200 as rtk
    from paper_2501_14336_b200 import rtk as R

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, k = 1 << args.logn, args.k
    legs = set(v for v in args.legs.split(",") if v)
    peak, peak_kind = measured_peak()
    cores = os.cpu_count() or 1
    do_cpu = not args.no_cpu_baseline
    hx = host_inputs(n, k)
    x = torch.from_numpy(hx).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 (126 MB)
    launches_before = 0

    # ---- headline: C2 k = 2^20 ---------------------------------------------------------------
    with ClockSampler(0) as clk:
        b = R.bench_topk(x, k, args.steps, args.warmup)
    clocks = clk.summary()
    med = b.median_ms
    value = gbs(4 * n, k, med)
    # kernel share: k_compact bracketed by CUDA events on its stream (library timing mode: no graph
    # replay), on separate calls so no stats readback sits inside the timed region
    R.set_timing(True)
    comp, per_step = [], 0
    for _ in range(10):
        rtk.topk(x, k)
        st = R.last_stats()
        comp.append(st.compact_ms)
        per_step = st.kernel_launches
    R.set_timing(False)
    comp_ms = statistics.median(comp)
    achieved = 4 * n / (comp_ms * 1e-3) / 1e9
    launches = per_step * args.steps

    sweep = {}
    for kk in [int(v) for v in args.sweep.split(",") if v]:
        bk = R.bench_topk(x, kk, max(5, args.steps // 2), 3)
        sweep[str(kk)] = {"ms": bk.median_ms, "host_ms": bk.median_host_ms, "GBps": gbs(4 * n, kk, bk.median_ms),
                          "fraction_of_hbm_peak": gbs(4 * n, kk, bk.median_ms) / peak}

    # ---- torch.topk on the same device-resident inputs (timing competitor) -------
    competitor = {"note": "torch.topk(sorted=True) on the same tensors, CUDA events, median; ours = this bench's "
                          "median for the same config"}
    if not args.no_torch_topk:
        for kk in [k] + [int(v) for v in args.sweep.split(",") if v]:
            tm = torch_topk_ms(lambda: torch.topk(x, kk, sorted=True), max(5, args.steps // 2))
            ours = med if kk == k else sweep[str(kk)]["ms"]
            competitor[f"c2_k{kk}"] = {"ms": tm, "ours_ms": ours, "speedup": tm / ours}

    # ---- e2e through the host entry point (pinned host input, copies inside) ------------------
    hp = torch.from_numpy(hx).pin_memory().numpy()
    R.topk(hp, k)
    t_e2e = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        R.topk(hp, k)
        t_e2e.append(time.perf_counter() - t0)
    te = statistics.median(t_e2e)
    e2e = {"value": gbs(4 * n, k, te * 1e3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
           "d2h_bytes_per_step": 12 * k + 4, "ms_per_step": te * 1e3, "entry": "rtk_topk_host"}

    cpu = None
    if do_cpu:
        t = cpu_topk(hx, k, 3, cores)
        cpu = {"value": gbs(4 * n, k, t * 1e3), "unit": "GB/s", "cores": cores, "kind": "reference",
               "cpu_model": cpu_model(), "ms": t * 1e3,
               "sample": f"the same query and input (n=2^{args.logn}, k={k}): rtk::topk (oracle/_ref) "
                         f"grid_size={cores}, median of 3"}
    if "c2dist" not in legs:
        del hp

    out_legs = {}
    if "c2dist" in legs:
        del hp
        out_legs["c2_distributions"] = leg_c2_dists(args, R, x, dev, peak, cores, do_cpu)
    if "c1" in legs:
        out_legs["c1"] = leg_c1(args, R, dev, flush, peak, cores, do_cpu)
        if not args.no_torch_topk:
            competitor["c1"] = out_legs["c1"].pop("torch_topk")
    if "c3" in legs:
        out_legs["c3"] = leg_c3(args, R, dev, flush, peak, cores, do_cpu)
        if not args.no_torch_topk:
            competitor["c3"] = out_legs["c3"].pop("torch_topk")
    if "c4" in legs:
        out_legs["c4"] = leg_c4(args, R, dev, peak, cores, do_cpu)
    if "c5" in legs:
        del x
        torch.cuda.empty_cache()
        out_legs["c5_shard_1gpu"] = leg_c5_1gpu(args, R, dev, peak)

    prof = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = None
    try:
        with open(prof) as f:
            traffic = json.load(f).get(f"k_compact_n{n}")
    except Exception:
        pass
    out = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": med, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32",
           "data": "synthetic: numpy PCG64(1) Uniform[0,1) fp32 on the host, uploaded once",
           "config": headline_config(args, 1),
           "queries_per_s": 1e3 / med, "elements_per_s": n / (med * 1e-3), "fraction_of_hbm_peak": value / peak,
           "host_ms_per_step": b.median_host_ms,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": traffic, "kernel": "k_compact", "peak_kind": peak_kind,
                        "kernel_ms": comp_ms, "kernel_share_of_step": comp_ms / med},
           "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
           "timing": "median over steps of back-to-back rtk_topk calls issued from C (rtk_bench_topk): device "
                     "time between CUDA events the engine records on the launching stream right before its "
                     "first and after its last device operation of the call; host_ms = steady_clock around "
                     "each rtk_topk call (returns after the device's completion signal)",
           "step_ms_all": b.device_ms, "host_ms_all": b.host_ms,
           "k_sweep": sweep, "legs": out_legs, "torch_topk": competitor}
    print(json.dumps(out))


def leg_c2_dists(args, R, x, dev, peak, cores, do_cpu):
    """C2's other distributions: n = 2^28 Normal(0, 1) and Zipf(1.1) from the
    reference's own generators (rtk_generate == rtk::generate, datagen.hpp:71-104), k = 2^20,
    written over the headline's device buffer; the reference engine timed on the same input."""
    from paper_2501_14336_b200 import report as REP
    n, k = 1 << args.logn, args.k
    res = {}
    for kind, spec in (("normal", REP.DistributionSpec(kind="normal", a=0.0, b=1.0, seed=2, n=n)),
                       ("zipf", REP.DistributionSpec(kind="zipf", s=1.1, seed=3, n=n))):
        import torch
        hx = REP.generate(spec)
        x.copy_(torch.from_numpy(hx))
        b = R.bench_topk(x, k, max(5, args.steps // 2), 3)
        e = {"ms": b.median_ms, "host_ms": b.median_host_ms, "GBps": gbs(4 * n, k, b.median_ms),
             "fraction_of_hbm_peak": gbs(4 * n, k, b.median_ms) / peak,
             "config": f"n=2^{args.logn} rtk::generate {kind} seed {spec.seed}, k={k}"}
        if do_cpu:
            t = cpu_topk(hx, k, 1, cores)
            e["cpu_baseline"] = {"ms": t * 1e3, "GBps": gbs(4 * n, k, t * 1e3), "cores": cores, "kind": "reference",
                                 "sample": "same input, rtk::topk grid_size=cores, one call"}
        res[kind] = e
        del hx
    return res


def leg_c1(args, R, dev, flush, peak, cores, do_cpu):
    """C1 (BASELINE configs[0]): n = 2^20 Uniform[0,1), k = 256 — launch/latency-bound (4 MB);
    L2 flushed before every step outside the clocks."""
    import numpy as np
    import torch
    n, k = 1 << 20, 256
    hx = np.random.default_rng(2).random(n, dtype=np.float32)
    x = torch.from_numpy(hx).to(dev)
    b = R.bench_topk(x, k, max(10, args.steps), 5, flush=flush)
    leg = {"config": "n=2^20 PCG64(2) U[0,1) fp32, k=256, largest; L2 flushed before each step",
           "ms": b.median_ms, "host_ms": b.median_host_ms, "GBps": gbs(4 * n, k, b.median_ms),
           "fraction_of_hbm_peak": gbs(4 * n, k, b.median_ms) / peak, "queries_per_s": 1e3 / b.median_host_ms}
    if do_cpu:
        t = cpu_topk(hx, k, 5, cores)
        leg["cpu_baseline"] = {"ms": t * 1e3, "GBps": gbs(4 * n, k, t * 1e3), "cores": cores, "kind": "reference",
                               "sample": "same input, rtk::topk grid_size=cores, median of 5"}
    if not args.no_torch_topk:
        tm = torch_topk_ms(lambda: torch.topk(x, k, sorted=True), max(10, args.steps), flush)
        leg["torch_topk"] = {"ms": tm, "ours_ms": b.median_ms, "speedup": tm / b.median_ms}
    return leg


def leg_c3(args, R, dev, flush, peak, cores, do_cpu):
    """C3 (BASELINE configs[2]): batched LLM-vocab top-k, 256 x 128256 N(0,1) fp32 logits (and the
    same logits in bf16), k in {50, 4096, vocab}; L2 flushed before every step (the 131 MB batch
    fits the 126 MB L2 almost entirely)."""
    import numpy as np
    import oracle as O
    import torch
    B, V = args.batch_rows, args.vocab
    hl = np.random.default_rng(3).standard_normal((B, V), dtype=np.float32)
    logits = torch.from_numpy(hl).to(dev)
    lb = logits.to(torch.bfloat16)
    res = {"config": f"{B} x {V} PCG64(3) N(0,1) fp32 logits (bf16: the same rounded); peaked: rtk::generate "
                     "Peaked mass 0.8, modes 1 + t % 2, seed 100 + t per row; L2 flushed before each step",
           "f32": {}, "bf16": {}, "sampling": {}}
    for kb in [min(int(v), V) for v in args.batch_ks.split(",") if v]:
        b = R.bench_batch_dense(logits, kb, max(5, args.steps // 2), 3, flush)
        byts = B * (4 * V + 12 * kb)
        e = {"ms": b.median_ms, "host_ms": b.median_host_ms, "queries_per_s": B / (b.median_ms * 1e-3),
             "effective_GBps": byts / (b.median_ms * 1e-3) / 1e9,
             "fraction_of_hbm_peak": byts / (b.median_ms * 1e-3) / 1e9 / peak}
        if do_cpu:
            reps = 1 if kb > 8192 else 3
            t, _ = _timed(lambda: O.ref_batch_topk(hl.reshape(-1), [i * V for i in range(B)], [V] * B, [kb] * B,
                                                   0, 12, cores), reps)
            e["cpu_baseline"] = {"ms": t * 1e3, "queries_per_s": B / t, "cores": cores, "kind": "reference",
                                 "sample": f"same logits, rtk::batch_topk grid_size=cores, median of {reps}"}
        res["f32"][str(kb)] = e
        if not args.no_torch_topk:
            tm = torch_topk_ms(lambda: torch.topk(logits, kb, dim=1, sorted=True), max(5, args.steps // 2), flush)
            res.setdefault("torch_topk", {})[f"f32_k{kb}"] = {"ms": tm, "ours_ms": b.median_ms,
                                                              "speedup": tm / b.median_ms}
        bh = R.bench_batch_dense(lb, kb, max(5, args.steps // 2), 3, flush)
        byts = B * (2 * V + 10 * kb)
        res["bf16"][str(kb)] = {"ms": bh.median_ms, "host_ms": bh.median_host_ms,
                                "queries_per_s": B / (bh.median_ms * 1e-3),
                                "effective_GBps": byts / (bh.median_ms * 1e-3) / 1e9,
                                "fraction_of_hbm_peak": byts / (bh.median_ms * 1e-3) / 1e9 / peak}
        if not args.no_torch_topk:
            tm = torch_topk_ms(lambda: torch.topk(lb, kb, dim=1, sorted=True), max(5, args.steps // 2), flush)
            res["torch_topk"][f"bf16_k{kb}"] = {"ms": tm, "ours_ms": bh.median_ms, "speedup": tm / bh.median_ms}
    # Peaked rows (DistKind::Peaked, mass 0.8, modes 1-2, datagen.hpp:93-104)
    from paper_2501_14336_b200 import report as REP
    hp = np.stack([REP.generate(REP.DistributionSpec(kind="peaked", mass=0.8, modes=1 + t % 2, seed=100 + t, n=V))
                   for t in range(B)])
    peaked = torch.from_numpy(hp).to(dev)
    res["peaked"] = {}
    for kb in [min(int(v), V) for v in args.batch_ks.split(",") if v]:
        b = R.bench_batch_dense(peaked, kb, max(5, args.steps // 2), 3, flush)
        byts = B * (4 * V + 12 * kb)
        e = {"ms": b.median_ms, "queries_per_s": B / (b.median_ms * 1e-3),
             "fraction_of_hbm_peak": byts / (b.median_ms * 1e-3) / 1e9 / peak}
        if do_cpu and kb <= 8192:
            t, _ = _timed(lambda: O.ref_batch_topk(hp.reshape(-1), [i * V for i in range(B)], [V] * B, [kb] * B,
                                                   0, 12, cores), 1)
            e["cpu_baseline"] = {"ms": t * 1e3, "queries_per_s": B / t, "cores": cores, "kind": "reference",
                                 "sample": "same rows, rtk::batch_topk grid_size=cores, one call"}
        res["peaked"][str(kb)] = e
    del peaked
    # LLM sampling consumer: top-k -> softmax -> top-p -> one draw per row
    u = torch.rand(B, device=dev, generator=torch.Generator(device=dev).manual_seed(4))
    for kb, tp in ((50, 0.9), (4096, 0.95)):
        ev = []
        for it in range(3 + max(5, args.steps // 2)):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            R.topk_sample(logits, kb, top_p=tp, temperature=1.0, uniform=u)
            e1.record()
            if it >= 3:
                ev.append((e0, e1))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in ev)
        res["sampling"][f"k{kb}_p{tp}"] = {"ms": ms, "rows_per_s": B / (ms * 1e-3)}
    return res


def leg_c4(args, R, dev, peak, cores, do_cpu):
    """C4 (BASELINE configs[3]): n = 2^26 Uniform[128.6, 128.7) fp32 (one first-window bin, heavy
    ties), k = 2^16, scaled_topk Off / Always / Adaptive (tau 0.5, seed 31)."""
    import numpy as np
    import oracle as O
    import torch
    n, k = 1 << 26, 1 << 16
    hx = (np.float32(128.6) + np.float32(0.1) * np.random.default_rng(5).random(n, dtype=np.float32)).astype(np.float32)
    x = torch.from_numpy(hx).to(dev)
    res = {"config": "n=2^26 128.6 + 0.1 * PCG64(5) U[0,1) fp32, k=2^16, largest, scaled_topk tau=0.5 seed=31; "
                     "input 256 MB > L2"}
    for name, mode in (("off", 0), ("always", 1), ("adaptive", 2)):
        pol = R.ScalePolicy(mode=R.ScaleMode(mode), trigger_fraction=0.5, seed=31)
        b = R.bench_scaled(x, k, max(5, args.steps // 2), 3, policy=pol)
        e = {"ms": b.median_ms, "host_ms": b.median_host_ms, "GBps": gbs(4 * n, k, b.median_ms),
             "fraction_of_hbm_peak": gbs(4 * n, k, b.median_ms) / peak}
        if do_cpu:
            t, _ = _timed(lambda: O.ref_scaled_topk(hx, k, 0, 12, mode, 0.5, 31, cores), 1)
            e["cpu_baseline"] = {"ms": t * 1e3, "GBps": gbs(4 * n, k, t * 1e3), "cores": cores, "kind": "reference",
                                 "sample": "same input, rtk::scaled_topk grid_size=cores, one call"}
        res[name] = e
    return res


def leg_c5_1gpu(args, R, dev, peak):
    """The C5 shard shape on one GPU (2^29 Philox elements, k = 2^16): the per-GPU baseline the
    N > 1 runs scale from."""
    ns, k = 1 << args.shard_logn, args.shard_k
    x = R.generate_philox(ns, C5_SEED, 0, device=dev)
    b = R.bench_topk(x, k, max(5, args.steps // 2), 3)
    return {"config": f"n=2^{args.shard_logn} Philox seed {C5_SEED} elements [0, 2^{args.shard_logn}), k={k}",
            "ms": b.median_ms, "host_ms": b.median_host_ms, "GBps": gbs(4 * ns, k, b.median_ms),
            "fraction_of_hbm_peak": gbs(4 * ns, k, b.median_ms) / peak}


def multi_gpu(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2501_14336_b200 as rtk
    from paper_2501_14336_b200 import rtk as R
    from paper_2501_14336_b200 import sharded as SH

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    peak, peak_kind = measured_peak()
    ns, k = 1 << args.shard_logn, args.shard_k
    n = world * ns
    x = R.generate_philox(ns, C5_SEED, rank * ns, device=dev)
    comm = SH.NcclComm(rank, world, local)
    lens = [ns] * world
    stream = torch.cuda.current_stream(dev)

    def step():
        return SH.topk_sharded(x, k, lens, comm)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for a, b in ev:
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([statistics.median(ms)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    med = float(t.item())
    per_step = rtk.last_stats(local).kernel_launches  # the merge call's; + the local call's below
    rtk.topk(x, k)
    per_step += rtk.last_stats(local).kernel_launches

    # e2e: this rank's shard from pinned host memory, the sharded call, the result back to the host
    hx = x.cpu().pin_memory()
    xd = torch.empty_like(x)
    te = []
    for i in range(args.e2e_steps + 1):
        dist.barrier()
        t0 = time.perf_counter()
        xd.copy_(hx, non_blocking=True)
        r = SH.topk_sharded(xd, k, lens, comm)
        vals, idx = r.values.cpu(), r.indices.cpu()
        if i:
            te.append(time.perf_counter() - t0)
    tt = torch.tensor([statistics.median(te)], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    te_s = float(tt.item())
    if rank == 0:
        value = gbs(4 * n, k, med)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": med, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (Philox on each rank's device)",
            "config": c5_config(args, world), "elements_per_s": n / (med * 1e-3),
            "fraction_of_hbm_peak_per_gpu": value / world / peak,
            "roofline": {"bound": "hbm", "achieved": value / world, "peak": peak, "unit": "GB/s",
                         "frac": value / world / peak, "traffic": None, "kernel": "whole step per GPU",
                         "peak_kind": peak_kind},
            "cpu_baseline": None,
            "e2e": {"value": gbs(4 * n, k, te_s * 1e3), "unit": "GB/s", "h2d_bytes_per_step": 4 * ns,
                    "d2h_bytes_per_step": 12 * k, "ms_per_step": te_s * 1e3,
                    "note": "per rank: pinned H2D of its shard + rtk_topk_sharded + D2H of the result; max over ranks"},
            "gpu_launches": per_step * args.steps, "clocks": clk.summary(),
            "timing": "torch CUDA events around each rtk_topk_sharded step on each rank, median over steps, max "
                      "over ranks", "step_ms_rank0": ms}))
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

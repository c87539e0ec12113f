#!/usr/bin/env python3
"""bench.py — B200 radix top-k benchmark (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], the headline): ONE fp32 query, n = 2^28 Uniform[0,1)
elements resident in HBM per GPU, k = 2^20 (largest), values + u64 indices in the reference's
canonical order. The metric is the paper/north-star "effective GB/s" = algorithmic bytes
(4n + 12k per query: read every key once, write k values + k u64 indices) / time.

* value     device-resident input, CUDA events on the launching stream around rtk_topk.
* e2e       the same metric through the host entry point rtk_topk_host (pinned host input,
            H2D of the 1 GiB input and D2H of the result inside the timed region).
* roofline  the dominant kernel (k_compact, the single streaming pass) timed with CUDA events
            inside the library on its stream; algorithmic bytes per launch = 4n.
* cpu_baseline  the reference's own CPU engine (oracle/_ref: rtk::topk compiled from the
            reference headers) on this box's host cores, on a bounded sample.

Multi-GPU (torchrun, N>1): weak scaling of the same query shape — each rank owns a 2^28 shard
of one N*2^28-element query, runs the local top-k, the k candidates are all-gathered over NCCL
and merged with rtk_merge_shards. Time = max over ranks.

--impl reference: the reference CPU engine (oracle/_ref) on the host cores, same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


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


def cpu_reference_leg(n: int, k: int, reps: int, seed: int = 1):
    """Time the reference's CPU engine (oracle/_ref) on the host cores: effective GB/s."""
    import numpy as np
    import oracle as O
    cores = os.cpu_count() or 1
    x = np.random.default_rng(seed).random(n, dtype=np.float32)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.ref_topk(x, k, 0, 12, cores)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return (4 * n + 12 * k) / t / 1e9, cores, t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--logn", type=int, default=28)
    ap.add_argument("--k", type=int, default=1 << 20)
    ap.add_argument("--sweep", type=str, default="256,16384", help="extra k values (device value only)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch-ks", type=str, default="50,4096,128256",
                    help="C3 batched LLM-vocab top-k: k values measured into batch_llm (empty = skip)")
    ap.add_argument("--batch-rows", type=int, default=256)
    ap.add_argument("--c4", type=int, default=1, help="C4 adversarial scaled_topk leg (1 = on)")
    ap.add_argument("--vocab", type=int, default=128256)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n, k = 1 << args.logn, args.k
    metric = "topk_effective_GBps"
    config = {"workload": f"single query fp32 Uniform[0,1) n=2^{args.logn} per GPU, k={k}, largest, "
                          "values+u64 indices, sorted (BASELINE configs[1])",
              "n_per_gpu": n, "k": k, "dtype": "f32", "order": "largest",
              "l2": "input 1 GiB per GPU > 126 MB L2 (no flush needed)",
              "parallelism": f"n-sharded x{world}: local top-k + NCCL allgather + merge" if world > 1 else "single"}

    if args.impl == "reference":
        if rank != 0:
            return
        # bounded sample of the same workload per step: n_s = 2^26, k scaled by n_s / n
        ns = min(n, 1 << 26)
        ks = max(1, k * ns // n)
        for _ in range(args.warmup):
            cpu_reference_leg(ns, ks, 1)
        vals = [cpu_reference_leg(ns, ks, 1)[0] for _ in range(args.steps)]
        gbs = statistics.median(vals)
        cores = os.cpu_count() or 1
        sample = f"n=2^{ns.bit_length() - 1} U[0,1) k={ks} per step (k scaled by n_s/n), rtk::topk grid_size={cores}"
        print(json.dumps({"impl": "reference", "metric": metric, "value": gbs, "unit": "GB/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "higher_is_better": True, "dtype": "f32", "data": "synthetic",
                          "config": config,
                          "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference",
                                           "sample": sample},
                          "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    import torch
    import paper_2501_14336_b200 as rtk
    from paper_2501_14336_b200 import rtk as R

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1 + rank)
    x = torch.rand(n, device=dev, dtype=torch.float32, generator=gen)
    stream = torch.cuda.current_stream(dev)

    def step(kk):
        r = rtk.topk(x, kk)
        if world > 1:
            import torch.distributed as dist
            vals = torch.empty(world * kk, dtype=torch.float32, device=dev)
            idx = torch.empty(world * kk, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(vals, r.values)
            dist.all_gather_into_tensor(idx, r.indices)
            r = rtk.merge_shards(vals, idx, [kk] * world, [g * n for g in range(world)], kk)
        return r

    def python_loop(kk, steps, warmup):
        for _ in range(warmup):
            step(kk)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            a.record(stream)
            step(kk)
            b.record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev]

    def timed(kk, steps, warmup):
        if world == 1:
            # steps issued from C through rtk_topk (the drop-in boundary; the reference's call
            # sites are C++ loops over rtk::topk), CUDA events per step on the stream
            torch.cuda.synchronize()
            _, ms = R.bench_topk(x, kk, steps, warmup)
        else:
            ms = python_loop(kk, steps, warmup)
        # kernel share: k_compact bracketed by CUDA events on its stream (library timing mode:
        # no graph replay), on separate steps so no stats readback sits inside the timed region
        # (on the local top-k call: with N > 1 the merge that follows is a separate small call)
        R.set_timing(True, local)
        comp = []
        per_step = 0
        for _ in range(min(steps, 10)):
            rtk.topk(x, kk)
            st = R.last_stats(local)
            comp.append(st.compact_ms)
            per_step = st.kernel_launches
        R.set_timing(False, local)
        if world > 1:  # + the merge of the gathered candidates (rtk_merge_shards)
            step(kk)
            per_step += R.last_stats(local).kernel_launches
        launches = per_step * steps
        if world > 1:
            t = torch.tensor([statistics.mean(ms)], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            mean_ms = float(t.item())
        else:
            mean_ms = statistics.mean(ms)
        return mean_ms, ms, comp, launches

    peak, peak_kind = measured_peak()
    with ClockSampler(local) as clk:
        mean_ms, ms, comp, launches = timed(k, args.steps, args.warmup)
    clocks = clk.summary()
    py_ms = statistics.mean(python_loop(k, max(5, args.steps // 2), 2)) if world == 1 else None
    total_bytes = world * (4 * n) + 12 * k
    value = total_bytes / (mean_ms * 1e-3) / 1e9

    sweep = {}
    for kk in [int(v) for v in args.sweep.split(",") if v]:
        m2, _, c2, _ = timed(kk, max(5, args.steps // 2), 2)
        sweep[str(kk)] = {"ms_per_step": m2, "GBps": (world * 4 * n + 12 * kk) / (m2 * 1e-3) / 1e9,
                          "compact_ms": statistics.mean(c2)}

    comp_ms = statistics.mean(comp)
    achieved = 4 * n / (comp_ms * 1e-3) / 1e9

    # C4: adversarial distribution (one first-pass bin, ~6.5K distinct values => heavy ties),
    # scaled_topk with the reference's three scale policies (scaling.hpp:42-86)
    adversarial = {}
    if args.c4 and rank == 0:
        na, ka = 1 << 26, 1 << 16
        xa = (128.6 + 0.1 * torch.rand(na, device=dev, generator=gen)).float()
        for name, mode in (("off", 0), ("always", 1), ("adaptive", 2)):
            pol = R.ScalePolicy(mode=R.ScaleMode(mode), trigger_fraction=0.5, seed=31)
            # steps issued from C (rtk_bench_scaled): events before the scale decision's kernels
            # and after the call's last device operation, as for the C2 value
            ms_a, _ = R.bench_scaled(xa, ka, max(5, args.steps // 2), 3, policy=pol)
            adversarial[name] = {"ms": ms_a, "GBps": (4 * na + 12 * ka) / (ms_a * 1e-3) / 1e9,
                                 "fraction_of_hbm_peak": (4 * na + 12 * ka) / (ms_a * 1e-3) / 1e9 / peak}
        del xa

    # C3: batched LLM sampling top-k, rows sharded across ranks (no collective)
    batch_llm, batch_bf16, sampling = {}, {}, {}
    if args.batch_ks:
        from paper_2501_14336_b200 import sharded as SH
        r0, r1 = SH.row_shard(args.batch_rows, world, rank)
        rows_here = r1 - r0
        V = args.vocab
        logits = torch.randn(rows_here, V, device=dev, generator=gen)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2: flush between steps
        for kb in [int(v) for v in args.batch_ks.split(",") if v]:
            kb = min(kb, V)
            # steps issued from C (rtk_bench_batched), L2 flushed between steps outside the events
            torch.cuda.synchronize()
            ms_b, _ = R.bench_batch_dense(logits, kb, max(5, args.steps // 2), 3, flush)
            if world > 1:
                t = torch.tensor([ms_b], device=dev)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                ms_b = float(t.item())
            q = args.batch_rows / (ms_b * 1e-3)
            byts = args.batch_rows * (4 * V + 12 * kb)
            batch_llm[str(kb)] = {"ms_per_batch": ms_b, "queries_per_s": q, "effective_GBps": byts / (ms_b * 1e-3) / 1e9,
                                  "fraction_of_hbm_peak": byts / (ms_b * 1e-3) / 1e9 / peak}
        # the same batches with bf16 logits (16-bit keys): half the bytes per element
        batch_bf16 = {}
        lb = logits.to(torch.bfloat16)
        for kb in [int(v) for v in args.batch_ks.split(",") if v]:
            kb = min(kb, V)
            torch.cuda.synchronize()
            ms_h, _ = R.bench_batch_dense(lb, kb, max(5, args.steps // 2), 3, flush)
            byts = args.batch_rows * (2 * V + 10 * kb)
            batch_bf16[str(kb)] = {"ms_per_batch": ms_h, "queries_per_s": args.batch_rows / (ms_h * 1e-3),
                                   "effective_GBps": byts / (ms_h * 1e-3) / 1e9,
                                   "fraction_of_hbm_peak": byts / (ms_h * 1e-3) / 1e9 / peak}
        # LLM sampling consumer: top-k 50 -> softmax -> top-p 0.9 -> one draw per
        # row, through rtk.topk_sample (Python loop, torch events, L2 flushed outside the events)
        sampling = {}
        u = torch.rand(rows_here, device=dev, generator=gen)
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
            ms_s = statistics.median(a.elapsed_time(b) for a, b in ev)
            sampling[f"k{kb}_p{tp}"] = {"ms_per_batch": ms_s, "queries_per_s": args.batch_rows / (ms_s * 1e-3)}
        del logits, flush, lb

    # e2e through the host entry point (rank 0 / N=1 semantics: per-GPU query from pinned host)
    e2e = None
    if rank == 0:
        hx = x.cpu().pin_memory()
        hv = hx.numpy()
        R.topk(hv, k)
        t_e2e = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            R.topk(hv, k)
            t_e2e.append(time.perf_counter() - t0)
        te = statistics.median(t_e2e)
        e2e = {"value": (4 * n + 12 * k) / te / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
               "d2h_bytes_per_step": 12 * k + 4, "ms_per_step": te * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ns = 1 << 26
        ks = max(1, k * ns // n)
        gbs, cores, t = cpu_reference_leg(ns, ks, 3)
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference",
               "sample": f"rtk::topk (reference engine, oracle/_ref) n=2^26 U[0,1) k={ks}, "
                         f"grid_size={cores}, median of 3 ({t:.2f} s each)"}

    if rank == 0:
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        traffic = None
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"k_compact_n{n}")
        except Exception:
            pass
        out = {"metric": metric, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (torch.rand on device)",
               "config": config,
               "queries_per_s": world / (mean_ms * 1e-3) if world == 1 else 1 / (mean_ms * 1e-3),
               "elements_per_s": world * n / (mean_ms * 1e-3),
               "fraction_of_hbm_peak": value / peak,
               "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                            "frac": achieved / peak, "traffic": traffic, "kernel": "k_compact",
                            "peak_kind": peak_kind, "kernel_ms": comp_ms,
                            "kernel_share_of_step": comp_ms / mean_ms},
               "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
               "timing": "steps issued back-to-back from C through rtk_topk (rtk_bench_topk); per step two "
                         "CUDA events the engine records on the launching stream right before its first and "
                         "after its last device operation of the call (host planning and the host's wait for "
                         "the completion signal are outside; they are inside e2e and python_loop_ms); "
                         "python_loop_ms = the same call through the Python mirror (rtk.topk) with torch "
                         "events around the whole call",
               "python_loop_ms": py_ms,
               "k_sweep": sweep,
               "adversarial_c4": {"config": "n=2^26 Uniform[128.6,128.7) fp32, k=2^16, largest, scaled_topk "
                                            "tau=0.5 seed=31 (device-resident)", "results": adversarial},
               "batch_llm_bf16": {"config": "the same logits rounded to bf16 (2 B per element; bytes = "
                                            "rows * (2V + 10k))", "results": batch_bf16},
               "llm_sampling": {"config": "the fp32 logits batch: top-k -> softmax -> top-p -> one draw per row "
                                          "(rtk.topk_sample, Python loop, torch events)", "results": sampling},
               "batch_llm": {"config": f"{args.batch_rows} x {args.vocab} fp32 N(0,1) logits, rows sharded over "
                                       f"{world} GPU(s), L2 flushed between batches", "results": batch_llm},
               "step_ms_all": ms}
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

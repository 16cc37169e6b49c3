#!/usr/bin/env python3
"""xorgensGP throughput on B200: RN/s (32-bit, device-timed), % of HBM roofline.

Default workload (BASELINE.json configs[1]): fill of 2^30 uint32 per GPU,
P = 2^14 streams x 2^16 words, base_seed 1, block-major, bit-exact with the
reference.  A "step" is one BlockEnsemble::generate(2^16) pass over the
persistent ensemble (streams continue across steps, exactly like repeated
generate() calls in the reference, proj/src/parallel.cpp:97-135 and
proj/src/bench.cpp:95-112) -- one pair_kernel launch (xg_pairs.cuh).

Other workloads (--workload): fill_f32, fill_f64 (config 3), fill_2p34
(config 4: 2^34 words over N GPUs, strong scaling), mc_pi (config 5: 2^40
samples over N GPUs, one NCCL all-reduce of the uint64 hit count).

  python bench.py [--gpus N --steps K --warmup W] [--workload W] [--impl reference]
Multi-GPU: launched by torchrun, one rank per GPU; each rank owns a disjoint
stream range; timing = max over ranks of CUDA-event time.
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

def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_ncu(workload: str) -> dict:
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(workload, {})
    except Exception:
        return {}


def load_traffic(workload: str):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every
    ~2 ms during the timed region (nvidia-smi as a fallback)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                if nv is not None:
                    sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                    try:
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                    except Exception:
                        rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                    self.samples.append((float(sm), int(rs)))
                    self._stop.wait(0.002)
                else:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip().split(",")
                    self.samples.append((float(out[0]), 0))
                    self.max_mhz = float(out[1])
                    self._stop.wait(0.05)
            except Exception:
                self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        sm = [s for s, _ in self.samples]
        reasons = sorted({name for _, r in self.samples for bit, name in self.REASONS.items()
                          if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "sm_mhz_min": min(sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def write_probe_gbs(out, stream, reps: int = 5):
    """Write-only HBM ceiling on the same buffer (libxg_probe.so, bench-only)."""
    import ctypes

    import torch

    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1108_0486_b200", "lib", "libxg_probe.so"))
    lib.xg_probe_write.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    nbytes = out.numel() * out.element_size()
    ptr, sp = ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream.cuda_stream)
    for _ in range(3):
        lib.xg_probe_write(ptr, nbytes, sp)
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lib.xg_probe_write(ptr, nbytes, sp)
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / (best / 1e3) / 1e9


def dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # XG_BENCH_BACKEND=gloo (testing only): exercise the N>1 flow with every
    # rank on the visible GPUs round-robin, e.g. two ranks on one GPU.
    backend = os.environ.get("XG_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    if world > 1 and not dist.is_initialized():
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    elif world == 1:
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------
# CPU baseline / reference arm: the reference's own code (oracle/_ref),
# BlockEnsemble(p, 1, P, 63).generate(per_block) on all host threads,
# wall-clocked around generate() as measure_ensemble_throughput does.
# --------------------------------------------------------------------------

def reference_rate(streams: int, per_block: int, trials: int, warmup: int = 1, budget_s: float = 30.0,
                   min_trials: int = 3):
    from oracle import REF_SO, Oracle, Reference

    threads = os.cpu_count() or 1
    if os.path.exists(REF_SO):
        ref = Reference()
        p = Oracle().gp32()
        h = ref.ensemble(p, 1, streams, 63)
        rates = []
        t0 = time.perf_counter()
        for i in range(warmup + trials):
            secs, _ = ref.generate_timed(h, per_block, threads)
            if i >= warmup:
                rates.append(streams * per_block / secs)
            if time.perf_counter() - t0 > budget_s and len(rates) >= min_trials:
                break
        ref.destroy(h)
        kind = "reference"
    else:  # the C restatement, when the reference could not be compiled
        import numpy as np  # noqa: F401

        o = Oracle()
        e = o.ensemble(1, streams)
        rates = []
        for i in range(warmup + trials):
            t = time.perf_counter()
            e.fill_u32(per_block)
            dt = time.perf_counter() - t
            if i >= warmup:
                rates.append(streams * per_block / dt)
        kind = "port"
    return {"value": statistics.mean(rates), "unit": "RN/s", "cores": threads, "kind": kind,
            "sample": f"BlockEnsemble(xorgensgp32, base_seed=1, blocks={streams}, lanes=63)"
                      f".generate({per_block}) = {streams * per_block} words per trial, "
                      f"{len(rates)} trials after {warmup} warm-up, workers={threads}, "
                      f"wall clock around generate() (proj/src/bench.cpp:95-112)",
            "trials": len(rates), "min": min(rates), "max": max(rates)}


def run_reference_arm(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    streams = 1 << 14
    per_block = 1 << 13  # 2^27 words per step (8 B/word in the reference: 1 GiB of vectors)
    base = reference_rate(streams, per_block, trials=max(1, args.steps), warmup=args.warmup,
                          budget_s=120.0)
    v = base["value"]
    line = {
        "impl": "reference", "metric": "RN/s (32-bit, device-timed) at 1/2/4/8 B200; % of HBM write BW",
        "value": v, "unit": "RN/s", "n_gpus": world, "steps": base["trials"], "warmup": args.warmup,
        "ms_per_step": streams * per_block / v * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "xorgensGP fill, xorgensgp32, base_seed 1, 2^14 streams "
                               f"(reference BlockEnsemble::generate, {per_block} words/stream/step "
                               "bounded sample of the 2^30-word config)",
                   "streams": streams, "per_stream": per_block},
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": v, "unit": "RN/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def workload_geometry(wl: str, world: int, rank: int):
    """Per-rank stream slice and per-stream length of each workload, and the
    words the whole job consumes per step.  Weak scaling: every rank owns
    2^14 streams of its own (global ids rank*2^14 ...), 2^30 values per GPU.
    Strong scaling: one global ensemble split by xg_partition."""
    import paper_1108_0486_b200 as xg

    if wl in ("fill_u32", "fill_f32", "fill_f64", "skip"):
        P, per = 1 << 14, 1 << 16
        words = P * per * (2 if wl == "fill_f64" else 1)
        return rank * P, P, per, "weak", words * world
    if wl == "rank":  # fused GF(2) matrix-rank test: 2^14 streams x 2^12 32x32 matrices per GPU
        P = 1 << 14
        return rank * P, P, 1 << 12, "weak", (P << 17) * world
    if wl == "lc":  # linear complexity test: 2^14 streams x 256 blocks of 1000 bits per GPU
        P = 1 << 14
        return rank * P, P, 256, "weak", P * 256 * 1000 // 32 * world
    if wl == "stream1":  # config 1 on the GPU: ONE stream (seed 1 + rank), 10^8 words
        return rank, 1, 10**8, "weak", 10**8 * world
    if wl == "fill_2p34":
        first, count = xg.partition(1 << 18, world, rank)
        return first, count, 1 << 16, "strong", 1 << 34
    if wl == "mc_pi":
        total_streams = 1 << 17
        first, count = xg.partition(total_streams, world, rank)
        return first, count, (1 << 40) // total_streams, "strong", 1 << 41
    raise ValueError(wl)


def timed_loop(fn, stream, steps, warmup, world, counter=None):
    """W warm-ups, then K timed steps bracketed by barrier + synchronize;
    per-step CUDA events on the launching stream.  Returns (total_ms,
    [step_ms], launches): `counter()` (our kernel-launch count) read around
    the timed steps only."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    c0 = counter() if counter else 0
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(steps):
        evs[2 * i].record(stream)
        fn()
        evs[2 * i + 1].record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    launches = (counter() - c0) if counter else 0
    step_ms = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(steps)]
    total = start.elapsed_time(end)
    return total, step_ms, launches


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="GPUs in the job; N>1 runs under torchrun (one rank per GPU)")
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 200 for fills, 5 for mc_pi)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="fill_u32",
                    choices=["fill_u32", "fill_f32", "fill_f64", "fill_2p34", "mc_pi", "skip", "stream1",
                             "rank", "lc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.steps is None:
        args.steps = 5 if args.workload == "mc_pi" else (10 if args.impl == "reference" else 500)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    import paper_1108_0486_b200 as xg

    world, rank, local = dist_setup()
    if args.gpus != world and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun",
              file=sys.stderr)
    stream = torch.cuda.current_stream()
    p = xg.xorgensgp32_params()
    wl = args.workload
    hbm_peak, peak_src = load_peaks()

    first, count, per, scaling, job_words_per_step = workload_geometry(wl, world, rank)
    ens = xg.BlockEnsemble(p, 1, count, 63, first_stream=first, device=local)

    out = None
    bytes_per_val = {"fill_u32": 4, "fill_f32": 4, "fill_f64": 8, "fill_2p34": 4, "mc_pi": 0,
                     "skip": 0, "stream1": 4, "rank": 0, "lc": 0}[wl]
    words_per_val = {"fill_f64": 2, "mc_pi": 2, "rank": 32, "lc": 1000 / 32}.get(wl, 1)
    if wl in ("fill_u32", "fill_2p34", "stream1"):
        out = torch.empty((count, per), dtype=torch.uint32, device="cuda")
        fn = lambda: ens.fill_u32(per, out=out)  # noqa: E731
    elif wl == "fill_f32":
        out = torch.empty((count, per), dtype=torch.float32, device="cuda")
        fn = lambda: ens.fill_f32(per, out=out)  # noqa: E731
    elif wl == "fill_f64":
        out = torch.empty((count, per), dtype=torch.float64, device="cuda")
        fn = lambda: ens.fill_f64(per, out=out)  # noqa: E731
    elif wl == "skip":  # generator core only (no stores): the integer-issue ceiling
        hits = None
        fn = lambda: ens.skip(per)  # noqa: E731
    elif wl == "lc":  # linear complexity test: words to a buffer, Berlekamp-Massey per block
        hits = torch.zeros(1001, dtype=torch.int64, device="cuda")
        fn = lambda: ens.linear_complexity_test(1000, per, hist=hits)  # noqa: E731
    elif wl == "rank":  # fused matrix-rank test: bins only, no HBM traffic
        hits = torch.zeros(3, dtype=torch.int64, device="cuda")
        fn = lambda: ens.rank_test(per, counts=hits)  # noqa: E731
    else:
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        fn = lambda: ens.mc_pi(per, hits=hits)  # noqa: E731

    vals_per_step = count * per
    words_per_step = vals_per_step * words_per_val
    with ClockSampler(local) as clk:
        total_ms, step_ms, launches = timed_loop(fn, stream, args.steps, args.warmup, world,
                                                 counter=xg.kernel_launches)
    t_max = max_over_ranks(total_ms, world)
    value = job_words_per_step * args.steps / (t_max / 1e3)
    kern_ms = statistics.mean(step_ms)
    state_bytes = 2 * count * 129 * 4                     # window + weyl read and written back
    alg_bytes = vals_per_step * bytes_per_val + state_bytes

    result = {
        "metric": "RN/s (32-bit, device-timed) at 1/2/4/8 B200; % of HBM write BW",
        "value": value, "unit": "RN/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None,
        "dtype": {"fill_f32": "u32->f32", "fill_f64": "u32->f64"}.get(wl, "u32"),
        "data": "synthetic (seeded generator state; no input data)",
        "config": {"workload": {
            "fill_u32": "xorgensGP fill of 2^30 uint32 per GPU, bit-exact vs CPU per stream",
            "fill_f32": "uniform float32 [0,1) fill of 2^30 values per GPU, fused conversion",
            "fill_f64": "uniform float64 [0,1) fill of 2^30 values (2^31 words) per GPU, fused conversion",
            "fill_2p34": "disjoint-stream fill of 2^34 uint32 across N GPUs",
            "mc_pi": "fused in-register Monte Carlo pi, 2^40 samples across N GPUs",
            "skip": "generator core only (advance 2^30 words, no stores)",
            "stream1": "one stream per GPU (BASELINE config 1: seed 1, 10^8 uint32), one warp",
            "rank": "fused GF(2) 32x32 matrix-rank test (reference matrix_rank_test), "
                    "2^14 streams x 2^12 matrices per GPU",
            "lc": "linear complexity test (reference linear_complexity_test, K = 1000), "
                  "2^14 streams x 256 blocks per GPU"}[wl],
            "params": "xorgensgp32 (128,65,15,14,12,17) w=32", "base_seed": 1,
            "streams_per_gpu": count, "values_per_stream": per,
            "layout": "block-major out[g*per_stream+k]",
            "l2": "output per step >> 126 MB L2 (no flush needed)" if bytes_per_val else
                  "no HBM traffic (in-register consumer)",
            "parallelism": f"dp{world} (disjoint stream ranges, no data-path collective)"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if wl == "stream1":
        # One warp: the dependency chain of the recurrence, not HBM, bounds it.
        result["roofline"] = {"bound": "latency (one warp per stream)", "achieved": value / world,
                              "peak": None, "unit": "RN/s per GPU", "frac": None, "traffic": None,
                              "kernel_ms_mean": kern_ms}
    elif bytes_per_val:
        achieved = alg_bytes / (kern_ms / 1e3) / 1e9
        result["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                              "frac": achieved / hbm_peak, "traffic": load_traffic(wl),
                              "peak_source": peak_src,
                              "alg_bytes_per_launch": alg_bytes,
                              "kernel_ms_mean": kern_ms, "kernel_ms_min": min(step_ms)}
        # write-only ceiling on the same buffer, same run (context for frac)
        if out is not None:
            try:
                result["roofline"]["write_only_probe_gbs"] = write_probe_gbs(out, stream)
            except OSError:
                pass
    elif wl == "lc":
        import paper_1108_0486_b200 as xg_

        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(hits)
        chi2, pv = xg_.linear_complexity_statistic(hits, 1000)
        result["lc"] = {"blocks": int(hits.sum().item()), "chi2": chi2, "p_value": pv,
                        "blocks_per_s": value / (1000 / 32), "kernel_ms_mean": kern_ms}
        result["roofline"] = {"bound": "int-issue (Berlekamp-Massey, one warp per block)",
                              "achieved": value / world, "peak": None, "unit": "RN/s per GPU",
                              "frac": None, "traffic": None}
    elif wl == "rank":
        import paper_1108_0486_b200 as xg_

        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(hits)
        c = [int(v) for v in hits.tolist()]
        chi2, pv = xg_.matrix_rank_statistic(c)
        result["rank"] = {"counts_rank32_31_le30": c, "chi2": chi2, "p_value": pv,
                          "matrices_per_s": value / 32, "kernel_ms_mean": kern_ms}
        pipes = load_ncu(wl)
        result["roofline"] = {
            "bound": "int-issue", "achieved": value / world, "peak": None, "unit": "RN/s per GPU",
            "frac": None, "traffic": load_traffic(wl),
            "alu_pipe_pct": pipes.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": pipes.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "pipe_source": "profiles/ncu_summary.json (ncu --set full)"}
    elif wl == "skip":
        result["roofline"] = {"bound": "int-issue", "achieved": value / world, "peak": None,
                              "unit": "RN/s per GPU", "frac": None, "traffic": None,
                              "kernel_ms_mean": kern_ms}
    else:
        # in-register consumer: report integer-issue context
        hits_v = int(hits.item())
        if world > 1:
            import torch.distributed as dist
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            dist.all_reduce(hits)  # the one NCCL collective of the workload (uint64 sum)
            t1.record(stream)
            torch.cuda.synchronize()
            hits_v = int(hits.item())
            result["allreduce_ms"] = t0.elapsed_time(t1)
        samples = (args.steps + args.warmup) * (1 << 40)
        result["mc"] = {"hits": hits_v, "samples": samples, "pi_estimate": 4.0 * hits_v / samples,
                        "kernel_ms_mean": kern_ms}
        # In-register consumer: no HBM roofline.  The ceiling is the integer
        # pipes; report their ncu utilisation (profiles/ncu_summary.json).
        pipes = load_ncu(wl)
        result["roofline"] = {
            "bound": "int-issue", "achieved": value / world, "peak": None, "unit": "RN/s per GPU",
            "frac": None, "traffic": load_traffic(wl),
            "alu_pipe_pct": pipes.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": pipes.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "pipe_source": "profiles/ncu_summary.json (ncu --set full)"}

    # e2e through the public host API (generate into pinned host memory)
    if not args.no_e2e and wl == "fill_u32":
        host = torch.empty((count, per), dtype=torch.uint32, pin_memory=True)
        e2e_steps = max(3, min(args.steps, 5))
        for _ in range(1):
            ens.generate_into_host(per, host)
        barrier(world)
        t = time.perf_counter()
        for _ in range(e2e_steps):
            ens.generate_into_host(per, host)
        dt = max_over_ranks(time.perf_counter() - t, world)
        result["e2e"] = {"value": words_per_step * world * e2e_steps / dt, "unit": "RN/s",
                         "h2d_bytes_per_step": 0, "d2h_bytes_per_step": words_per_step * 4,
                         "api": "BlockEnsemble.generate -> xg_generate_host (pinned host buffer)",
                         "steps": e2e_steps}
        del host
    if rank == 0 and world == 1 and not args.no_cpu and wl == "lc":
        try:
            from oracle import Battery, Oracle

            nb = 3000  # bounded sample: 3e6 bits through the reference's own test
            words = Oracle().ensemble(1, 1).fill_u32(nb * 1000 // 32)[0]
            t0 = time.perf_counter()
            Battery().linear_complexity(words, 1000, nb)
            dt = time.perf_counter() - t0
            result["cpu_baseline"] = {
                "value": nb * 1000 / 32 / dt, "unit": "RN/s", "cores": 1, "kind": "reference",
                "sample": f"reference linear_complexity_test (proj/src/stattests/tests.cpp:128-178), "
                          f"{nb} blocks of 1000 bits of one stream, 1 thread (serial in the reference)",
                "blocks_per_s": nb / dt}
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    if rank == 0 and world == 1 and not args.no_cpu and wl == "rank":
        try:
            from oracle import Battery, Oracle

            m = 200_000  # bounded sample: 6.4e6 words through the reference's own test
            words = Oracle().ensemble(1, 1).fill_u32(32 * m)[0]
            t0 = time.perf_counter()
            Battery().matrix_rank(words, m)
            dt = time.perf_counter() - t0
            result["cpu_baseline"] = {
                "value": 32 * m / dt, "unit": "RN/s", "cores": 1, "kind": "reference",
                "sample": f"reference matrix_rank_test (proj/src/stattests/tests.cpp:81-126) over "
                          f"{m} 32x32 matrices of one stream, 1 thread (the reference test is serial)",
                "matrices_per_s": m / dt}
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    if rank == 0 and world == 1 and not args.no_cpu and wl == "stream1":
        try:
            from oracle import Reference

            result["cpu_baseline"] = {
                "value": Reference().serial_rate(1, 10**8, 20), "unit": "RN/s", "cores": 1,
                "kind": "reference",
                "sample": "XorgensState(xorgensgp32, 1): 10^8 next_word in 20 chunks, best "
                          "chunk rate (measure_throughput, proj/src/bench.cpp:67-93)"}
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    if rank == 0 and world == 1 and not args.no_cpu and wl in ("fill_u32", "fill_f32", "fill_f64"):
        try:
            cb = reference_rate(1 << 14, 1 << 14, trials=100, budget_s=10.0)
            for k in ("trials", "min", "max"):
                cb.pop(k, None)
            # BASELINE config 1: one serial stream on one core, the reference's
            # measure_throughput method (proj/src/bench.cpp:67-93), seed 1, 10^8 words.
            try:
                from oracle import Reference

                cb["serial_1core_rn_per_s"] = Reference().serial_rate(1, 10**8, 20)
            except Exception:  # noqa: BLE001
                pass
            result["cpu_baseline"] = cb
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

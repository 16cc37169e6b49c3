#!/usr/bin/env python3
"""xorgensGP throughput on B200: RN/s (32-bit, device-timed), % of HBM write BW.

Default workload (BASELINE.json configs[1]): fill of 2^30 uint32 per GPU,
P = 2^14 streams x 2^16 words, base_seed 1, block-major, bit-exact with the
reference.  A "step" is one BlockEnsemble::generate(2^16) pass over the
persistent ensemble (streams continue across steps, exactly like repeated
generate() calls in the reference, proj/src/parallel.cpp:97-135 and
proj/src/bench.cpp:95-112) -- one pair_kernel launch (xg_pairs.cuh).

The default line also carries, each under the same clock and with its own
roofline, parity check and CPU baseline, the other BASELINE configs as
``extra_workloads``: fill_f32 / fill_f64 (config 3, weak), fill_2p34 (config
4: 2^34 words over N GPUs, strong) and mc_pi (config 5: 2^40 samples over N
GPUs, the uint64 hit count all-reduced over NCCL inside every step).

After the timed loop every workload re-runs on a FRESH ensemble and its
output is digested on the device (xg_digest_u32) and compared stream by
stream with tests/golden/full_size.json (the reference's own words):
``parity.ok``.

  python bench.py [--gpus N --steps K --warmup W] [--workload W] [--impl reference]
--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one rank per GPU, NCCL); each rank owns a disjoint stream range; timing =
max over ranks of CUDA-event time.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import tempfile
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RN/s (32-bit, device-timed) at 1/2/4/8 B200; % of HBM write BW"
FULL_SIZE = os.path.join(ROOT, "tests", "golden", "full_size.json")
CHUNK = 1 << 14  # streams per golden chunk
WORKLOADS = ["fill_u32", "fill_f32", "fill_f64", "fill_2p34", "mc_pi", "skip", "stream1", "rank", "lc"]
EXTRA = ("fill_f32", "fill_f64", "fill_2p34", "mc_pi", "stream1")


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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every
    ~2 ms during the timed region (nvidia-smi as a fallback)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.power = []
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
                    try:
                        pw = nv.nvmlDeviceGetPowerUsage(self._h) / 1e3
                    except Exception:
                        pw = None
                    self.samples.append((float(sm), int(rs)))
                    if pw is not None:
                        self.power.append(pw)
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
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
               "samples": len(self.samples), "sm_mhz_min": min(sm),
               "source": "nvml" if self._nvml is not None else "nvidia-smi"}
        if self.power:
            out["power_w_median"] = statistics.median(self.power)
            out["power_w_max"] = max(self.power)
        return out


# --------------------------------------------------------------------------
# process group
# --------------------------------------------------------------------------

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _nccl_debug_env(env) -> None:
    """NCCL INFO logging (communicator init lines: rank, nRanks, NVLS/P2P
    transport) so the ranks of every N-GPU run are visible in the log; a
    quieter preset (VERSION / WARN / unset) is raised to INFO."""
    if env.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "WARN"):
        env["NCCL_DEBUG"] = "INFO"
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
    # NCCL logs to stdout by default; stdout carries only the JSON line, so
    # the log goes to a per-process file that forward_nccl_log() copies to
    # stderr.
    env.setdefault("NCCL_DEBUG_FILE", os.path.join(tempfile.gettempdir(), "xg_bench_nccl.%h.%p.log"))


def forward_nccl_log() -> None:
    """Copy this process's NCCL log (communicator init: rank, nRanks,
    channels) to stderr and remove it."""
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    if not path.startswith(os.path.join(tempfile.gettempdir(), "xg_bench_nccl.")):
        return
    import glob

    for f in glob.glob(path.replace("%h", "*").replace("%p", str(os.getpid()))):
        try:
            with open(f) as fh:
                sys.stderr.write(fh.read())
            os.remove(f)
        except OSError:
            pass


def self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this script under
    torch.distributed.run with N ranks on this node (the driver's own
    launch line), so `python bench.py --gpus N` is an N-GPU job."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    _nccl_debug_env(env)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def dist_setup(dry: bool = False):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # XG_BENCH_BACKEND=gloo (testing only): exercise the N>1 flow with every
    # rank on the visible GPUs round-robin, e.g. two ranks on one GPU.
    backend = "gloo" if dry else os.environ.get("XG_BENCH_BACKEND", "nccl")
    if not dry and backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    if not dry:
        torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            _nccl_debug_env(os.environ)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    elif world == 1 and not dry and backend == "nccl" and not dist.is_initialized():
        # N = 1: a one-rank NCCL communicator, so the job's collective (the
        # MC hit-count all-reduce) runs through NCCL at every N, this one too.
        _nccl_debug_env(os.environ)
        try:
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}",
                                    rank=0, world_size=1, device_id=torch.device(f"cuda:{local}"))
        except Exception as e:  # noqa: BLE001 -- reported in the line's `comm`
            _COMM_ERR.append(f"{type(e).__name__}: {e}"[:200])
    return world, rank, local


_COMM_ERR: list = []


def _dist_ready() -> bool:
    import torch.distributed as dist

    return dist.is_initialized()


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _coll_device():
    import torch.distributed as dist

    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_ok(ok: bool, world: int) -> bool:
    if world == 1:
        return ok
    import torch
    import torch.distributed as dist

    t = torch.tensor([1 if ok else 0], dtype=torch.int64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def comm_info(world: int) -> dict:
    import torch.distributed as dist

    if world == 1 and not dist.is_initialized():
        return {"backend": None, "nranks": 1, "init_error": _COMM_ERR[0] if _COMM_ERR else None}

    return {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
            "nccl_debug": os.environ.get("NCCL_DEBUG")}


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------

def workload_geometry(wl: str, world: int, rank: int):
    """(first stream, streams, values per stream, scaling, job words per step)
    of a rank.  Weak scaling: every rank owns 2^14 streams of its own (global
    ids rank*2^14 ...), 2^30 values per GPU.  Strong scaling: one global
    ensemble split by xg_partition."""
    import paper_1108_0486_b200 as xg

    if wl in ("fill_u32", "fill_f32", "fill_f64", "skip"):
        P, per = CHUNK, 1 << 16
        words = P * per * (2 if wl == "fill_f64" else 1)
        return rank * P, P, per, "weak", words * world
    if wl == "rank":  # fused GF(2) matrix-rank test: 2^14 streams x 2^12 32x32 matrices per GPU
        P = CHUNK
        return rank * P, P, 1 << 12, "weak", (P << 17) * world
    if wl == "lc":  # linear complexity test: 2^14 streams x 256 blocks of 1000 bits per GPU
        P = CHUNK
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


WORKLOAD_TEXT = {
    "fill_u32": "xorgensGP fill of 2^30 uint32 per GPU, bit-exact vs CPU per stream",
    "fill_f32": "uniform float32 [0,1) fill of 2^30 values per GPU, fused conversion",
    "fill_f64": "uniform float64 [0,1) fill of 2^30 values (2^31 words) per GPU, fused conversion",
    "fill_2p34": "disjoint-stream fill of 2^34 uint32 across N GPUs",
    "mc_pi": "fused in-register Monte Carlo pi, 2^40 samples across N GPUs, NCCL scalar reduce",
    "skip": "generator core only (advance 2^30 words, no stores)",
    "stream1": "one stream per GPU (BASELINE config 1: seed 1, 10^8 uint32), cut into jump-ahead "
               "segments (GF(2) Krylov products, csrc/xg_jump.cuh) generated in parallel",
    "rank": "fused GF(2) 32x32 matrix-rank test (reference matrix_rank_test), "
            "2^14 streams x 2^12 matrices per GPU",
    "lc": "linear complexity test (reference linear_complexity_test, K = 1000), "
          "2^14 streams x 256 blocks per GPU",
}
BYTES_PER_VAL = {"fill_u32": 4, "fill_f32": 4, "fill_f64": 8, "fill_2p34": 4, "stream1": 4}
WORDS_PER_VAL = {"fill_f64": 2, "mc_pi": 2, "rank": 32, "lc": 1000 / 32}


def config_for(wl: str, world: int) -> dict:
    """The workload's config object -- shared verbatim by the reference arm."""
    _, count, per, scaling, _ = workload_geometry(wl, world, 0)
    return {"workload": WORKLOAD_TEXT[wl], "params": "xorgensgp32 (128,65,15,14,12,17) w=32",
            "base_seed": 1, "streams_per_gpu": count, "values_per_stream": per,
            "layout": "block-major out[g*per_stream+k]",
            "l2": "output per step >> 126 MB L2 (no flush needed)" if wl in BYTES_PER_VAL else
                  "no HBM traffic (in-register consumer)",
            "parallelism": f"dp{world} (disjoint stream ranges"
                           + (", one uint64 all-reduce per step)" if wl == "mc_pi" else
                              ", no data-path collective)")}


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


def _load_full_size():
    with open(FULL_SIZE) as f:
        return json.load(f)


def parity_check(wl: str, world: int, rank: int, local: int, out=None) -> dict:
    """Re-run the workload on a FRESH ensemble of this rank's streams and
    compare it with the reference-derived goldens (tests/golden/full_size.json,
    per chunk of 2^14 streams): device digests of every stream for the fills,
    the exact hit count of 2^15 samples per stream for MC.  The verdict is
    the AND over ranks."""
    import numpy as np
    import torch

    import paper_1108_0486_b200 as xg
    from paper_1108_0486_b200.digest import chunk_record, row_digests

    fs = _load_full_size()
    first, count, per, _, _ = workload_geometry(wl, world, rank)
    p = xg.xorgensgp32_params()
    res = {"checked": False}
    if wl == "stream1":
        # BASELINE config 1: seed 1, 10^8 words -- xor, sum_k w_k (k + 1)
        # mod 2^64 and the last word of the reference's stream (every rank
        # checks the seed-1 stream through the same one-stream path)
        with open(os.path.join(ROOT, "tests", "golden", "ref_vectors.json")) as f:
            g = json.load(f)["config1"]
        e = xg.BlockEnsemble(p, g["seed"], 1, 63, device=local)
        buf = e.fill_u32(g["n"], out=out)
        x, _, ws = row_digests(buf)
        last = int(buf[0, -1:].cpu().numpy().view(np.uint32)[0])
        ok = (f"{int(x[0]):08x}" == g["xor"] and f"{int(ws[0]) % 2**64:016x}" == g["sum"]
              and f"{last:08x}" == g["last"])
        res = {"checked": True, "ok_rank0": ok, "streams": 1, "values_per_stream": g["n"],
               "golden": "tests/golden/ref_vectors.json config1 (reference XorgensState, seed 1)",
               "method": "fresh one-stream ensemble (jump-ahead path), device digest (xor, "
                         "weighted sum) and last word vs the reference's"}
        del buf
    elif first % CHUNK or count % CHUNK:
        res["why"] = "rank slice is not whole golden chunks"
    elif wl in ("fill_u32", "fill_2p34", "fill_f32", "fill_f64"):
        key = {"fill_u32": "u32", "fill_2p34": "u32"}.get(wl, wl[5:])
        chunks = fs[key]["chunks"]
        c0, nc = first // CHUNK, count // CHUNK
        if c0 + nc > len(chunks):
            res["why"] = f"golden covers {len(chunks)} chunks; rank needs {c0 + nc}"
        else:
            e = xg.BlockEnsemble(p, 1, count, 63, first_stream=first, device=local)
            fill = {"u32": e.fill_u32, "f32": e.fill_f32, "f64": e.fill_f64}[key]
            buf = fill(per, out=out)
            x, s, ws = row_digests(buf)
            elems = per * (2 if key == "f64" else 1)
            ok = all(chunk_record(x[i * CHUNK:(i + 1) * CHUNK], s[i * CHUNK:(i + 1) * CHUNK],
                                  ws[i * CHUNK:(i + 1) * CHUNK], elems) == chunks[c0 + i]
                     for i in range(nc))
            res = {"checked": True, "ok_rank0": ok, "streams": count, "values_per_stream": per,
                   "golden": f"tests/golden/full_size.json {key} chunks [{c0}, {c0 + nc})",
                   "method": "fresh ensemble, xg_digest_u32 per stream (xor, sum, weighted sum) "
                             "vs digests of the reference's own words"}
            del buf
    elif wl == "mc_pi":
        hits_g = fs["mc"]["chunk_hits"]
        c0, nc = first // CHUNK, count // CHUNK
        spp = fs["mc"]["samples_per_stream"]
        e = xg.BlockEnsemble(p, 1, count, 63, first_stream=first, device=local)
        h = e.mc_pi(spp)
        mine = int(h.item())
        ok = mine == sum(hits_g[c0:c0 + nc])
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([mine], dtype=torch.int64, device=_coll_device())
            dist.all_reduce(t)
            ok = ok and int(t.item()) == fs["mc"]["total_hits_2p32"]
        res = {"checked": True, "ok_rank0": ok, "samples_per_stream": spp,
               "total_samples": spp * (1 << 17),
               "golden": "tests/golden/full_size.json mc (exact hits, 2^32 samples over the "
                         "2^17 streams)",
               "method": "fresh ensemble, exact hit count per rank slice + all-reduced total"}
    else:
        res["why"] = "no full-size golden for this workload (see tests/)"
    if res["checked"]:
        res["ok"] = all_ok(res["ok_rank0"], world)
        del res["ok_rank0"]
    else:
        all_ok(True, world)  # keep the collective sequence aligned across ranks
    return res


def probe_shapes(out, stream) -> dict:
    """Write-only store patterns over `out` (libxg_probe.so): memset, the
    fill's store shape (one warp per row, 8- or 16-byte stores, 4 rows per
    CTA, <= 4 resident CTAs per SM) and a grid-stride stream; each returns
    nonzero on failure."""
    import ctypes

    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1108_0486_b200", "lib", "libxg_probe.so"))
    vp = ctypes.c_void_p
    lib.xg_probe_memset.argtypes = [vp, ctypes.c_size_t, vp]
    lib.xg_probe_rows.argtypes = [vp, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, vp]
    lib.xg_probe_gridstride.argtypes = [vp, ctypes.c_size_t, vp]
    nbytes = out.numel() * out.element_size()
    row = out.shape[1] * out.element_size()
    ptr, sp = vp(out.data_ptr()), vp(stream.cuda_stream)
    shapes = {
        "memset": lambda: lib.xg_probe_memset(ptr, nbytes, sp),
        "rows_stg64_4w_cap4": lambda: lib.xg_probe_rows(ptr, nbytes, row, 8, 4, 4, sp),
        "rows_stg128_4w_cap4": lambda: lib.xg_probe_rows(ptr, nbytes, row, 16, 4, 4, sp),
        "rows_stg256_4w_cap4": lambda: lib.xg_probe_rows(ptr, nbytes, row, 32, 4, 4, sp),
        "rows_stg64_4w_cap2": lambda: lib.xg_probe_rows(ptr, nbytes, row, 8, 4, 2, sp),
        "rows_stg128_8w_nocap": lambda: lib.xg_probe_rows(ptr, nbytes, row, 16, 8, 0, sp),
        "gridstride_stg128": lambda: lib.xg_probe_gridstride(ptr, nbytes, sp),
    }
    return shapes


def write_ceiling(out, stream, reps: int = 5) -> dict:
    """Write-only HBM ceilings on the same buffer, same run: the best of
    `reps` timed passes of every probe_shapes() pattern, GB/s."""
    import torch

    nbytes = out.numel() * out.element_size()
    shapes = probe_shapes(out, stream)
    res = {}
    for name, fn in shapes.items():
        for _ in range(3):
            fn()
        best = float("inf")
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rc = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if rc:
                break
            best = min(best, e0.elapsed_time(e1))
        if best < float("inf"):
            res[name] = nbytes / (best / 1e3) / 1e9
    return res


def make_step(wl, ens, count, per, world, local):
    """The step function and its buffers."""
    import torch

    dev = f"cuda:{local}"
    ctx = {"out": None, "hits": None}
    if wl in ("fill_u32", "fill_2p34", "stream1"):
        out = ctx["out"] = torch.empty((count, per), dtype=torch.uint32, device=dev)
        fn = lambda: ens.fill_u32(per, out=out)  # noqa: E731
    elif wl == "fill_f32":
        out = ctx["out"] = torch.empty((count, per), dtype=torch.float32, device=dev)
        fn = lambda: ens.fill_f32(per, out=out)  # noqa: E731
    elif wl == "fill_f64":
        out = ctx["out"] = torch.empty((count, per), dtype=torch.float64, device=dev)
        fn = lambda: ens.fill_f64(per, out=out)  # noqa: E731
    elif wl == "skip":  # generator core only (no stores): the integer-issue ceiling
        fn = lambda: ens.skip(per)  # noqa: E731
    elif wl == "lc":
        hits = ctx["hits"] = torch.zeros(1001, dtype=torch.int64, device=dev)
        fn = lambda: ens.linear_complexity_test(1000, per, hist=hits)  # noqa: E731
    elif wl == "rank":
        hits = ctx["hits"] = torch.zeros(3, dtype=torch.int64, device=dev)
        fn = lambda: ens.rank_test(per, counts=hits)  # noqa: E731
    else:  # mc_pi: per-rank hits, then the job's one collective, inside the step
        hits = ctx["hits"] = torch.zeros(1, dtype=torch.int64, device=dev)
        total = ctx["total"] = torch.zeros(1, dtype=torch.int64, device=dev)
        import torch.distributed as dist

        if dist.is_initialized():
            def fn():
                hits.zero_()
                ens.mc_pi(per, hits=hits)
                total.copy_(hits)
                dist.all_reduce(total)  # NCCL uint64 sum over the job, every step (N = 1: one rank)
        else:
            def fn():
                hits.zero_()
                ens.mc_pi(per, hits=hits)
                total.copy_(hits)
    return fn, ctx


def alu_ceiling(wl: str, sm_mhz, sms: int):
    """Integer-pipe ceiling of an in-register workload: ALU warp-instructions
    per word from the committed ncu capture (sm__inst_executed_pipe_alu.sum /
    words of that launch) at the measured 2 ALU warp-instructions per SM per
    clock (profiles/README.md, micro-benchmark) and the live SM clock."""
    n = load_ncu(wl)
    per_word = n.get("alu_warp_inst_per_word")
    if not per_word or not sm_mhz:
        return None, n
    return 2.0 * sms * sm_mhz * 1e6 / per_word, n


def run_workload(wl, steps, warmup, world, rank, local, hbm_peak, peak_src):
    """Time one workload; returns (entry dict, step fn, ctx, ensemble)."""
    import torch

    import paper_1108_0486_b200 as xg

    stream = torch.cuda.current_stream()
    p = xg.xorgensgp32_params()
    first, count, per, scaling, job_words = workload_geometry(wl, world, rank)
    ens = xg.BlockEnsemble(p, 1, count, 63, first_stream=first, device=local)
    fn, ctx = make_step(wl, ens, count, per, world, local)
    with ClockSampler(local) as clk:
        total_ms, step_ms, launches = timed_loop(fn, stream, steps, warmup, world,
                                                 counter=xg.kernel_launches)
    t_max = max_over_ranks(total_ms, world)
    value = job_words * steps / (t_max / 1e3)
    kern_ms = statistics.mean(step_ms)
    clocks = clk.summary()
    entry = {"metric": METRIC, "value": value, "unit": "RN/s", "n_gpus": world, "steps": steps,
             "warmup": warmup, "ms_per_step": t_max / steps, "scaling": scaling,
             "dtype": {"fill_f32": "u32->f32", "fill_f64": "u32->f64"}.get(wl, "u32"),
             "config": config_for(wl, world), "gpu_launches": launches, "clocks": clocks,
             "step_ms_median": statistics.median(step_ms), "step_ms_min": min(step_ms),
             "step_ms_cv": (statistics.pstdev(step_ms) / kern_ms) if len(step_ms) > 1 else 0.0}
    vals = count * per
    if wl in BYTES_PER_VAL and wl != "stream1":
        # algorithmic bytes of the launch: output + the 129-word state read and
        # written back per stream
        alg = vals * BYTES_PER_VAL[wl] + 2 * count * 129 * 4
        achieved = alg / (kern_ms / 1e3) / 1e9
        entry["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                             "frac": achieved / hbm_peak,
                             "traffic": load_ncu(wl).get("dram_bytes_per_launch"),
                             "peak_source": peak_src, "alg_bytes_per_launch": alg,
                             "kernel_ms_mean": kern_ms, "kernel_ms_min": min(step_ms),
                             "kernel": "pair_kernel<GP32, %s>" % {"fill_f32": "kF32",
                                                                 "fill_f64": "kF64"}.get(wl, "kU32")}
    elif wl == "stream1":
        # the whole step (jump products + segment fills) against the HBM
        # roofline of its 4 B/word output
        achieved = vals * 4 / (kern_ms / 1e3) / 1e9
        entry["roofline"] = {"bound": "hbm (one stream as jump-ahead segments; step includes the "
                                      "GF(2) products)", "achieved": achieved, "peak": hbm_peak,
                             "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": None,
                             "peak_source": peak_src, "kernel_ms_mean": kern_ms}
    else:
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        ceil, n = alu_ceiling(wl, clocks.get("sm_mhz"), sms)
        words_per_gpu_s = vals * WORDS_PER_VAL.get(wl, 1) / (kern_ms / 1e3)
        entry["roofline"] = {
            "bound": "alu-pipe (integer, in-register)", "achieved": words_per_gpu_s,
            "peak": ceil, "unit": "RN/s per GPU", "frac": (words_per_gpu_s / ceil) if ceil else None,
            "traffic": n.get("dram_bytes_per_launch"),
            "peak_model": "2 ALU warp-instr/SM/clk x SMs x live SM clock / ALU warp-instr per word "
                          f"({n.get('alu_warp_inst_per_word')}, ncu)",
            "alu_pipe_pct_ncu": n.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct_ncu": n.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "kernel_ms_mean": kern_ms}
    if wl == "mc_pi":
        total = int(ctx["total"].item())
        samples_last = (1 << 40)
        entry["mc"] = {"hits_last_step": total, "samples_per_step": samples_last,
                       "pi_estimate": 4.0 * total / samples_last,
                       "abs_err_over_sigma": abs(4.0 * total / samples_last - 3.141592653589793)
                       / (4.0 * (0.7853981633974483 * 0.2146018366025517 / samples_last) ** 0.5),
                       "allreduce_in_step": _dist_ready(),
                       "allreduce": (f"torch.distributed all_reduce (NCCL, {world} rank"
                                     f"{'s' if world > 1 else ''}) of the uint64 hit count"
                                     if _dist_ready() else None)}
    return entry, fn, ctx, ens


# --------------------------------------------------------------------------
# CPU baselines (rank 0, N = 1) and the reference arm: the reference's own
# code (oracle/_ref) on the host cores.
# --------------------------------------------------------------------------

def _host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_generate_rate(streams: int, per_block: int, trials: int, warmup: int = 1,
                            budget_s: float = 60.0, min_trials: int = 3):
    """BlockEnsemble(p, 1, streams, 63).generate(per_block) on all host
    threads, wall clock around generate() as measure_ensemble_throughput
    (proj/src/bench.cpp:95-112)."""
    from oracle import REF_SO, Oracle, Reference

    threads = _host_threads()
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
    med = statistics.median(rates)
    return {"value": med, "unit": "RN/s", "cores": threads, "kind": kind,
            "sample": f"BlockEnsemble(xorgensgp32, base_seed=1, blocks={streams}, lanes=63)"
                      f".generate({per_block}) = {streams * per_block} words per trial (the full "
                      f"config), {len(rates)} trials after {warmup} warm-up, workers={threads}, "
                      f"wall clock around generate() (proj/src/bench.cpp:95-112); value = median",
            "cpu_model": cpu_model(), "trials": len(rates), "mean": statistics.mean(rates),
            "median": med, "min": min(rates), "max": max(rates),
            "cv": statistics.pstdev(rates) / statistics.mean(rates) if len(rates) > 1 else 0.0}


def _threaded(fn, first: int, count: int, piece: int):
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=_host_threads()) as ex:
        return list(ex.map(lambda f: fn(f, min(piece, first + count - f)),
                           range(first, first + count, piece)))


def cpu_baseline_for(wl: str) -> dict:
    """Bounded CPU samples of each workload on all host threads."""
    from oracle import Oracle, Reference

    threads = _host_threads()
    o = Oracle()
    p = o.gp32()
    if wl == "fill_u32":
        cb = reference_generate_rate(CHUNK, 1 << 16, trials=10, warmup=1, budget_s=25.0)
        try:
            cb["serial_1core_rn_per_s"] = Reference().serial_rate(1, 10**8, 20)
            cb["serial_sample"] = ("XorgensState(xorgensgp32, 1): 10^8 next_word, best chunk of 20 "
                                   "(measure_throughput, proj/src/bench.cpp:67-93): config 1")
        except Exception:  # noqa: BLE001
            pass
        return cb
    ref = Reference()
    if wl in ("fill_f32", "fill_f64"):
        # The reference has no conversions: its XorgensState words + the same
        # conversion, per-stream loops on all threads.
        f64 = wl == "fill_f64"
        streams, per = 8192, 1 << 16
        t = time.perf_counter()
        _threaded(lambda f, c: ref.streams_convert(p, 1, f, c, per, f64), 0, streams, 64)
        dt = time.perf_counter() - t
        words = streams * per * (2 if f64 else 1)
        return {"value": words / dt, "unit": "RN/s", "cores": threads, "kind": "reference",
                "values_per_s": streams * per / dt, "cpu_model": cpu_model(),
                "sample": f"{streams} per-stream XorgensState loops (proj/src/xorgens.cpp) x {per} "
                          f"{wl[5:]} values (conversion of DESIGN.md section 3 on reference words; the "
                          f"reference has none), {threads} threads"}
    if wl == "fill_2p34":
        streams, per = 8192, 1 << 16
        t = time.perf_counter()
        _threaded(lambda f, c: ref.streams_xor(p, 1, f, c, per), 0, streams, 64)
        dt = time.perf_counter() - t
        return {"value": streams * per / dt, "unit": "RN/s", "cores": threads, "kind": "reference",
                "cpu_model": cpu_model(),
                "sample": f"{streams} per-stream XorgensState loops (proj/src/xorgens.cpp) of the "
                          f"2^34 config's streams x {per} words, {threads} threads "
                          "(BASELINE.md: generate() would need 128 GiB)"}
    if wl == "mc_pi":
        streams, spp = 8192, 1 << 15
        t = time.perf_counter()
        parts = _threaded(lambda f, c: ref.stream_digests(p, 1, f, c, 0, 0, spp)["mc"], 0, streams, 64)
        dt = time.perf_counter() - t
        hits = int(sum(int(x.sum()) for x in parts))
        return {"value": 2 * streams * spp / dt, "unit": "RN/s", "cores": threads,
                "kind": "reference", "cpu_model": cpu_model(),
                "samples_per_s": streams * spp / dt, "hits": hits,
                "sample": f"reference XorgensState words of {streams} streams x {spp} samples + "
                          f"the exact integer predicate, {threads} threads (reduced N)"}
    if wl == "stream1":
        return {"value": Reference().serial_rate(1, 10**8, 20), "unit": "RN/s", "cores": 1,
                "kind": "reference", "cpu_model": cpu_model(),
                "sample": "XorgensState(xorgensgp32, 1): 10^8 next_word in 20 chunks, best "
                          "chunk rate (measure_throughput, proj/src/bench.cpp:67-93)"}
    return {"value": None, "unavailable": f"no CPU baseline for {wl}"}


def run_reference_arm(args):
    # under torchrun: WORLD_SIZE ranks, rank 0 measures; without it the job
    # size is --gpus (the host-side reference does not depend on it)
    world = int(os.environ.get("WORLD_SIZE", str(max(1, args.gpus))))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # The exact per-GPU config of our arm: 2^14 streams x 2^16 words per
    # generate() (8 GiB of vector<uint64_t>).
    base = reference_generate_rate(CHUNK, 1 << 16, trials=max(1, args.steps), warmup=args.warmup,
                                   budget_s=150.0)
    v = base["value"]
    line = {
        "impl": "reference", "metric": METRIC,
        "value": v, "unit": "RN/s", "n_gpus": world, "steps": base["trials"], "warmup": args.warmup,
        "ms_per_step": CHUNK * (1 << 16) / v * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator state; no input data)",
        "config": config_for("fill_u32", world),
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                              "median", "mean", "cv", "min", "max", "trials")},
        "e2e": {"value": v, "unit": "RN/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def sustained(fn, stream, seconds: float, world: int, local: int, words_per_step: int,
              ms_per_step: float, out=None) -> dict:
    """The same step back to back for ~`seconds` (power-capped steady state),
    timed with CUDA events, max over ranks; clocks sampled throughout.  The
    step count comes from the burst timing (max over ranks), so every rank
    runs the same number of steps."""
    import torch

    steps = max(100, int(seconds * 1e3 / max(ms_per_step, 1e-3)) // 100 * 100)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            fn()
            if i % 1000 == 999:
                torch.cuda.synchronize()  # bound the launch queue
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    res = {"value": words_per_step * steps / (ms / 1e3), "steps": steps, "ms_per_step": ms / steps,
           "clocks": clk.summary()}
    if out is not None:
        # the write-only ceilings under the same sustained load: memset (copy
        # engine, no SM work) and the fill's store shape without the generator
        nbytes = out.numel() * out.element_size()
        res["write_ceiling_sustained_gbs"] = {}
        try:
            shapes = probe_shapes(out, stream)
        except OSError:
            shapes = {}
        for name in ("memset", "rows_stg64_4w_cap4"):
            if name not in shapes:
                continue
            fn_w = shapes[name]
            with ClockSampler(local) as wclk:
                torch.cuda.synchronize()
                w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                w0.record(stream)
                for i in range(steps):
                    fn_w()
                    if i % 1000 == 999:
                        torch.cuda.synchronize()
                w1.record(stream)
                torch.cuda.synchronize()
            wms = w0.elapsed_time(w1)
            res["write_ceiling_sustained_gbs"][name] = {
                "gbs": nbytes * steps / (wms / 1e3) / 1e9, "clocks": wclk.summary()}
        best = max((v["gbs"] for v in res["write_ceiling_sustained_gbs"].values()), default=None)
        if best:
            res["frac_vs_write_ceiling_sustained"] = (
                words_per_step / max(world, 1) * out.element_size() * steps / (ms / 1e3) / 1e9 / best)
    return res


def host_api_bench(cb: dict) -> dict:
    """The reference's two host-side methods over the C++ drop-in
    (paper_1108_0486_b200/tools/xg_hostbench.cpp): measure_throughput through
    xg::gpu::XorgensSource (WordSource::next per word) and
    measure_ensemble_throughput through xg::gpu::BlockEnsemble::generate
    (vector<vector<uint64_t>>, 2^14 blocks x 2^16), next to the reference's
    own numbers on the same host (cpu_baseline)."""
    exe = os.path.join(ROOT, "paper_1108_0486_b200", "lib", "xg_hostbench")
    try:
        r = subprocess.run([exe, str(10**8), "5", str(CHUNK), str(1 << 30)], capture_output=True,
                           text=True, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        return {"unavailable": str(e)}
    d["reference"] = {
        "measure_throughput_rn_per_s": cb.get("serial_1core_rn_per_s"),
        "measure_ensemble_throughput_rn_per_s": cb.get("value"),
        "source": "cpu_baseline (oracle/_ref: XorgensState::next_word serial best-chunk rate; "
                  "BlockEnsemble::generate on all host threads)"}
    return d


def extra_e2e(wl: str, ens, fn, ctx, world: int, rank: int) -> dict:
    """End to end through the public API for the extra workloads: the f32 /
    f64 fills into pinned host memory (xg_generate_host_f32/f64: device fill
    + PCIe copy inside the timed region); MC with the job's hit count read
    back to the host every step.  The 2^34 fill would need 64 GiB of host
    memory per job and is not copied."""
    import torch

    first, count, per, _, job_words = workload_geometry(wl, world, rank)
    if wl in ("fill_f32", "fill_f64"):
        dt_ = torch.float32 if wl == "fill_f32" else torch.float64
        host = torch.empty((count, per), dtype=dt_, pin_memory=True)
        call = ens.generate_f32_into_host if wl == "fill_f32" else ens.generate_f64_into_host
        call(per, host)
        barrier(world)
        t = time.perf_counter()
        steps = 3
        for _ in range(steps):
            call(per, host)
        dt = max_over_ranks(time.perf_counter() - t, world)
        nbytes = host.numel() * host.element_size()
        del host
        return {"value": job_words * steps / dt, "unit": "RN/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": nbytes, "steps": steps,
                "api": f"BlockEnsemble.generate_{wl[5:]}_into_host -> xg_generate_host_{wl[5:]} "
                       "(pinned host buffer)"}
    if wl == "mc_pi":
        barrier(world)
        t = time.perf_counter()
        steps = 2
        for _ in range(steps):
            fn()
            int(ctx["total"].item())  # the job's hit count on the host
        dt = max_over_ranks(time.perf_counter() - t, world)
        return {"value": job_words * steps / dt, "unit": "RN/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 8, "steps": steps,
                "api": "BlockEnsemble.mc_pi (+ NCCL all-reduce at N > 1) -> hit count read back"}
    if wl == "stream1":
        # ONE generator's 10^8 words into pinned host memory (what a user of
        # the reference's XorgensState loop gets), jump-ahead on the device
        host = torch.empty((count, per), dtype=torch.uint32, pin_memory=True)
        ens.generate_into_host(per, host)
        barrier(world)
        t = time.perf_counter()
        steps = 3
        for _ in range(steps):
            ens.generate_into_host(per, host)
        dt = max_over_ranks(time.perf_counter() - t, world)
        del host
        return {"value": job_words * steps / dt, "unit": "RN/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": count * per * 4, "steps": steps,
                "api": "XorgensState stream -> BlockEnsemble.generate -> xg_generate_host (pinned host "
                       "buffer; one stream, jump-ahead segments)"}
    return {"value": None, "why": "the 2^34-word output (64 GiB per job) is not copied to the host"}


def dry_run(args) -> int:
    """CPU-only check of the N-rank plumbing (gloo): world, ranks, slices."""
    world, rank, _ = dist_setup(dry=True)
    geo = {wl: workload_geometry(wl, world, rank) for wl in ("fill_u32", "fill_2p34", "mc_pi")}
    t = max_over_ranks(float(rank + 1), world)
    if world > 1:
        import torch.distributed as dist

        g = [None] * world
        dist.all_gather_object(g, geo)
    else:
        g = [geo]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_requested": args.gpus,
                          "max_over_ranks": t, "comm": comm_info(world), "slices": g}), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0 if world == args.gpus else 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="GPUs in the job; N > 1 runs one rank per GPU (self-launched under "
                         "torch.distributed.run when WORLD_SIZE is unset)")
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 200 for fills, 5 for mc_pi)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="fill_u32", choices=WORKLOADS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra_workloads block")
    ap.add_argument("--sustained-s", type=float, default=3.0,
                    help="seconds of back-to-back steps for the sustained rate (0 = skip)")
    ap.add_argument("--dry-run", action="store_true", help="CPU-only check of the N-rank plumbing")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.steps is None:
        args.steps = 5 if args.workload == "mc_pi" else (10 if args.impl == "reference" else 200)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.dry_run:
        return dry_run(args)

    import torch

    import paper_1108_0486_b200 as xg

    world, rank, local = dist_setup()
    if args.gpus != world:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    stream = torch.cuda.current_stream()
    wl = args.workload
    hbm_peak, peak_src = load_peaks()

    entry, fn, ctx, ens = run_workload(wl, args.steps, args.warmup, world, rank, local, hbm_peak,
                                       peak_src)
    first, count, per, _, job_words = workload_geometry(wl, world, rank)
    result = {"metric": METRIC, "value": entry.pop("value"), "unit": "RN/s", "n_gpus": world,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": entry.pop("ms_per_step"),
              "higher_is_better": True, "scaling": entry.pop("scaling"), "vs_baseline": None,
              "dtype": entry.pop("dtype"), "data": "synthetic (seeded generator state; no input data)",
              "config": entry.pop("config"), "gpu_launches": entry.pop("gpu_launches"),
              "clocks": entry.pop("clocks"), "roofline": entry.pop("roofline"),
              "comm": comm_info(world), "host_cpu": cpu_model()}
    for k in ("step_ms_median", "step_ms_min", "step_ms_cv", "mc"):
        if k in entry:
            result[k] = entry[k]
    out = ctx.get("out")
    if out is not None and wl in ("fill_u32", "fill_f32", "fill_f64", "fill_2p34"):
        try:
            wc = write_ceiling(out, stream)
            best = max(wc.values())
            ach = result["roofline"]["achieved"]
            result["roofline"].update({"write_ceiling_gbs": best, "frac_vs_write_ceiling": ach / best,
                                       "write_probes_gbs": wc})
        except OSError:
            pass
    if wl == "fill_u32" and args.sustained_s > 0:
        result["sustained"] = sustained(fn, stream, args.sustained_s, world, local, job_words,
                                        result["ms_per_step"], out=ctx.get("out"))
    # e2e through the public host API (generate into pinned host memory)
    if not args.no_e2e and wl in ("fill_u32", "stream1"):
        # (stream1: ONE generator's 10^8 words into host memory -- the
        # reference's XorgensSource loop, served by the jump-ahead path)
        host = torch.empty((count, per), dtype=torch.uint32, pin_memory=True)
        e2e_steps = max(3, min(args.steps, 5))
        ens.generate_into_host(per, host)
        barrier(world)
        t = time.perf_counter()
        for _ in range(e2e_steps):
            ens.generate_into_host(per, host)
        dt = max_over_ranks(time.perf_counter() - t, world)
        result["e2e"] = {"value": count * per * world * e2e_steps / dt, "unit": "RN/s",
                         "h2d_bytes_per_step": 0, "d2h_bytes_per_step": count * per * 4,
                         "api": "BlockEnsemble.generate -> xg_generate_host (pinned host buffer)",
                         "steps": e2e_steps}
        del host
    result["parity"] = parity_check(wl, world, rank, local, out=out)
    del ens, ctx, fn, out
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            result["cpu_baseline"] = cpu_baseline_for(wl)
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unavailable": str(e)}

    if rank == 0 and world == 1 and wl == "fill_u32" and not args.no_e2e:
        result["e2e_host_api"] = host_api_bench(result.get("cpu_baseline", {}))

    if wl == "fill_u32" and not args.no_extra:
        extras = {}
        for xw in EXTRA:
            steps = min(args.steps, 5) if xw == "mc_pi" else args.steps
            e, xfn, xctx, xens = run_workload(xw, steps, args.warmup, world, rank, local, hbm_peak,
                                              peak_src)
            if not args.no_e2e:
                e["e2e"] = extra_e2e(xw, xens, xfn, xctx, world, rank)
            xout = xctx.get("out")
            if xout is not None:
                try:
                    wc = write_ceiling(xout, stream)
                    e["roofline"]["write_ceiling_gbs"] = max(wc.values())
                    e["roofline"]["frac_vs_write_ceiling"] = (e["roofline"]["achieved"] /
                                                              max(wc.values()))
                except OSError:
                    pass
            e["parity"] = parity_check(xw, world, rank, local, out=xout)
            del xctx, xens, xout, xfn
            torch.cuda.empty_cache()
            if rank == 0 and world == 1 and not args.no_cpu:
                try:
                    e["cpu_baseline"] = cpu_baseline_for(xw)
                except Exception as ex:  # noqa: BLE001
                    e["cpu_baseline"] = {"value": None, "unavailable": str(ex)}
            e.pop("metric", None)
            extras[xw] = e
        result["extra_workloads"] = extras
        result["gpu_launches_all"] = result["gpu_launches"] + sum(
            e["gpu_launches"] for e in extras.values())
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()
    forward_nccl_log()
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

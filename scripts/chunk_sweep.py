#!/usr/bin/env python3
"""Throughput of the generation kernels vs ensemble size P (A/B aid for the
chunk-lane kernel's geometry).  CUDA-event timing on the launching stream,
warm-up first; RN/s = P * words / time.

usage: python scripts/chunk_sweep.py TAG [workloads] [P list]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1108_0486_b200 as xg  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "?"
wls = (sys.argv[2] if len(sys.argv) > 2 else "mc,skip,fill_u32,fill_f32,fill_f64").split(",")
Ps = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else
                       "16384,18944,37888,65536,131072").split(",")]
p = xg.xorgensgp32_params()
s = torch.cuda.current_stream()


def timeit(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for wl in wls:
    for P in Ps:
        e = xg.BlockEnsemble(p, 1, P, 63)
        if wl == "mc":
            words = max(64, (1 << 38) // P // 64 * 64)
            hits = torch.zeros(1, dtype=torch.int64, device="cuda")
            fn = lambda: e.mc_pi(words // 2, hits=hits)  # noqa: E731
            reps = 3
        elif wl == "skip":
            words = max(64, (1 << 32) // P // 64 * 64)
            fn = lambda: e.skip(words)  # noqa: E731
            reps = 20
        else:
            words = max(64, (1 << 30) // P // 64 * 64)
            dt = {"fill_u32": torch.uint32, "fill_f32": torch.float32, "fill_f64": torch.float64}[wl]
            vals = words // 2 if wl == "fill_f64" else words
            out = torch.empty((P, vals), dtype=dt, device="cuda")
            f = getattr(e, wl)
            fn = lambda: f(vals, out=out)  # noqa: E731
            reps = 20
        ms = timeit(fn, reps)
        print(json.dumps({"tag": tag, "wl": wl, "P": P, "words": words, "ms": round(ms, 4),
                          "rn_s": P * words / ms * 1e3}), flush=True)
        del e
        torch.cuda.empty_cache()

#!/usr/bin/env python3
"""Fill rate versus ensemble size P (streams): one warp per stream, so small
ensembles are latency-bound.  Prints one JSON line per P (CUDA events on the
launching stream, best of 5 after 2 warm-ups).  XG_CTA8=1 forces 8-stream
CTAs (the sizing before small ensembles were spread over the SMs)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0486_b200 as xg  # noqa: E402

p = xg.xorgensgp32_params()
for P in (1, 8, 64, 148, 296, 512, 600, 700, 1184, 2048, 4096, 9472, 16384):
    per = 1 << 20 if P <= 256 else max(1 << 16, (1 << 28) // P)
    per -= per % 128
    e = xg.BlockEnsemble(p, 1, P, 63)
    out = torch.empty((P, per), dtype=torch.uint32, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(2):
        e.fill_u32(per, out=out)
    best = None
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        e.fill_u32(per, out=out)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    print(json.dumps({"streams": P, "per_stream": per, "ms": best,
                      "rn_per_s": P * per / (best / 1e3),
                      "per_stream_rn_per_s": per / (best / 1e3),
                      "cta8": bool(os.environ.get("XG_CTA8"))}), flush=True)
    del out, e

#!/usr/bin/env python3
"""u32 fill rate versus stream count P at a fixed 2^30 words per launch
(per_stream = 2^30 / P): how the number of concurrent write streams and the
wave structure affect the HBM-bound fill.  Best and mean of 20 launches."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0486_b200 as xg  # noqa: E402

p = xg.xorgensgp32_params()
total = 1 << 30
for P in [int(a) for a in (sys.argv[1:] or
          (592, 1184, 2368, 4096, 4736, 8192, 9472, 11840, 14208, 16384, 18944, 32768, 65536))]:
    per = (total // P) // 128 * 128
    e = xg.BlockEnsemble(p, 1, P, 63)
    out = torch.empty((P, per), dtype=torch.uint32, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):
        e.fill_u32(per, out=out)
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        e.fill_u32(per, out=out)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"P": P, "per": per, "best_ms": min(ts), "mean_ms": statistics.mean(ts),
                      "rn_per_s_best": P * per / min(ts) * 1e3,
                      "rn_per_s_mean": P * per / statistics.mean(ts) * 1e3}), flush=True)
    del out, e

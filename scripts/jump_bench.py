#!/usr/bin/env python3
"""One-stream fill rate with the jump-ahead path (csrc/xg_jump.cuh) against
the same stream on one warp (a 2-stream ensemble takes the direct path;
its rate / 2 is one warp's), plus the one-time cost of the G^(2^i) powers
and O(log n) skips.  CUDA events on the launching stream; not product."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0486_b200 as xg  # noqa: E402

p = xg.xorgensgp32_params()
s = torch.cuda.current_stream()


def timed(fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {}
e = xg.BlockEnsemble(p, 1, 1, 63)
t0 = time.perf_counter()
e.fill_u32(1 << 20)
torch.cuda.synchronize()
res["first_call_ms (G^(2^i) for i <= 26 + one fill)"] = (time.perf_counter() - t0) * 1e3
for n in [1 << 20, 1 << 22, 10**8, 1 << 28, 1 << 30]:
    out = torch.empty((1, n), dtype=torch.uint32, device="cuda")
    e.fill_u32(n, out=out)
    reps = 20 if n <= 1 << 28 else 10
    ms = timed(lambda: e.fill_u32(n, out=out), reps)
    res[f"jump_fill_u32 n={n}"] = {"ms": ms, "rn_per_s": n / (ms / 1e3)}
    del out
# one warp per stream (the direct path): 513 streams (more than the jump
# paths take), per-stream rate
d = xg.BlockEnsemble(p, 1, 513, 63)
n = 1 << 18
out = torch.empty((513, n), dtype=torch.uint32, device="cuda")
d.fill_u32(n, out=out)
ms = timed(lambda: d.fill_u32(n, out=out), 5)
res["direct one warp (513 streams x 2^18, per stream)"] = {"ms": ms, "rn_per_s": n / (ms / 1e3)}
# a batch skip: 2^14 streams jump 2^22 words (generating them: ~25 ms)
b = xg.BlockEnsemble(p, 1, 1 << 14, 63)
b.skip(1 << 22)
res["skip(2^22) of 2^14 streams (batch jump), ms"] = timed(lambda: b.skip(1 << 22), 5)
del out
f = xg.BlockEnsemble(p, 1, 1, 63)
t0 = time.perf_counter()
f.skip(1 << 62)
torch.cuda.synchronize()
res["first skip(2^62) incl. powers up to 2^62, ms"] = (time.perf_counter() - t0) * 1e3
ms = timed(lambda: f.skip((1 << 62) - 1), 5)
res["skip(2^62 - 1) (62 products), ms"] = ms
ms = timed(lambda: f.skip(1 << 40), 10)
res["skip(2^40) (1 product), ms"] = ms
print(json.dumps(res, indent=1))

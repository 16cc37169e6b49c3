#!/usr/bin/env python3
"""Kernel launch list of one-stream jump fills (run under ncu --metrics
gpu__time_duration.sum): the per-level GF(2) products, the Weyl kernel and
the segment fills.  Not product."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0486_b200 as xg  # noqa: E402
p = xg.xorgensgp32_params()
e = xg.BlockEnsemble(p, 1, 1, 63)
for n in [int(a) for a in sys.argv[1:]] or [1 << 20, 10**8]:
    out = torch.empty((1, n), dtype=torch.uint32, device="cuda")
    e.fill_u32(n, out=out)  # powers computed here
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"n={n}")
    e.fill_u32(n, out=out)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()

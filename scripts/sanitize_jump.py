#!/usr/bin/env python3
"""The many-stream jump paths for compute-sanitizer memcheck / synccheck
(racecheck: the shared-memory GF(2) kernels are covered by sanitize_smoke.py;
the squarings of the powers take hours under racecheck): jump_fill_many
(power-of-two and odd lengths, remainders on the side stream), batch skips.
Checks results against the oracle too."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0486_b200 as xg  # noqa: E402
from oracle import Oracle  # noqa: E402

o = Oracle()
p = xg.xorgensgp32_params()
M = 1 << 20
for P, n in ((8, M), (100, 2 * M), (5, M + 3), (300, (1 << 18) + 77)):
    e = xg.BlockEnsemble(p, 11, P, 63)
    oe = o.ensemble(11, P)
    assert np.array_equal(e.fill_u32(n).cpu().numpy(), oe.fill_u32(n))
    assert np.array_equal(e.fill_u32(64).cpu().numpy(), oe.fill_u32(64))
e = xg.BlockEnsemble(p, 12, 3, 63)
oe = o.ensemble(12, 3)
assert np.array_equal(e.fill_f64(M + 5).cpu().numpy().view(np.uint64), oe.fill_f64(M + 5).view(np.uint64))
e.skip(M + 1)
oe.fill_u32(M + 1)
assert np.array_equal(e.fill_u32(64).cpu().numpy(), oe.fill_u32(64))
torch.cuda.synchronize()
print("sanitize jump many-stream ok")

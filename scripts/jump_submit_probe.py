#!/usr/bin/env python3
"""Is a one-stream jump fill (10^8 words) bound by the host's launch
submission or by the device?  CPU time to enqueue a call against the device
time per call (s5i: 47 us submitted, 143 us on the device -- device-bound, so
CUDA-graph replay would only trim the inter-kernel gaps).  Not product."""
import time, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1108_0486_b200 as xg
p = xg.xorgensgp32_params()
e = xg.BlockEnsemble(p, 1, 1, 63)
n = 10**8
out = torch.empty((1, n), dtype=torch.uint32, device="cuda")
for _ in range(3): e.fill_u32(n, out=out)
torch.cuda.synchronize()
# CPU submission time per call: enqueue many calls back to back (no sync)
reps = 50
t = time.perf_counter()
for _ in range(reps): e.fill_u32(n, out=out)
t_sub = (time.perf_counter() - t) / reps
torch.cuda.synchronize()
t_all = (time.perf_counter() - t) / reps
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); [e.fill_u32(n, out=out) for _ in range(reps)]; b.record(); torch.cuda.synchronize()
print(f"cpu submit per call {t_sub*1e6:.1f} us; wall per call {t_all*1e6:.1f} us; gpu per call {a.elapsed_time(b)/reps*1e3:.1f} us")
# with a big queue ahead (GPU busy), does the GPU time per call shrink?
big = xg.BlockEnsemble(p, 1, 16384, 63); bo = torch.empty((16384, 1<<16), dtype=torch.uint32, device="cuda")
torch.cuda.synchronize()
a.record()
for _ in range(reps): e.fill_u32(n, out=out)
b.record(); torch.cuda.synchronize()
print("again", a.elapsed_time(b)/reps*1e3)

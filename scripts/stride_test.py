import json, os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1108_0486_b200 as xg
p = xg.xorgensgp32_params()
for P, per in ((2048, 131072), (2048, 131072 + 64), (9472, 65536), (9472, 65536 + 64), (9472, 65536 + 2048),
               (16384, 65536), (16384, 65536 + 64), (4096, 65536), (4096, 65536 + 64)):
    e = xg.BlockEnsemble(p, 1, P, 63)
    out = torch.empty((P, per), dtype=torch.uint32, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):
        e.fill_u32(per, out=out)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); e.fill_u32(per, out=out); b.record(s); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    best = min(ts)
    print(json.dumps({"P": P, "per": per, "best_ms": best, "rn_per_s": P * per / best * 1e3}), flush=True)
    del out, e

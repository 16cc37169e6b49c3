import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1108_0486_b200 as xg
for nbits, count in ((16384, 2048), (65536, 512)):
    w = (nbits + 31) // 32
    d = torch.randint(-2**31, 2**31 - 1, (count, w), dtype=torch.int32, device='cuda')
    xg.berlekamp_massey(d, nbits); torch.cuda.synchronize()
    t = time.perf_counter(); L = xg.berlekamp_massey(d, nbits); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"BM {nbits} bits x {count}: {dt*1e3:.1f} ms, {count/dt:.0f} seq/s, mean L {L.float().mean().item():.1f}")

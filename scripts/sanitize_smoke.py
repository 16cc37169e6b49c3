#!/usr/bin/env python3
"""Small calls through every kernel mode, for compute-sanitizer
(memcheck / racecheck / synccheck).  Checks results against the oracle too."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_0486_b200 as xg  # noqa: E402
from oracle import Oracle  # noqa: E402

o = Oracle()
p = xg.xorgensgp32_params()
for var_params in (p, xg.GeneratorParams(128, 95, 17, 12, 13, 15, 32, 2654435769, 16),
                   xg.GeneratorParams(128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11)):
    e = xg.BlockEnsemble(var_params, 3, 13, 32)
    oe = o.ensemble(3, 13, o.params(var_params.r, var_params.s, var_params.a, var_params.b,
                                    var_params.c, var_params.d, var_params.w, var_params.omega,
                                    var_params.gamma))
    for n in (1, 128, 130, 384, 515, 516, 1280):
        assert np.array_equal(e.fill_u32(n).cpu().numpy(), oe.fill_u32(n))
        assert np.array_equal(e.fill_f32(n).cpu().numpy().view(np.uint32), oe.fill_f32(n).view(np.uint32))
        assert np.array_equal(e.fill_f64(n).cpu().numpy().view(np.uint64), oe.fill_f64(n).view(np.uint64))
        assert np.array_equal(e.fill_raw_u32(n).cpu().numpy(), oe.fill_raw_u32(n))
        assert int(e.mc_pi(96).item()) == int(oe.mc_hits(96).sum())
    st = xg.XorgensState(var_params, 9)
    [st.next_word() for _ in range(50)]
    e.generate(300)
torch.cuda.synchronize()
print("sanitize smoke ok")

# statistical-test kernels (fused rank, Berlekamp-Massey both ways, counting kernels)
e = xg.BlockEnsemble(p, 5, 9, 63)
oe = o.ensemble(5, 9)
assert np.array_equal(e.rank_test(5).cpu().numpy().astype(np.uint64), oe.rank_counts(5).sum(axis=0))
h1 = e.linear_complexity_test(100, 40)
h2 = e.linear_complexity_test(2000, 38)
assert int(h1.sum()) == 9 * 40 and int(h2.sum()) == 9 * 38
seqs = torch.randint(-2**31, 2**31 - 1, (3, 160), dtype=torch.int32, device="cuda")
L = xg.berlekamp_massey(seqs, 5000)
assert all(2000 < int(v) < 3000 for v in L.tolist())
from paper_1108_0486_b200.battery import BatteryConfig, run_battery_gpu  # noqa: E402
rep = run_battery_gpu(p, 3, BatteryConfig.quick())
assert rep["num_tests"] == 5
print("sanitize stattests ok")

# round 2: the digest kernel, the next_word ring (past two slots, interleaved
# with a fill) and generate() into caller rows
from paper_1108_0486_b200.digest import row_digests  # noqa: E402
w = e.fill_u32(1000)
x, s, ws = row_digests(w)
ref = w.cpu().numpy()
assert np.array_equal(x, np.bitwise_xor.reduce(ref, axis=1))
st = xg.XorgensState(p, 77)
got = [st.next_word() for _ in range(70000)]
got += st.ensemble.fill_u32(333).cpu().numpy()[0].tolist()
got += [st.next_word() for _ in range(70000)]
assert np.array_equal(np.array(got, dtype=np.uint64), o.stream(77, len(got)))
import ctypes  # noqa: E402
rows = [np.zeros(777, dtype=np.uint64) for _ in range(9)]
arr = (ctypes.c_void_p * 9)(*[r.ctypes.data for r in rows])
e2 = xg.BlockEnsemble(p, 5, 9, 63)
assert xg._lib.lib.xg_generate_host_rows(e2.handle, 777, arr, None) == 0
assert np.array_equal(np.stack(rows), o.ensemble(5, 9).fill_u32(777).astype(np.uint64))
print("sanitize round-2 paths ok")

# generate() through host tiles (the C++ drop-in path) and the f32/f64 host generates
FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                      ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint)
seen = []
cb = FN(lambda ctx, s0, w0, ns, nw, tile, eb, part, parts: seen.append((s0, w0, ns, nw)) if part == 0 else None)
e3 = xg.BlockEnsemble(p, 6, 7, 63)
assert xg._lib.lib.xg_generate_host_tiles(e3.handle, 999, cb, None, 2, None) == 0 and seen
h32 = np.empty((7, 333), dtype=np.float32)
e3.generate_f32_into_host(333, h32)
h64 = np.empty((7, 200), dtype=np.float64)
e3.generate_f64_into_host(200, h64)
oe3 = o.ensemble(6, 7)
oe3.fill_u32(999)
assert np.array_equal(h32.view(np.uint32), oe3.fill_f32(333).view(np.uint32))
assert np.array_equal(h64.view(np.uint64), oe3.fill_f64(200).view(np.uint64))
w2 = torch.randint(0, 2**31, (64 * 9,), dtype=torch.int32, device="cuda")
cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
assert xg._lib.lib.xg_rank_words(w2.data_ptr(), 17, cnt.data_ptr(), None) == 0
hist = torch.zeros(129, dtype=torch.int64, device="cuda")
assert xg._lib.lib.xg_lc_words(w2.data_ptr(), w2.numel(), 128, 40, hist.data_ptr(), None) == 0
torch.cuda.synchronize()
assert int(cnt.sum()) == 17 and int(hist.sum()) == 40
print("sanitize round-2 host tiles / f32-f64 host / word-buffer tests ok")

# jump-ahead (csrc/xg_jump.cuh): one-stream fills >= 2^20 words (Krylov
# product, four-Russians and dense GF(2) kernels, side-stream last segment)
# on two parameter kinds (the 4096-row squarings of a jump skip are left to
# the parity tests: hours under racecheck)
for jp in (p, xg.GeneratorParams(128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11)):
    op = o.params(jp.r, jp.s, jp.a, jp.b, jp.c, jp.d, jp.w, jp.omega, jp.gamma)
    ej = xg.BlockEnsemble(jp, 21, 1, xg.lane_bound(jp))
    n = (1 << 20) + 4099
    assert np.array_equal(ej.fill_u32(n).cpu().numpy()[0], o.stream(21, n, op))
    assert np.array_equal(ej.fill_u32(64).cpu().numpy()[0], o.stream(21, n + 64, op)[-64:])
torch.cuda.synchronize()
print("sanitize jump-ahead ok")

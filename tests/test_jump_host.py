"""CPU checks of the jump-ahead mathematics (no GPU): the minimal polynomial
the library reduces x^n by (xg_jump_minpoly, host code of csrc/xg_gpu.cu)
against an independent Berlekamp-Massey here, and its defining property on
the oracle's raw stream: m(G) s = 0, i.e. the window 4096 raw words ahead is
the XOR of the windows k words ahead over the coefficients of m (Krylov form
of DESIGN.md section 4a)."""
import ctypes

import numpy as np
import pytest

import paper_1108_0486_b200 as xg
from paper_1108_0486_b200 import _lib
from oracle import Params

SETS = [
    (128, 65, 15, 14, 12, 17, 32, 2654435769, 16),   # xorgensgp32
    (128, 95, 17, 12, 13, 15, 32, 2654435769, 16),   # J = 1 runtime set
]
# a valid J = 2 set whose raw stream has linear complexity 4095 (not full
# period): no degree-4096 minimal polynomial, so its jumps take the doubling
# path with exact powers of G (tests/test_gpu_jump.py covers it on the GPU)
NOT_FULL = (128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11)


def minpoly(ps):
    out = (ctypes.c_uint64 * 64)()
    rc = _lib.lib.xg_jump_minpoly(ctypes.byref(_lib.xg_params_t(*ps)), out)
    return rc, np.array(list(out), dtype=np.uint64)


def bits_of(words64):
    return np.array([(int(words64[k // 64]) >> (k % 64)) & 1 for k in range(4096)], dtype=np.uint8)


def berlekamp_massey(b):
    n = len(b)
    c = np.zeros(n + 1, np.uint8)
    bb = np.zeros(n + 1, np.uint8)
    c[0] = bb[0] = 1
    L, m = 0, 1
    for i in range(n):
        d = b[i] ^ (int(np.bitwise_and(c[1:L + 1], b[i - 1::-1][:L]).sum()) & 1 if L else 0)
        if not d:
            m += 1
        elif 2 * L <= i:
            t = c.copy()
            c[m:] ^= bb[:n + 1 - m]
            L, bb, m = i + 1 - L, t, 1
        else:
            c[m:] ^= bb[:n + 1 - m]
            m += 1
    return L, c


@pytest.mark.parametrize("ps", SETS)
def test_minpoly_annihilates_the_raw_stream(oracle, ps):
    rc, m = minpoly(ps)
    assert rc == 0
    mk = bits_of(m)
    for seed in (1, 12345):
        raw = oracle.ensemble(seed, 1, Params(*ps)).fill_raw_u32(2 * 4096 + 200)[0]
        # windows of the raw run: s_i = raw[i .. i + 128); check s_{4096+t} for a few t
        for t in (0, 1, 77, 4000):
            acc = np.zeros(128, dtype=np.uint32)
            for k in np.nonzero(mk)[0]:
                acc ^= raw[t + k:t + k + 128]
            assert np.array_equal(acc, raw[t + 4096:t + 4096 + 128]), (seed, t)


def test_minpoly_equals_independent_berlekamp_massey(oracle):
    ps = SETS[0]
    rc, m = minpoly(ps)
    assert rc == 0
    raw = oracle.ensemble(3, 1, Params(*ps)).fill_raw_u32(2 * 4096)[0]
    L, c = berlekamp_massey((raw & 1).astype(np.uint8))
    assert L == 4096
    mk = bits_of(m)
    assert all(int(mk[k]) == int(c[L - k]) for k in range(4096))  # m_k = c_(L-k)


def test_minpoly_rejects_other_sets():
    tiny = xg.tiny_r2w8_params() if hasattr(xg, "tiny_r2w8_params") else None
    out = (ctypes.c_uint64 * 64)()
    if tiny is not None:
        assert _lib.lib.xg_jump_minpoly(ctypes.byref(tiny._c()), out) == _lib.XG_EUNSUPPORTED
    bad = _lib.xg_params_t(128, 64, 15, 14, 12, 17, 32, 2654435769, 16)  # gcd(r, s) != 1
    assert _lib.lib.xg_jump_minpoly(ctypes.byref(bad), out) == 3
    assert _lib.lib.xg_jump_minpoly(None, out) == _lib.XG_EINVAL


def test_set_without_full_degree_falls_back(oracle):
    rc, _ = minpoly(NOT_FULL)
    assert rc == _lib.XG_EUNSUPPORTED
    raw = oracle.ensemble(3, 1, Params(*NOT_FULL)).fill_raw_u32(2 * 4096)[0]
    assert berlekamp_massey((raw & 1).astype(np.uint8))[0] == 4095

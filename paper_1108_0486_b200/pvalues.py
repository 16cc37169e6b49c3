"""p-values exactly as the reference computes them (proj/src/stattests/pvalues.cpp):
the same series / continued-fraction code, so statistics computed from GPU
counts reproduce the reference's reports.  Host-side arithmetic only."""
from __future__ import annotations

import ctypes
import ctypes.util
import math

# std::lgamma is the C library's; CPython's math.lgamma is its own
# implementation and can differ in the last bit, so call libm directly.
_libm = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
_libm.lgamma.restype = ctypes.c_double
_libm.lgamma.argtypes = [ctypes.c_double]
_lgamma = _libm.lgamma

__all__ = ["regularized_gamma_p", "regularized_gamma_q", "chi_square_pvalue",
           "poisson_upper_tail"]


def _gamma_p_series(a: float, x: float) -> float:
    ap, s = a, 1.0 / a
    term = s
    for _ in range(10000):
        ap += 1.0
        term *= x / ap
        s += term
        if abs(term) < abs(s) * 1e-17:
            break
    return s * math.exp(-x + a * math.log(x) - _lgamma(a))


def _gamma_q_cf(a: float, x: float) -> float:
    tiny = 1e-300
    b = x + 1.0 - a
    c = 1.0 / tiny
    d = 1.0 / b
    h = d
    for i in range(1, 10000):
        an = -float(i) * (i - a)
        b += 2.0
        d = an * d + b
        if abs(d) < tiny:
            d = tiny
        c = b + an / c
        if abs(c) < tiny:
            c = tiny
        d = 1.0 / d
        delta = d * c
        h *= delta
        if abs(delta - 1.0) < 1e-17:
            break
    return h * math.exp(-x + a * math.log(x) - _lgamma(a))


def regularized_gamma_p(a: float, x: float) -> float:
    if x == 0.0:
        return 0.0
    return _gamma_p_series(a, x) if x < a + 1.0 else 1.0 - _gamma_q_cf(a, x)


def regularized_gamma_q(a: float, x: float) -> float:
    if x == 0.0:
        return 1.0
    return 1.0 - _gamma_p_series(a, x) if x < a + 1.0 else _gamma_q_cf(a, x)


def poisson_upper_tail(k: int, lam: float) -> float:
    return 1.0 if k == 0 else regularized_gamma_p(float(k), lam)


def chi_square_pvalue(stat: float, dof: int) -> float:
    """pvalues.cpp:67-73."""
    return regularized_gamma_q(dof / 2.0, stat / 2.0)

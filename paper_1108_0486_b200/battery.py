"""The reference's statistical battery (proj/src/stattests/battery.cpp:72-112)
run on the GPU over one generator stream.

Every test's counting runs on the device -- monobit / runs
(``xg_bits_ones_runs``), the 32 x 32 matrix-rank test (``xg_rank_test``,
fused into the generator), the linear complexity test
(``xg_linear_complexity_test``, one Berlekamp-Massey per block and warp) and
birthday spacings (``xg_birthday_duplicates``, a block radix sort per round)
-- and only the integer results come back; the statistics, p-values and
verdicts are then computed exactly as proj/src/stattests/tests.cpp and
pvalues.cpp compute them.  The stream is consumed in the reference's order
and amounts (a fresh BitSource per bit test, so a test that ends inside a
word drops the rest of that word), so the report equals the reference's
``run_battery`` over the same words test for test.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Dict, List

from ._lib import lib
from .pvalues import poisson_upper_tail, regularized_gamma_p, regularized_gamma_q  # noqa: F401
from .xorgens import (BlockEnsemble, GeneratorParams, UnsupportedParamsError, _raise, _torch,
                      fast_path, lane_bound, linear_complexity_statistic, matrix_rank_statistic)

__all__ = ["BatteryConfig", "run_battery_gpu", "regularized_gamma_p", "regularized_gamma_q"]


@dataclass
class BatteryConfig:
    """proj/include/xg/stattests/battery.hpp:15-34 (defaults) and
    battery.cpp:11-20 (quick)."""

    run_monobit: bool = True
    run_runs: bool = True
    run_matrix_rank: bool = True
    run_linear_complexity: bool = True
    run_birthday: bool = True
    monobit_bits: int = 100_000_000
    runs_bits: int = 100_000_000
    rank_matrices: int = 100_000
    lc_block_length: int = 1000
    lc_blocks: int = 100_000
    birthday_draws: int = 4096
    birthday_bits: int = 32
    birthday_rounds: int = 762

    @staticmethod
    def defaults() -> "BatteryConfig":
        return BatteryConfig()

    @staticmethod
    def quick() -> "BatteryConfig":
        return BatteryConfig(monobit_bits=1_000_000, runs_bits=1_000_000, rank_matrices=1_000,
                             lc_block_length=500, lc_blocks=200, birthday_rounds=8)


def _verdict(p: float) -> str:
    """tests.cpp:23-30."""
    tail = min(p, 1.0 - p)
    if tail < 1e-10:
        return "fail"
    if tail < 1e-4:
        return "suspect"
    return "pass"


# ---- the battery -----------------------------------------------------------

def run_battery_gpu(params: GeneratorParams, seed: int, config: BatteryConfig = None,
                    device: int = 0) -> Dict:
    """run_battery (battery.cpp:72-112) over XorgensState(params, seed)'s
    stream, counting on the GPU.  Returns the report as the reference's
    to_json lays it out (battery.cpp:114-130): tests with name, n, statistic,
    p and verdict, and the overall verdict."""
    torch = _torch()
    cfg = config or BatteryConfig.defaults()
    if params.w != 32:
        raise ValueError("the GPU battery reads 32-bit words")
    if cfg.run_matrix_rank and not (fast_path(params) and params.r - params.s < 64):
        # The fused rank test runs in the pair-lane kernel only (xg_rank_test:
        # r = 128, r - s < 64); refuse before any test consumes the stream.
        raise UnsupportedParamsError(
            "the GPU matrix-rank test needs r = 128 and r - s < 64 (set run_matrix_rank=False)")
    with torch.cuda.device(device):
        return _run_battery(params, seed, cfg, device)


def _run_battery(params: GeneratorParams, seed: int, cfg: BatteryConfig, device: int) -> Dict:
    torch = _torch()
    dev = f"cuda:{device}"
    e = BlockEnsemble(params, seed, 1, lane_bound(params), device=device)
    tests: List[Dict] = []

    def bits_counts(nbits: int):
        words = e.fill_u32((nbits + 31) // 32)
        out = torch.zeros(2, dtype=torch.int64, device=dev)
        _raise(lib.xg_bits_ones_runs(ctypes.c_void_p(words.data_ptr()), nbits,
                                     ctypes.c_void_p(out.data_ptr()), e._stream()))
        ones, trans = (int(v) for v in out.tolist())
        return ones, trans

    if cfg.run_monobit:  # tests.cpp:33-47
        n = cfg.monobit_bits
        if n < 100:
            raise ValueError("monobit needs n >= 100")
        ones, _ = bits_counts(n)
        abs_s = abs(float(2 * ones - n))
        p = math.erfc(abs_s / math.sqrt(2.0 * float(n)))
        tests.append({"name": "monobit", "n": n, "statistic": abs_s / math.sqrt(float(n)),
                      "p": p, "verdict": _verdict(p)})
    if cfg.run_runs:  # tests.cpp:49-79
        n = cfg.runs_bits
        if n < 100:
            raise ValueError("runs test needs n >= 100")
        ones, trans = bits_counts(n)
        runs = 1 + trans
        nn = float(n)
        pi = float(ones) / nn
        if abs(pi - 0.5) >= 2.0 / math.sqrt(nn):
            tests.append({"name": "runs", "n": n, "statistic": float(runs), "p": 0.0,
                          "verdict": "not_applicable"})
        else:
            v = float(runs)
            p = math.erfc(abs(v - 2.0 * nn * pi * (1.0 - pi)) /
                          (2.0 * math.sqrt(2.0 * nn) * pi * (1.0 - pi)))
            tests.append({"name": "runs", "n": n, "statistic": v, "p": p, "verdict": _verdict(p)})
    if cfg.run_matrix_rank:  # tests.cpp:81-126
        m = cfg.rank_matrices
        if m < 38:
            raise ValueError("rank test needs >= 38 matrices")
        chi2, p = matrix_rank_statistic(e.rank_test(m))
        tests.append({"name": "matrix_rank", "n": m * 32 * 32, "statistic": chi2,
                      "p": p, "verdict": _verdict(p)})
    if cfg.run_linear_complexity:  # tests.cpp:128-178
        k, nb = cfg.lc_block_length, cfg.lc_blocks
        if k < 128 or nb < 38:
            raise ValueError("linear complexity test needs K >= 128 and >= 38 blocks")
        chi2, p = linear_complexity_statistic(e.linear_complexity_test(k, nb), k)
        tests.append({"name": "linear_complexity", "n": nb * k, "statistic": chi2, "p": p,
                      "verdict": _verdict(p)})
    if cfg.run_birthday:  # tests.cpp:175-212
        n, t, rounds = cfg.birthday_draws, cfg.birthday_bits, cfg.birthday_rounds
        if t == 0 or t > 32:
            raise ValueError("t_bits must fit in the source word size")
        if rounds == 0 or n < 2:
            raise ValueError("birthday spacings needs draws and rounds")
        lam = float(n) * float(n) * float(n) / math.pow(2.0, t + 2.0)
        if lam < 1.0 or lam > 16.0:
            raise ValueError("n^3 / 2^{t+2} must lie in [1, 16]")
        words = e.fill_u32(n * rounds)
        dup = torch.zeros(1, dtype=torch.int64, device=dev)
        _raise(lib.xg_birthday_duplicates(ctypes.c_void_p(words.data_ptr()), n, rounds, t,
                                          ctypes.c_void_p(dup.data_ptr()), e._stream()))
        d = int(dup.item())
        p = poisson_upper_tail(d, lam * rounds)
        tests.append({"name": "birthday_spacings", "n": rounds * n * 32, "statistic": float(d),
                      "p": p, "verdict": _verdict(p)})
    overall = "pass"
    for tr in tests:
        if tr["verdict"] == "fail":
            overall = "fail"
        elif tr["verdict"] == "suspect" and overall != "fail":
            overall = "suspect"
    return {"seed": seed, "num_tests": len(tests), "overall": overall, "tests": tests}

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
from .xorgens import (BlockEnsemble, GeneratorParams, _raise, _torch, fast_path, lane_bound,
                      linear_complexity_statistic, matrix_rank_statistic)

__all__ = ["BatteryConfig", "BatteryInputError", "run_battery_gpu", "run_battery_on_words",
           "regularized_gamma_p", "regularized_gamma_q"]


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
    def parse(text: str) -> "BatteryConfig":
        """BatteryConfig::parse (battery.cpp:38-70): `key = value` lines, `#`
        comments; unknown keys and malformed lines raise ValueError."""
        c = BatteryConfig()
        keys = {"monobit.enabled": ("run_monobit", _parse_bool), "monobit.bits": ("monobit_bits", int),
                "runs.enabled": ("run_runs", _parse_bool), "runs.bits": ("runs_bits", int),
                "matrix_rank.enabled": ("run_matrix_rank", _parse_bool),
                "matrix_rank.matrices": ("rank_matrices", int),
                "linear_complexity.enabled": ("run_linear_complexity", _parse_bool),
                "linear_complexity.block_length": ("lc_block_length", int),
                "linear_complexity.blocks": ("lc_blocks", int),
                "birthday.enabled": ("run_birthday", _parse_bool),
                "birthday.draws": ("birthday_draws", int), "birthday.bits": ("birthday_bits", int),
                "birthday.rounds": ("birthday_rounds", int)}
        for line in text.splitlines():
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ValueError("battery config line is not key = value: " + line)
            key, value = (x.strip() for x in line.split("=", 1))
            if key not in keys:
                raise ValueError("unknown battery config key: " + key)
            attr, conv = keys[key]
            try:
                setattr(c, attr, conv(value))
            except ValueError as e:
                raise ValueError(f"bad value for {key}: {value}") from e
        return c

    @staticmethod
    def quick() -> "BatteryConfig":
        return BatteryConfig(monobit_bits=1_000_000, runs_bits=1_000_000, rank_matrices=1_000,
                             lc_block_length=500, lc_blocks=200, birthday_rounds=8)


def _parse_bool(v: str) -> bool:
    """battery.cpp:30-34."""
    if v in ("true", "on", "1"):
        return True
    if v in ("false", "off", "0"):
        return False
    raise ValueError(f"expected boolean, got '{v}'")


def _verdict(p: float) -> str:
    """tests.cpp:23-30."""
    tail = min(p, 1.0 - p)
    if tail < 1e-10:
        return "fail"
    if tail < 1e-4:
        return "suspect"
    return "pass"


# ---- the battery -----------------------------------------------------------

class BatteryInputError(RuntimeError):
    """The word source ran out (the reference throws runtime_error from
    FileWordSource, xgen exits 66)."""


class _GenWords:
    """The stream of XorgensState(params, seed) on the GPU (raw=True: the
    Weyl-ablated RawXorgens stream), w = 8, 16 or 32.  Each call consumes the
    next words, as each of the reference's tests reads the same WordSource in
    turn through a fresh BitSource (w bits per word, MSB first)."""

    def __init__(self, params: GeneratorParams, seed: int, device: int, raw: bool):
        self.e = BlockEnsemble(params, seed, 1, lane_bound(params), device=device)
        self.raw = raw
        self.w = params.w
        self.fused = not raw and self.w == 32 and fast_path(params)
        self.fused_rank = self.fused and params.r - params.s < 64

    def _words(self, n: int):
        return (self.e.fill_raw_u32(n) if self.raw else self.e.fill_u32(n))[0]

    def stream(self):
        return self.e._stream()

    def take_bits(self, nbits: int):
        """The next ceil(nbits / w) words as a 32-bit MSB-first bit stream."""
        words = self._words((nbits + self.w - 1) // self.w)
        return words if self.w == 32 else _pack(words, self.w, False, self.stream())

    def take_draws(self, n: int):
        """The next n words, each at the top of 32 bits (birthday draws)."""
        words = self._words(n)
        return words if self.w == 32 else _pack(words, self.w, True, self.stream())

    def rank_bins(self, m: int, dev: str):
        if self.fused_rank:  # fused in the generator: no words stored
            return self.e.rank_test(m)
        return _rank_words(self.take_bits(1024 * m), m, dev, self.stream())

    def lc_hist(self, k: int, nb: int, dev: str):
        if self.fused:  # words staged by the library, the BitSource tail dropped
            return self.e.linear_complexity_test(k, nb)
        bits = self.take_bits(k * nb)
        return _lc_words(bits, k, nb, dev, self.stream())


class _BufWords:
    """32-bit words already on the device (e.g. a raw-le file), consumed in
    order like the reference's FileWordSource."""

    w = 32

    def __init__(self, words, stream):
        self.words = words
        self.pos = 0
        self.s = stream

    def _take(self, n: int):
        if self.pos + n > self.words.numel():
            raise BatteryInputError("input exhausted: the battery needs more words than the input holds")
        out = self.words[self.pos:self.pos + n]
        self.pos += n
        return out

    def take_bits(self, nbits: int):
        return self._take((nbits + 31) // 32)

    def take_draws(self, n: int):
        return self._take(n)

    def stream(self):
        return self.s

    def rank_bins(self, m: int, dev: str):
        return _rank_words(self.take_bits(1024 * m), m, dev, self.s)

    def lc_hist(self, k: int, nb: int, dev: str):
        return _lc_words(self.take_bits(k * nb), k, nb, dev, self.s)


def _pack(words, w: int, left_align: bool, stream):
    torch = _torch()
    n = words.numel()
    out = torch.empty(n if left_align else (n * w + 31) // 32, dtype=torch.int32, device=words.device)
    _raise(lib.xg_pack_words(ctypes.c_void_p(words.data_ptr()), n, w, int(left_align),
                             ctypes.c_void_p(out.data_ptr()), stream))
    return out


def _rank_words(words, m: int, dev: str, stream):
    torch = _torch()
    out = torch.zeros(3, dtype=torch.int64, device=dev)
    _raise(lib.xg_rank_words(ctypes.c_void_p(words.data_ptr()), m, ctypes.c_void_p(out.data_ptr()),
                             stream))
    return out


def _lc_words(words, k: int, nb: int, dev: str, stream):
    torch = _torch()
    hist = torch.zeros(k + 1, dtype=torch.int64, device=dev)
    _raise(lib.xg_lc_words(ctypes.c_void_p(words.data_ptr()), words.numel(), k, nb,
                           ctypes.c_void_p(hist.data_ptr()), stream))
    return hist


def run_battery_gpu(params: GeneratorParams, seed: int, config: BatteryConfig = None,
                    device: int = 0, raw: bool = False) -> Dict:
    """run_battery (battery.cpp:72-112) over XorgensState(params, seed)'s
    stream (raw=True: RawXorgens, the Weyl-ablated negative control), counting
    on the GPU.  Returns the report as the reference's to_json lays it out
    (battery.cpp:114-130): tests with name, n, statistic, p and verdict, and
    the overall verdict.  Every w = 32 set runs every test: the matrix-rank
    test is fused into the generator where the pair-lane kernel takes the set,
    else it runs over stored words (xg_rank_words)."""
    torch = _torch()
    cfg = config or BatteryConfig.defaults()
    if params.w not in (8, 16, 32):
        raise ValueError("the GPU battery reads 8-, 16- or 32-bit words")
    with torch.cuda.device(device):
        return _run_battery(_GenWords(params, seed, device, raw), cfg, device, seed)


def run_battery_on_words(words, config: BatteryConfig = None, seed: int = 0) -> Dict:
    """run_battery over a stream of 32-bit words already in device memory (a
    1-D CUDA tensor, e.g. a raw-le file), consumed in the reference's order;
    BatteryInputError when the words run out (the reference's FileWordSource
    throws, xgen exits 66)."""
    torch = _torch()
    cfg = config or BatteryConfig.defaults()
    if not words.is_cuda or words.dim() != 1 or words.element_size() != 4:
        raise ValueError("words must be a 1-D CUDA tensor of 32-bit words")
    dev = words.device.index or 0
    with torch.cuda.device(dev):
        src = _BufWords(words.contiguous(), ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        return _run_battery(src, cfg, dev, seed)


def _run_battery(src, cfg: BatteryConfig, device: int, seed: int) -> Dict:
    torch = _torch()
    dev = f"cuda:{device}"
    tests: List[Dict] = []

    def bits_counts(nbits: int):
        words = src.take_bits(nbits)
        out = torch.zeros(2, dtype=torch.int64, device=dev)
        _raise(lib.xg_bits_ones_runs(ctypes.c_void_p(words.data_ptr()), nbits,
                                     ctypes.c_void_p(out.data_ptr()), src.stream()))
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
        chi2, p = matrix_rank_statistic(src.rank_bins(m, dev))
        tests.append({"name": "matrix_rank", "n": m * 32 * 32, "statistic": chi2,
                      "p": p, "verdict": _verdict(p)})
    if cfg.run_linear_complexity:  # tests.cpp:128-178
        k, nb = cfg.lc_block_length, cfg.lc_blocks
        if k < 128 or nb < 38:
            raise ValueError("linear complexity test needs K >= 128 and >= 38 blocks")
        chi2, p = linear_complexity_statistic(src.lc_hist(k, nb, dev), k)
        tests.append({"name": "linear_complexity", "n": nb * k, "statistic": chi2, "p": p,
                      "verdict": _verdict(p)})
    if cfg.run_birthday:  # tests.cpp:175-212
        n, t, rounds = cfg.birthday_draws, cfg.birthday_bits, cfg.birthday_rounds
        if t == 0 or t > src.w:
            raise ValueError("t_bits must fit in the source word size")
        if rounds == 0 or n < 2:
            raise ValueError("birthday spacings needs draws and rounds")
        lam = float(n) * float(n) * float(n) / math.pow(2.0, t + 2.0)
        if lam < 1.0 or lam > 16.0:
            raise ValueError("n^3 / 2^{t+2} must lie in [1, 16]")
        words = src.take_draws(n * rounds)
        dup = torch.zeros(1, dtype=torch.int64, device=dev)
        _raise(lib.xg_birthday_duplicates(ctypes.c_void_p(words.data_ptr()), n, rounds, t,
                                          ctypes.c_void_p(dup.data_ptr()), src.stream()))
        d = int(dup.item())
        p = poisson_upper_tail(d, lam * rounds)
        tests.append({"name": "birthday_spacings", "n": rounds * n * src.w, "statistic": float(d),
                      "p": p, "verdict": _verdict(p)})
    overall = "pass"
    for tr in tests:
        if tr["verdict"] == "fail":
            overall = "fail"
        elif tr["verdict"] == "suspect" and overall != "fail":
            overall = "suspect"
    return {"seed": seed, "num_tests": len(tests), "overall": overall, "tests": tests}

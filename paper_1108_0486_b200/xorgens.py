"""Python mirror of the reference ``xg`` API over the GPU C ABI.

Names, argument meaning and error behaviour follow the reference C++ library
(paths relative to the reference tree):

* ``GeneratorParams``, ``ParamError``, ``check_params``, ``validate_params``,
  ``lane_bound``, ``recommended_weyl_increment``, ``default_output_shift``,
  ``period_description`` and the shipped sets -- proj/include/xg/params.hpp,
  proj/src/params.cpp.  Pure host logic (through the C ABI, no GPU needed).
* ``XorgensState`` (seeded or ``from_raw``), ``next_word``, ``logical_buffer``,
  ``weyl_value`` -- proj/include/xg/xorgens.hpp, proj/src/xorgens.cpp -- as a
  one-stream device ensemble served by ``xg_next_u32``.
* ``batch_step`` -- proj/src/parallel.cpp:8-42 (lane check, then words).
* ``BlockEnsemble`` -- proj/include/xg/parallel.hpp:35-59,
  proj/src/parallel.cpp:84-135: consecutive seeds, block-major ``generate``
  that continues streams, plus the device-buffer fills the GPU adds
  (``fill_u32/u64/f32/f64``, ``mc_pi``).
* ``XorgensSource`` -- the ``WordSource`` adapter (proj/include/xg/stream.hpp:17-34).

Error mapping: ``std::out_of_range`` -> :class:`OutOfRangeError` (an
``IndexError``), ``ParamValidationError`` -> :class:`ParamValidationError`
(a ``ValueError`` with ``.code``), ``std::invalid_argument`` -> ``ValueError``,
CUDA failures -> :class:`XgCudaError`.  Every computation runs in
libxg_gpu.so kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import math
import enum
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import lib, xg_params_t
from .pvalues import chi_square_pvalue

__all__ = [
    "GeneratorParams", "ParamError", "ParamValidationError", "OutOfRangeError", "XgCudaError",
    "UnsupportedParamsError", "check_params", "validate_params", "lane_bound",
    "recommended_weyl_increment", "default_output_shift", "period_description",
    "PeriodDescription", "xorgensgp32_params", "tiny_r2w8_params", "tiny_r2w16_params",
    "tiny_r4w16_params", "gpu_supported", "fast_path", "XorgensState", "seed_state", "batch_step",
    "BlockEnsemble", "XorgensSource", "partition", "kernel_launches", "matrix_rank_statistic",
    "RANK_P32", "linear_complexity_statistic", "LC_PI", "berlekamp_massey",
]


class ParamError(enum.IntEnum):
    """proj/include/xg/params.hpp:31-38 (same order)."""

    bad_word_size = 0
    s_out_of_range = 1
    gcd_not_one = 2
    shift_out_of_range = 3
    gamma_out_of_range = 4
    even_weyl_increment = 5


class ParamValidationError(ValueError):
    """proj/include/xg/params.hpp:42-49: invalid_argument carrying a ParamError."""

    def __init__(self, code: ParamError):
        super().__init__(lib.xg_strerror(int(code) + 1).decode())
        self._code = ParamError(code)

    def code(self) -> ParamError:
        return self._code


class OutOfRangeError(IndexError):
    """std::out_of_range in the reference (lanes, block counts, indices)."""


class UnsupportedParamsError(ValueError):
    """Valid parameters the GPU kernels do not implement (w=32, r=128, lane_bound>=32)."""


class XgCudaError(RuntimeError):
    """A CUDA runtime failure inside libxg_gpu.so."""


def _raise(rc: int, what: str = "") -> None:
    if rc == _lib.XG_OK:
        return
    msg = lib.xg_strerror(rc).decode() + (f" ({what})" if what else "")
    if 1 <= rc <= 6:
        raise ParamValidationError(ParamError(rc - 1))
    if rc == _lib.XG_ERANGE:
        raise OutOfRangeError(msg)
    if rc == _lib.XG_EINVAL:
        raise ValueError(msg)
    if rc == _lib.XG_EUNSUPPORTED:
        raise UnsupportedParamsError(msg)
    if rc == _lib.XG_ENOMEM:
        raise MemoryError(msg)
    raise XgCudaError(msg)


@dataclass(frozen=True)
class GeneratorParams:
    """proj/include/xg/params.hpp:17-29."""

    r: int = 0
    s: int = 0
    a: int = 0
    b: int = 0
    c: int = 0
    d: int = 0
    w: int = 32
    omega: int = 0
    gamma: int = 0

    def mask(self) -> int:
        return (1 << 64) - 1 if self.w >= 64 else (1 << self.w) - 1

    def _c(self) -> xg_params_t:
        return xg_params_t(self.r, self.s, self.a, self.b, self.c, self.d, self.w,
                           self.omega & ((1 << 64) - 1), self.gamma)

    @staticmethod
    def _from_c(p: xg_params_t) -> "GeneratorParams":
        return GeneratorParams(p.r, p.s, p.a, p.b, p.c, p.d, p.w, p.omega, p.gamma)


def check_params(p: GeneratorParams) -> Optional[ParamError]:
    """proj/src/params.cpp:22-37: None when valid, else the first violation."""
    rc = lib.xg_params_check(ctypes.byref(p._c()))
    return None if rc == 0 else ParamError(rc - 1)


def validate_params(p: GeneratorParams) -> GeneratorParams:
    """proj/src/params.cpp:39-43."""
    e = check_params(p)
    if e is not None:
        raise ParamValidationError(e)
    return p


def lane_bound(p: GeneratorParams) -> int:
    """proj/include/xg/params.hpp:59-61: min(s, r - s)."""
    return int(lib.xg_lane_bound(ctypes.byref(p._c())))


def recommended_weyl_increment(w: int) -> int:
    """proj/src/params.cpp:53-62; raises like the reference for a bad w."""
    v = int(lib.xg_recommended_weyl_increment(w))
    if v == 0:
        raise ParamValidationError(ParamError.bad_word_size)
    return v


def default_output_shift(w: int) -> int:
    """proj/include/xg/params.hpp:77."""
    return int(lib.xg_default_output_shift(w))


@dataclass(frozen=True)
class PeriodDescription:
    linear_exponent: int
    weyl_factor_exponent: int
    display: str


def period_description(p: GeneratorParams) -> PeriodDescription:
    """proj/src/params.cpp:45-51."""
    return PeriodDescription(p.r * p.w, p.w, f"~2^{p.r * p.w + p.w}")


def xorgensgp32_params() -> GeneratorParams:
    return GeneratorParams._from_c(lib.xg_params_xorgensgp32())


def tiny_r2w8_params() -> GeneratorParams:
    return GeneratorParams._from_c(lib.xg_params_tiny_r2w8())


def tiny_r2w16_params() -> GeneratorParams:
    return GeneratorParams._from_c(lib.xg_params_tiny_r2w16())


def tiny_r4w16_params() -> GeneratorParams:
    return GeneratorParams._from_c(lib.xg_params_tiny_r4w16())


def gpu_supported(p: GeneratorParams) -> bool:
    """True when the GPU can generate `p` (every valid set with r <= 16384)."""
    return lib.xg_gpu_supported(ctypes.byref(p._c())) == 0


def fast_path(p: GeneratorParams) -> bool:
    """True when `p` runs on the register-window kernels (w=32, r=128,
    lane_bound >= 32); other valid sets run on the general-parameter kernels."""
    return bool(lib.xg_fast_path(ctypes.byref(p._c())))


def partition(total_streams: int, world: int, rank: int) -> Tuple[int, int]:
    """Stream range (first, count) of `rank` in a `world`-device job."""
    first, count = ctypes.c_uint64(), ctypes.c_uint32()
    _raise(lib.xg_partition(total_streams, world, rank, ctypes.byref(first), ctypes.byref(count)))
    return first.value, count.value


def kernel_launches() -> int:
    return int(lib.xg_kernel_launches())


# ---- device plumbing (torch only for buffers, streams and devices) --------

def _torch():
    import torch

    if not torch.cuda.is_available():
        raise XgCudaError("no CUDA device: the xorgensGP path runs only on the GPU")
    return torch


def _stream_ptr(device: int):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _default_device(device: Optional[int]) -> int:
    torch = _torch()
    return torch.cuda.current_device() if device is None else int(device)


class _Handle:
    def __init__(self, ptr: ctypes.c_void_p, device: int):
        self.ptr = ptr
        self.device = device

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            lib.xg_ensemble_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()


# Random 32 x 32 GF(2) matrix: P(rank 32), P(rank 31), P(rank <= 30)
# (proj/src/stattests/tests.cpp:89-91).
RANK_P32 = (0.288788095153841, 0.577576190173205, 0.133635714672954)


def matrix_rank_statistic(counts) -> Tuple[float, float]:
    """(chi-square statistic, p-value) of rank-test bins, computed as
    proj/src/stattests/tests.cpp:111-123: chi2 over the three bins, p the
    chi-square survival function with 2 degrees of freedom, computed by the
    reference's own incomplete-gamma code (pvalues.py)."""
    c = [float(int(v)) for v in (counts.tolist() if hasattr(counts, "tolist") else counts)][:3]
    nm = sum(c)
    chi2 = 0.0
    for i in range(3):
        e = nm * RANK_P32[i]
        d = c[i] - e
        chi2 += d * d / e
    return chi2, chi_square_pvalue(chi2, 2)


# Linear complexity test bins (proj/src/stattests/tests.cpp:140-141).
LC_PI = (0.010417, 0.03125, 0.125, 0.5, 0.25, 0.0625, 0.020833)


def berlekamp_massey(seqs, nbits: int):
    """Linear complexity (proj/src/stattests/gf2.cpp:62-110) of every row of
    ``seqs`` -- a 2-D CUDA tensor of 32-bit words, each row one sequence of
    ``nbits`` bits packed MSB first -- on the GPU, one warp per row.  Returns
    an int32 CUDA tensor of the complexities."""
    torch = _torch()
    if seqs.dim() != 2 or seqs.element_size() != 4 or not seqs.is_cuda or not seqs.is_contiguous():
        raise ValueError("seqs must be a contiguous 2-D CUDA tensor of 32-bit words")
    if nbits > 32 * seqs.shape[1]:
        raise ValueError("rows hold fewer than nbits bits")
    out = torch.empty(seqs.shape[0], dtype=torch.int32, device=seqs.device)
    _raise(lib.xg_berlekamp_massey(ctypes.c_void_p(seqs.data_ptr()), nbits, seqs.shape[0],
                                   seqs.shape[1], ctypes.c_void_p(out.data_ptr()),
                                   _stream_ptr(seqs.device.index or 0)))
    return out


def linear_complexity_statistic(hist, block_length: int) -> Tuple[float, float]:
    """(chi-square statistic, p-value) from a histogram of per-block linear
    complexities, binned exactly as proj/src/stattests/tests.cpp:135-172
    (mu, the sign, T = sign * (L - mu) + 2/9, seven bins; p = chi-square
    survival with 6 degrees of freedom)."""
    h = [int(v) for v in (hist.tolist() if hasattr(hist, "tolist") else hist)]
    k = float(block_length)
    sign = 1.0 if block_length % 2 == 0 else -1.0
    mu = k / 2.0 + (9.0 - sign) / 36.0 - (k / 3.0 + 2.0 / 9.0) / math.pow(2.0, 1000.0 if k > 1000 else k)
    counts = [0] * 7
    for L, c in enumerate(h):
        if not c:
            continue
        t = sign * (float(L) - mu) + 2.0 / 9.0
        if t <= -2.5:
            b = 0
        elif t <= -1.5:
            b = 1
        elif t <= -0.5:
            b = 2
        elif t <= 0.5:
            b = 3
        elif t <= 1.5:
            b = 4
        elif t <= 2.5:
            b = 5
        else:
            b = 6
        counts[b] += c
    nb = float(sum(counts))
    chi2 = 0.0
    for i in range(7):
        diff = float(counts[i]) - nb * LC_PI[i]
        chi2 += diff * diff / (nb * LC_PI[i])
    return chi2, chi_square_pvalue(chi2, 6)


class BlockEnsemble:
    """``xg::BlockEnsemble`` on one GPU (proj/src/parallel.cpp:84-135).

    Block i is the stream seeded with ``base_seed + first_stream + i`` (uint64
    wrap); ``first_stream`` is 0 for the reference's own ensemble and is how a
    multi-GPU job hands each device a disjoint slice of one global ensemble.
    """

    def __init__(self, params: GeneratorParams, base_seed: int, num_blocks: int, lanes: int,
                 *, first_stream: int = 0, device: Optional[int] = None):
        # proj/src/parallel.cpp:86-91: params, then blocks, then lanes -- all
        # host-side, before any device work.
        validate_params(params)
        if num_blocks <= 0 or num_blocks >= 1 << 32:
            raise OutOfRangeError("ensemble needs at least one block")
        if lanes <= 0 or lanes > lane_bound(params):
            raise OutOfRangeError("lane count exceeds min(s, r - s)")
        if not gpu_supported(params):
            _raise(_lib.XG_EUNSUPPORTED)
        dev = _default_device(device)
        h = ctypes.c_void_p()
        _raise(lib.xg_ensemble_create(ctypes.byref(params._c()), base_seed & ((1 << 64) - 1),
                                      first_stream & ((1 << 64) - 1), num_blocks, lanes, dev,
                                      _stream_ptr(dev), ctypes.byref(h)), "ensemble_create")
        self._h = _Handle(h, dev)
        self._params = params
        self._base_seed = base_seed & ((1 << 64) - 1)
        self._first = first_stream
        self._n = num_blocks
        self._lanes = lanes

    @classmethod
    def from_raw(cls, params: GeneratorParams, buffers: np.ndarray, weyls: Sequence[int],
                 *, device: Optional[int] = None) -> "BlockEnsemble":
        """One stream per row of ``buffers`` (r words, oldest first), no warm-up
        (XorgensState::from_raw, proj/src/xorgens.cpp:34-38)."""
        dev = _default_device(device)
        buf = np.ascontiguousarray(np.asarray(buffers, dtype=np.uint64).reshape(len(weyls), -1))
        wy = np.ascontiguousarray(np.asarray(weyls, dtype=np.uint64))
        validate_params(params)
        if buf.shape[1] != params.r:
            raise ValueError("buffer size must equal r")
        h = ctypes.c_void_p()
        _raise(lib.xg_ensemble_create_from_raw(
            ctypes.byref(params._c()), len(wy), buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            wy.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), dev, _stream_ptr(dev),
            ctypes.byref(h)), "ensemble_create_from_raw")
        self = cls.__new__(cls)
        self._h = _Handle(h, dev)
        self._params = params
        self._base_seed = 0
        self._first = 0
        self._n = len(wy)
        self._lanes = lane_bound(params)
        return self

    # -- reference accessors (proj/include/xg/parallel.hpp:49-53)
    def num_blocks(self) -> int:
        return self._n

    def lanes(self) -> int:
        return self._lanes

    def base_seed(self) -> int:
        return self._base_seed

    def first_stream(self) -> int:
        return self._first

    @property
    def params(self) -> GeneratorParams:
        return self._params

    @property
    def device(self) -> int:
        return self._h.device

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h.ptr

    def _stream(self, stream=None):
        if stream is None:
            return _stream_ptr(self._h.device)
        return ctypes.c_void_p(getattr(stream, "cuda_stream", stream))

    # -- generation ----------------------------------------------------------
    def generate(self, per_block: int, workers: int = 0) -> np.ndarray:
        """BlockEnsemble::generate (proj/src/parallel.cpp:97-135) into host
        memory: a (num_blocks, per_block) array, block-major, continuing each
        block's stream -- uint32 for w <= 32, uint64 for w = 64.  ``workers``
        is accepted for API parity only."""
        del workers
        wide = self._params.w > 32
        out = np.empty((self._n, per_block), dtype=np.uint64 if wide else np.uint32)
        if per_block:
            fn = lib.xg_generate_host_words if wide else lib.xg_generate_host
            _raise(fn(self._h.ptr, per_block, out.ctypes.data_as(ctypes.c_void_p), self._stream()),
                   "generate")
        return out

    def _host_ptr(self, host_out, per_block: int, itemsize: int) -> ctypes.c_void_p:
        """Address of a caller host buffer (torch CPU tensor or numpy array)
        that must hold num_blocks * per_block contiguous elements of
        `itemsize` bytes -- the C ABI takes a bare pointer and cannot check."""
        if hasattr(host_out, "data_ptr"):
            ok = (not host_out.is_cuda and host_out.is_contiguous()
                  and host_out.element_size() == itemsize)
            n, ptr = host_out.numel(), host_out.data_ptr()
        else:
            ok = host_out.flags["C_CONTIGUOUS"] and host_out.itemsize == itemsize
            n, ptr = host_out.size, host_out.ctypes.data
        if not ok or n < self._n * per_block:
            raise ValueError(f"host buffer must be contiguous host memory of at least "
                             f"{self._n * per_block} elements of {itemsize} bytes")
        return ctypes.c_void_p(ptr)

    def generate_into_host(self, per_block: int, host_out, stream=None) -> None:
        """generate() into a caller buffer (e.g. a pinned torch tensor) of
        uint32 words."""
        ptr = self._host_ptr(host_out, per_block, 4)
        _raise(lib.xg_generate_host(self._h.ptr, per_block, ptr, self._stream(stream)), "generate")

    def generate_f32_into_host(self, per_block: int, host_out, stream=None) -> None:
        """per_block uniform f32 values of every block into a host buffer
        (block-major), converted on the device."""
        ptr = self._host_ptr(host_out, per_block, 4)
        _raise(lib.xg_generate_host_f32(self._h.ptr, per_block, ptr, self._stream(stream)),
               "generate_f32")

    def generate_f64_into_host(self, per_block: int, host_out, stream=None) -> None:
        """per_block uniform f64 values (two words each) of every block into a
        host buffer (block-major), converted on the device."""
        ptr = self._host_ptr(host_out, per_block, 8)
        _raise(lib.xg_generate_host_f64(self._h.ptr, per_block, ptr, self._stream(stream)),
               "generate_f64")

    def _fill(self, fn, per_block: int, out, torch_dtype, vals_per_block: int, stream):
        torch = _torch()
        if out is None:
            out = torch.empty((self._n, vals_per_block), dtype=torch_dtype,
                              device=f"cuda:{self._h.device}")
        if out.numel() < self._n * vals_per_block or not out.is_contiguous():
            raise ValueError("output buffer too small or not contiguous")
        if out.element_size() != torch.empty(0, dtype=torch_dtype).element_size() or not out.is_cuda:
            raise ValueError(f"output buffer must be a CUDA tensor of {torch_dtype} width")
        if out.device.index != self._h.device:
            raise ValueError(f"output buffer is on cuda:{out.device.index}, the ensemble on "
                             f"cuda:{self._h.device}")
        _raise(fn(self._h.ptr, per_block, ctypes.c_void_p(out.data_ptr()), self._stream(stream)))
        return out

    def fill_u32(self, per_block: int, out=None, stream=None):
        """Device fill, out[g, k] = word k of block g (continuing)."""
        return self._fill(lib.xg_fill_u32, per_block, out, _torch().uint32, per_block, stream)

    def fill_words(self, per_block: int, out=None, stream=None):
        """Every word as uint64 (the reference generate() element type); any w."""
        return self._fill(lib.xg_fill_words, per_block, out, _torch().uint64, per_block, stream)

    def fill_raw_u32(self, per_block: int, out=None, stream=None):
        """Weyl-ablated linear stream (RawXorgens::next, registry "xorgens-raw")."""
        return self._fill(lib.xg_fill_raw_u32, per_block, out, _torch().uint32, per_block, stream)

    def fill_u64(self, per_block: int, out=None, stream=None):
        """Two consecutive words per value, lo first."""
        return self._fill(lib.xg_fill_u64, per_block, out, _torch().uint64, per_block, stream)

    def fill_f32(self, per_block: int, out=None, stream=None):
        """Uniform [0,1): (word >> 8) * 2^-24."""
        return self._fill(lib.xg_fill_f32, per_block, out, _torch().float32, per_block, stream)

    def fill_f64(self, per_block: int, out=None, stream=None):
        """Uniform [0,1): (u64 >> 11) * 2^-53, u64 from two words, lo first."""
        return self._fill(lib.xg_fill_f64, per_block, out, _torch().float64, per_block, stream)

    def mc_pi(self, samples_per_block: int, hits=None, stream=None):
        """Fused in-register Monte Carlo: adds the hit count to ``hits`` (a
        1-element int64 CUDA tensor, created zeroed if None) and returns it."""
        torch = _torch()
        if hits is None:
            hits = torch.zeros(1, dtype=torch.int64, device=f"cuda:{self._h.device}")
        if (hits.numel() < 1 or hits.element_size() != 8 or not hits.is_cuda
                or hits.device.index != self._h.device):
            raise ValueError(f"hits must be an int64 tensor on cuda:{self._h.device}")
        _raise(lib.xg_mc_pi(self._h.ptr, samples_per_block, ctypes.c_void_p(hits.data_ptr()),
                            self._stream(stream)))
        return hits

    def rank_test(self, matrices_per_block: int, counts=None, stream=None):
        """Fused GF(2) matrix-rank test (the reference's matrix_rank_test,
        proj/src/stattests/tests.cpp:81-126, M = 32) over the next
        32*matrices_per_block words of every block: adds the (rank 32, 31,
        <= 30) bins to ``counts`` (a 3-element int64 CUDA tensor, created
        zeroed if None) and returns it.  ``matrix_rank_statistic(counts)``
        gives the chi-square statistic and p-value."""
        torch = _torch()
        if counts is None:
            counts = torch.zeros(3, dtype=torch.int64, device=f"cuda:{self._h.device}")
        if counts.numel() < 3 or counts.element_size() != 8 or not counts.is_cuda:
            raise ValueError("counts must be a CUDA tensor of at least 3 int64")
        _raise(lib.xg_rank_test(self._h.ptr, matrices_per_block, ctypes.c_void_p(counts.data_ptr()),
                                self._stream(stream)))
        return counts

    def linear_complexity_test(self, block_length: int, blocks_per_block: int, hist=None,
                               stream=None):
        """Linear complexity test (the reference's linear_complexity_test,
        proj/src/stattests/tests.cpp:128-178) on the GPU: the next
        ceil(block_length * blocks_per_block / 32) words of every block, read
        MSB first, in blocks of block_length bits; adds the histogram of the
        Berlekamp-Massey complexities to ``hist`` (an int64 CUDA tensor of
        block_length + 1 entries, created zeroed if None) and returns it.
        ``linear_complexity_statistic(hist, block_length)`` gives the
        reference's chi-square statistic and p-value."""
        torch = _torch()
        if hist is None:
            hist = torch.zeros(block_length + 1, dtype=torch.int64,
                               device=f"cuda:{self._h.device}")
        if hist.numel() < block_length + 1 or hist.element_size() != 8 or not hist.is_cuda:
            raise ValueError("hist must be a CUDA tensor of block_length + 1 int64")
        _raise(lib.xg_linear_complexity_test(self._h.ptr, block_length, blocks_per_block,
                                             ctypes.c_void_p(hist.data_ptr()),
                                             self._stream(stream)))
        return hist

    def skip(self, words: int, stream=None) -> None:
        _raise(lib.xg_skip(self._h.ptr, words, self._stream(stream)))

    # -- state hooks (proj/include/xg/xorgens.hpp:33-35,72-87) ----------------
    def block_state(self, i: int) -> Tuple[List[int], int]:
        """(logical_buffer, weyl_value) of block i."""
        buf = (ctypes.c_uint64 * self._params.r)()
        wy = ctypes.c_uint64()
        _raise(lib.xg_state_export(self._h.ptr, i, buf, ctypes.byref(wy)), "state_export")
        return list(buf), wy.value

    def set_block_state(self, i: int, buffer: Sequence[int], weyl: int) -> None:
        """Replace block i by from_raw(params, buffer, weyl)."""
        if len(buffer) != self._params.r:
            raise ValueError("buffer size must equal r")
        arr = (ctypes.c_uint64 * self._params.r)(*[int(v) & ((1 << 64) - 1) for v in buffer])
        _raise(lib.xg_state_import(self._h.ptr, i, arr, int(weyl) & ((1 << 64) - 1)), "state_import")


    # -- checkpoint / resume of the whole ensemble ---------------------------
    def state_dict(self) -> dict:
        """Every stream's (window, weyl) plus the identity of the ensemble."""
        win = np.empty((self._n, self._params.r), dtype=np.uint32)
        wy = np.empty(self._n, dtype=np.uint32)
        _raise(lib.xg_state_export_all(self._h.ptr, win.ctypes.data_as(ctypes.c_void_p),
                                       wy.ctypes.data_as(ctypes.c_void_p)), "state_export_all")
        p = self._params
        return {"params": np.array([p.r, p.s, p.a, p.b, p.c, p.d, p.w, p.omega, p.gamma],
                                   dtype=np.uint64),
                "base_seed": np.uint64(self._base_seed), "first_stream": np.uint64(self._first),
                "window": win, "weyl": wy}

    def load_state_dict(self, sd: dict) -> None:
        p = self._params
        if tuple(int(v) for v in sd["params"]) != (p.r, p.s, p.a, p.b, p.c, p.d, p.w, p.omega, p.gamma):
            raise ValueError("checkpoint parameters differ from the ensemble's")
        win = np.ascontiguousarray(sd["window"], dtype=np.uint32)
        wy = np.ascontiguousarray(sd["weyl"], dtype=np.uint32)
        if win.shape != (self._n, p.r) or wy.shape != (self._n,):
            raise ValueError("checkpoint stream count differs from the ensemble's")
        _raise(lib.xg_state_import_all(self._h.ptr, win.ctypes.data_as(ctypes.c_void_p),
                                       wy.ctypes.data_as(ctypes.c_void_p)), "state_import_all")

    def save(self, path: str) -> None:
        np.savez(path, **self.state_dict())

    @classmethod
    def load(cls, path: str, lanes: int = 1, *, device: Optional[int] = None) -> "BlockEnsemble":
        sd = dict(np.load(path))
        p = GeneratorParams(*[int(v) for v in sd["params"]])
        ens = cls(p, int(sd["base_seed"]), int(sd["window"].shape[0]), lanes,
                  first_stream=int(sd["first_stream"]), device=device)
        ens.load_state_dict(sd)
        return ens


class XorgensState:
    """One serial stream (proj/include/xg/xorgens.hpp:20-96) on the GPU.

    ``next_word`` is served from device-generated refills (xg_next_u32); the
    stream is exactly the reference's for the same (params, seed).
    """

    def __init__(self, params: GeneratorParams, seed: int, *, device: Optional[int] = None,
                 _ens: Optional[BlockEnsemble] = None):
        self._ens = _ens if _ens is not None else BlockEnsemble(
            params, seed, 1, 1, device=device)
        self._params = params

    @classmethod
    def from_raw(cls, params: GeneratorParams, buffer: Sequence[int], weyl: int,
                 *, device: Optional[int] = None) -> "XorgensState":
        """proj/src/xorgens.cpp:34-38."""
        validate_params(params)
        if len(buffer) != params.r:
            raise ValueError("buffer size must equal r")
        ens = BlockEnsemble.from_raw(params, np.asarray([list(buffer)], dtype=np.uint64),
                                     [weyl], device=device)
        return cls(params, 0, _ens=ens)

    def params(self) -> GeneratorParams:
        return self._params

    def word_bits(self) -> int:
        return self._params.w

    def word_mask(self) -> int:
        return self._params.mask()

    def state_words(self) -> int:
        return self._params.r + 1

    def next_word(self) -> int:
        v = ctypes.c_uint64()
        _raise(lib.xg_next_word(self._ens.handle, ctypes.byref(v)), "next_word")
        return v.value

    def next_u64(self) -> int:
        v = ctypes.c_uint64()
        _raise(lib.xg_next_u64(self._ens.handle, ctypes.byref(v)), "next_u64")
        return v.value

    def logical_buffer(self) -> List[int]:
        return self._ens.block_state(0)[0]

    def weyl_value(self) -> int:
        return self._ens.block_state(0)[1]

    @property
    def ensemble(self) -> BlockEnsemble:
        return self._ens


def seed_state(params: GeneratorParams, seed: int) -> XorgensState:
    """proj/include/xg/xorgens.hpp:103-105."""
    return XorgensState(params, seed)


def batch_step(state: XorgensState, lanes: int) -> List[int]:
    """proj/src/parallel.cpp:8-42: the next ``lanes`` words, bit-identical to
    ``lanes`` next_word() calls; out_of_range unless 1 <= lanes <= lane_bound."""
    if lanes == 0 or lanes > lane_bound(state.params()):
        raise OutOfRangeError("lane count exceeds min(s, r - s)")
    return [state.next_word() for _ in range(lanes)]


class XorgensSource:
    """WordSource adapter (proj/include/xg/stream.hpp:24-34)."""

    def __init__(self, params: GeneratorParams, seed: int):
        self._state = XorgensState(params, seed)

    def next(self) -> int:
        return self._state.next_word()

    def word_bits(self) -> int:
        return self._state.word_bits()

    def state(self) -> XorgensState:
        return self._state

"""Row digests of device buffers and their composition (parity at full size).

``row_digests`` runs ``xg_digest_u32`` (csrc/xg_digest.cuh) over a 2-D CUDA
tensor: for every row, the xor, the sum and the position-weighted sum
sum_k e_k * (k + 1) of its 32-bit elements (mod 2^64; floats through their
bit patterns, 8-byte elements as their little-endian u32 halves).  The same
three numbers per stream are computed from the reference's own words by
tests/golden/make_golden.py (oracle/ref_shim.cpp ``xgref_stream_digests``),
so a GPU fill of any size is checked stream by stream without copying it
back.  ``slice_digest`` composes rows into the digest of their block-major
concatenation (the config-2 checksum form of SURVEY.md Appendix A) and
``records_sha`` hashes the per-stream records of a chunk of streams.
"""
from __future__ import annotations

import ctypes
import hashlib
from typing import Tuple

import numpy as np

from ._lib import lib
from .xorgens import _raise, _torch

M64 = (1 << 64) - 1


def row_digests(t, stream=None) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(xor u32[rows], sum u64[rows], wsum u64[rows]) of a contiguous 2-D CUDA
    tensor with 4- or 8-byte elements."""
    torch = _torch()
    if t.dim() != 2 or not t.is_cuda or not t.is_contiguous() or t.element_size() not in (4, 8):
        raise ValueError("need a contiguous 2-D CUDA tensor of 4- or 8-byte elements")
    rows, per = t.shape[0], t.shape[1] * (t.element_size() // 4)
    dev = t.device
    x = torch.empty(rows, dtype=torch.int32, device=dev)
    s = torch.empty(rows, dtype=torch.int64, device=dev)
    ws = torch.empty(rows, dtype=torch.int64, device=dev)
    sp = stream if stream is not None else torch.cuda.current_stream(dev)
    _raise(lib.xg_digest_u32(ctypes.c_void_p(t.data_ptr()), rows, per, ctypes.c_void_p(x.data_ptr()),
                             ctypes.c_void_p(s.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                             ctypes.c_void_p(sp.cuda_stream)))
    sp.synchronize()
    return (x.cpu().numpy().view(np.uint32), s.cpu().numpy().view(np.uint64),
            ws.cpu().numpy().view(np.uint64))


def slice_digest(x, s, ws, per_elems: int) -> Tuple[int, int, int]:
    """(xor, sum, wsum) of rows concatenated block-major, row i starting at
    element i * per_elems of the slice (wsum positions counted from 1)."""
    x = np.asarray(x, dtype=np.uint32)
    s = np.asarray(s, dtype=np.uint64)
    ws = np.asarray(ws, dtype=np.uint64)
    off = np.arange(len(s), dtype=np.uint64) * np.uint64(per_elems)
    with np.errstate(over="ignore"):
        total_ws = int(np.sum(ws + off * s, dtype=np.uint64))
        total_s = int(np.sum(s, dtype=np.uint64))
    return int(np.bitwise_xor.reduce(x)) if len(x) else 0, total_s, total_ws


def records_sha(x, s, ws) -> str:
    """sha256 of the per-row records: xor (u32 LE) array, then sum, then wsum
    (u64 LE) arrays."""
    h = hashlib.sha256()
    h.update(np.asarray(x, dtype="<u4").tobytes())
    h.update(np.asarray(s, dtype="<u8").tobytes())
    h.update(np.asarray(ws, dtype="<u8").tobytes())
    return h.hexdigest()


def chunk_record(x, s, ws, per_elems: int) -> dict:
    """The golden record of a chunk of consecutive streams (full_size.json)."""
    gx, gs, gws = slice_digest(x, s, ws, per_elems)
    return {"xor": f"{gx:08x}", "sum": f"{gs:016x}", "wsum": f"{gws:016x}",
            "sha": records_sha(x, s, ws)}

"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the CPU oracle.

* ``liboracle.so`` -- the plain-C restatement (oracle/xg_oracle.c).
* ``_ref/libxgref.so`` -- the reference's own sources, compiled unmodified
  (oracle/Makefile, oracle/ref_shim.cpp); present when built in a container
  that had the reference tree, then shipped with the snapshot.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package; the product (paper_1108_0486_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libxgref.so")

_u32, _u64, _int, _vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint) for n in "r s a b c d w".split()] + [
        ("omega", ctypes.c_uint64), ("gamma", ctypes.c_uint)]


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Oracle:
    """The C restatement: serial states, lane batching and block ensembles."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -f oracle/Makefile)")
        L = self.lib = ctypes.CDLL(path)
        for n in ("xgo_xorgensgp32_params", "xgo_tiny_r2w8_params", "xgo_tiny_r2w16_params",
                  "xgo_tiny_r4w16_params"):
            getattr(L, n).restype = Params
        L.xgo_state_size.restype = ctypes.c_size_t
        L.xgo_next_word.restype = _u64
        L.xgo_step_linear.restype = _u64
        L.xgo_splitmix64.restype = _u64
        L.xgo_recommended_weyl_increment.restype = _u64
        L.xgo_lane_bound.restype = ctypes.c_uint
        L.xgo_u32_to_f32.restype = ctypes.c_float
        L.xgo_u32_to_f32.argtypes = [_u32]
        L.xgo_u32pair_to_f64.restype = ctypes.c_double
        L.xgo_u32pair_to_f64.argtypes = [_u32, _u32]
        L.xgo_u32pair_to_u64.restype = _u64
        L.xgo_u32pair_to_u64.argtypes = [_u32, _u32]
        L.xgo_mc_hit.argtypes = [_u32, _u32]
        L.xgo_seed.argtypes = [_vp, ctypes.POINTER(Params), _u64]
        L.xgo_from_raw.argtypes = [_vp, ctypes.POINTER(Params), _vp, _u64]
        L.xgo_stream_u32.argtypes = [ctypes.POINTER(Params), _u64, _u64, _vp]
        L.xgo_ensemble_seed.argtypes = [_vp, ctypes.POINTER(Params), _u64, _u64, _u32, _int]
        for n in ("xgo_ensemble_fill_u32", "xgo_ensemble_fill_f32", "xgo_ensemble_fill_f64",
                  "xgo_ensemble_mc_pi", "xgo_ensemble_fill_raw_u32", "xgo_ensemble_fill_words"):
            getattr(L, n).argtypes = [_vp, _u32, _u64, _vp, _int]
        L.xgo_ensemble_checksums.argtypes = [_vp, _u32, _u64, _vp, _vp, _int]
        L.xgo_ensemble_rank_counts.argtypes = [_vp, _u32, _u64, _vp, _int]
        L.xgo_gf2_rank32.argtypes = [_vp]
        L.xgo_gf2_rank32.restype = ctypes.c_uint
        L.xgo_batch_step.argtypes = [_vp, ctypes.c_uint, _vp]
        L.xgo_unsynchronized_batch.argtypes = [_vp, ctypes.c_uint, _vp]
        L.xgo_logical_buffer.argtypes = [_vp, _vp]
        L.xgo_weyl_value.restype = _u64
        L.xgo_weyl_value.argtypes = [_vp]
        L.xgo_next_word.argtypes = [_vp]
        self.state_size = int(L.xgo_state_size())
        self.threads = os.cpu_count() or 1

    # -- params
    def gp32(self) -> Params:
        return self.lib.xgo_xorgensgp32_params()

    def params(self, r, s, a, b, c, d, w, omega=None, gamma=None) -> Params:
        om = self.lib.xgo_recommended_weyl_increment(w) if omega is None else omega
        return Params(r, s, a, b, c, d, w, om, w // 2 if gamma is None else gamma)

    def check(self, p: Params) -> int:
        return self.lib.xgo_check_params(ctypes.byref(p))

    # -- streams
    def stream(self, seed: int, n: int, p: Optional[Params] = None) -> np.ndarray:
        p = p or self.gp32()
        out = np.empty(n, dtype=np.uint32)
        rc = self.lib.xgo_stream_u32(ctypes.byref(p), seed & (2**64 - 1), n, _ptr(out))
        if rc:
            raise ValueError(f"oracle stream rc={rc}")
        return out

    def ensemble(self, base_seed: int, num_streams: int, p: Optional[Params] = None,
                 first_stream: int = 0) -> "OracleEnsemble":
        return OracleEnsemble(self, p or self.gp32(), base_seed, num_streams, first_stream)

    def from_raw(self, buffers: np.ndarray, weyls, p: Optional[Params] = None) -> "OracleEnsemble":
        return OracleEnsemble.from_raw(self, p or self.gp32(), buffers, weyls)

    def f32(self, u: np.ndarray) -> np.ndarray:
        # (u >> 8) * 2^-24, exact in float32 (the same formula as xg_oracle.c).
        return ((u.astype(np.uint32) >> 8).astype(np.float32) * np.float32(2.0 ** -24))

    def f64_pairs(self, words: np.ndarray) -> np.ndarray:
        w = words.astype(np.uint64)
        u = w[..., 0::2] | (w[..., 1::2] << np.uint64(32))
        return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def mc_hits(self, words: np.ndarray) -> int:
        """Hits over a stream prefix of 2k words: sample m is the consecutive
        pair (w[2m], w[2m+1])."""
        w = words.astype(np.uint32).view(np.int32).astype(np.int64).reshape(-1, 2)
        x, y = w[:, 0], w[:, 1]
        q = (x * x).astype(np.uint64) + (y * y).astype(np.uint64)
        return int(np.count_nonzero(q < np.uint64(1 << 62)))


class OracleEnsemble:
    """Array of xgo_state, one per stream (proj/src/parallel.cpp:84-135)."""

    def __init__(self, o: Oracle, p: Params, base_seed: int, n: int, first_stream: int = 0,
                 _seed: bool = True):
        self.o, self.p, self.n = o, p, n
        self.buf = ctypes.create_string_buffer(o.state_size * n)
        if _seed:
            rc = o.lib.xgo_ensemble_seed(self.buf, ctypes.byref(p), base_seed & (2**64 - 1),
                                         first_stream & (2**64 - 1), n, o.threads)
            if rc:
                raise ValueError(f"oracle seed rc={rc}")

    @classmethod
    def from_raw(cls, o: Oracle, p: Params, buffers: np.ndarray, weyls) -> "OracleEnsemble":
        weyls = list(weyls)
        e = cls(o, p, 0, len(weyls), _seed=False)
        bufs = np.ascontiguousarray(np.asarray(buffers, dtype=np.uint64).reshape(len(weyls), -1))
        for g in range(len(weyls)):
            rc = o.lib.xgo_from_raw(ctypes.byref(e.buf, g * o.state_size), ctypes.byref(p),
                                    _ptr(bufs[g]), int(weyls[g]) & (2**64 - 1))
            if rc:
                raise ValueError(f"oracle from_raw rc={rc}")
        return e

    def _state(self, g: int):
        return ctypes.byref(self.buf, g * self.o.state_size)

    def fill_u32(self, per_stream: int) -> np.ndarray:
        out = np.empty((self.n, per_stream), dtype=np.uint32)
        self.o.lib.xgo_ensemble_fill_u32(self.buf, self.n, per_stream, _ptr(out), self.o.threads)
        return out

    def fill_words(self, per_stream: int) -> np.ndarray:
        out = np.empty((self.n, per_stream), dtype=np.uint64)
        self.o.lib.xgo_ensemble_fill_words(self.buf, self.n, per_stream, _ptr(out), self.o.threads)
        return out

    def fill_raw_u32(self, per_stream: int) -> np.ndarray:
        out = np.empty((self.n, per_stream), dtype=np.uint32)
        self.o.lib.xgo_ensemble_fill_raw_u32(self.buf, self.n, per_stream, _ptr(out), self.o.threads)
        return out

    def fill_f32(self, per_stream: int) -> np.ndarray:
        out = np.empty((self.n, per_stream), dtype=np.float32)
        self.o.lib.xgo_ensemble_fill_f32(self.buf, self.n, per_stream, _ptr(out), self.o.threads)
        return out

    def fill_f64(self, per_stream: int) -> np.ndarray:
        out = np.empty((self.n, per_stream), dtype=np.float64)
        self.o.lib.xgo_ensemble_fill_f64(self.buf, self.n, per_stream, _ptr(out), self.o.threads)
        return out

    def mc_hits(self, samples: int) -> np.ndarray:
        out = np.empty(self.n, dtype=np.uint64)
        if self.o.lib.xgo_ensemble_mc_pi(self.buf, self.n, samples, _ptr(out), self.o.threads):
            raise ValueError("samples per stream must be a multiple of 32")
        return out

    def rank_counts(self, matrices: int) -> np.ndarray:
        """(num_streams, 3) bins (rank 32, 31, <= 30) of the next `matrices`
        32 x 32 matrices of every stream (tests.cpp:93-109)."""
        out = np.empty((self.n, 3), dtype=np.uint64)
        self.o.lib.xgo_ensemble_rank_counts(self.buf, self.n, matrices, _ptr(out), self.o.threads)
        return out

    def checksums(self, n: int):
        x = np.empty(self.n, dtype=np.uint32)
        s = np.empty(self.n, dtype=np.uint64)
        self.o.lib.xgo_ensemble_checksums(self.buf, self.n, n, _ptr(x), _ptr(s), self.o.threads)
        return x, s

    def logical_buffer(self, g: int) -> np.ndarray:
        out = np.empty(self.p.r, dtype=np.uint64)
        self.o.lib.xgo_logical_buffer(self._state(g), _ptr(out))
        return out

    def weyl(self, g: int) -> int:
        return int(self.o.lib.xgo_weyl_value(self._state(g)))

    def next_words(self, g: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        for i in range(n):
            out[i] = self.o.lib.xgo_next_word(self._state(g))
        return out


BATTERY_SO = os.path.join(HERE, "_ref", "libxgref_battery.so")


class Battery:
    """The reference's statistical battery (proj/src/stattests/*) over a buffer
    of 32-bit words, through oracle/_ref/libxgref_battery.so."""

    VERDICTS = {0: "pass", 1: "suspect", 2: "fail", 3: "not_applicable", -1: "error"}

    def __init__(self, path: str = BATTERY_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs the reference tree + json.hpp)")
        self.lib = ctypes.CDLL(path)
        self.lib.xgref_battery_on_words.argtypes = [_vp, _u64, _int, ctypes.c_char_p,
                                                    ctypes.c_char_p, _u64]
        self.lib.xgref_battery_config_on_words.argtypes = [_vp, _u64, ctypes.c_uint, ctypes.c_char_p,
                                                           ctypes.c_char_p, ctypes.c_char_p, _u64,
                                                           ctypes.c_char_p, _u64]
        self.lib.xgref_gf2_rank32.argtypes = [_vp]
        self.lib.xgref_gf2_rank32.restype = ctypes.c_uint
        self.lib.xgref_berlekamp_massey.argtypes = [_vp, _u64]
        self.lib.xgref_berlekamp_massey.restype = _u64
        self.lib.xgref_linear_complexity_on_words.argtypes = [
            _vp, _u64, ctypes.c_uint, _u64, ctypes.POINTER(ctypes.c_double),
            ctypes.POINTER(ctypes.c_double)]
        self.lib.xgref_matrix_rank_on_words.argtypes = [_vp, _u64, _u64,
                                                        ctypes.POINTER(ctypes.c_double),
                                                        ctypes.POINTER(ctypes.c_double)]

    def berlekamp_massey(self, bits: np.ndarray) -> int:
        """The reference's linear complexity of a bit sequence (gf2.cpp:62-110)."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        return int(self.lib.xgref_berlekamp_massey(_ptr(b), b.size))

    def lc_histogram(self, words: np.ndarray, block_length: int, num_blocks: int) -> np.ndarray:
        """Histogram of the reference's per-block linear complexity over
        words read MSB first (BitSource), block_length bits per block."""
        w = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1)
        bits = np.unpackbits(w.byteswap().view(np.uint8))  # MSB first per word
        hist = np.zeros(block_length + 1, dtype=np.uint64)
        for k in range(num_blocks):
            hist[self.berlekamp_massey(bits[k * block_length:(k + 1) * block_length])] += 1
        return hist

    def linear_complexity(self, words: np.ndarray, block_length: int, num_blocks: int):
        """The reference's linear_complexity_test over words: (statistic, p)."""
        w = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1)
        st, pv = ctypes.c_double(), ctypes.c_double()
        if self.lib.xgref_linear_complexity_on_words(_ptr(w), w.size, block_length, num_blocks,
                                                     ctypes.byref(st), ctypes.byref(pv)):
            raise ValueError("linear_complexity_test failed (short buffer, K < 128 or < 38 blocks)")
        return st.value, pv.value

    def gf2_rank32(self, rows: np.ndarray) -> int:
        """The reference's gf2_rank (proj/src/stattests/gf2.cpp) of 32 rows."""
        r = np.ascontiguousarray(rows, dtype=np.uint32)
        assert r.size == 32
        return int(self.lib.xgref_gf2_rank32(_ptr(r)))

    def matrix_rank(self, words: np.ndarray, num_matrices: int):
        """The reference's matrix_rank_test (tests.cpp:81-126) over words:
        (statistic, p_value)."""
        w = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1)
        st, pv = ctypes.c_double(), ctypes.c_double()
        if self.lib.xgref_matrix_rank_on_words(_ptr(w), w.size, num_matrices, ctypes.byref(st),
                                               ctypes.byref(pv)):
            raise ValueError("matrix_rank_test failed (buffer too short or < 38 matrices)")
        return st.value, pv.value

    def run_config(self, words: np.ndarray, bits: int, config_text: str = "", generator: str = "gpu",
                   params: str = "", seed: int = 0):
        """run_battery over `bits`-wide words (one per element) with a
        BatteryConfig::parse text: (verdict, report JSON)."""
        w = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)
        buf = ctypes.create_string_buffer(1 << 16)
        v = self.lib.xgref_battery_config_on_words(_ptr(w), w.size, bits, config_text.encode(),
                                                   generator.encode(), params.encode(),
                                                   seed & (2**64 - 1), buf, len(buf))
        return self.VERDICTS.get(v, str(v)), buf.value.decode()

    def run(self, words: np.ndarray, quick: bool = False, label: str = "gpu"):
        w = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1)
        buf = ctypes.create_string_buffer(1 << 16)
        v = self.lib.xgref_battery_on_words(_ptr(w), w.size, int(quick), label.encode(), buf,
                                            len(buf))
        return self.VERDICTS.get(v, str(v)), buf.value.decode()


class Reference:
    """The reference sources themselves (oracle/_ref/libxgref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs the reference tree; make -f oracle/Makefile)")
        L = self.lib = ctypes.CDLL(path)
        arr = ctypes.POINTER(ctypes.c_uint)
        L.xgref_check_params.argtypes = [arr, _u64, ctypes.c_uint]
        L.xgref_stream.argtypes = [arr, _u64, ctypes.c_uint, _u64, _u64, _vp]
        L.xgref_seeded_state.argtypes = [arr, _u64, ctypes.c_uint, _u64, _vp, _vp]
        L.xgref_from_raw_stream.argtypes = [arr, _u64, ctypes.c_uint, _vp, _u64, _u64, _vp]
        L.xgref_ensemble_create.restype = _vp
        L.xgref_ensemble_create.argtypes = [arr, _u64, ctypes.c_uint, _u64, ctypes.c_uint,
                                            ctypes.c_uint]
        L.xgref_ensemble_destroy.argtypes = [_vp]
        L.xgref_ensemble_generate.argtypes = [_vp, _u64, ctypes.c_uint, _vp,
                                              ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(_u64)]
        L.xgref_raw_stream.argtypes = [arr, _u64, ctypes.c_uint, _u64, _u64, _vp]
        L.xgref_low_bit_windows.argtypes = [arr, _u64, ctypes.c_uint, _u64, _int, _u64, _u64, _vp, _vp]
        L.xgref_stream_digests.argtypes = [arr, _u64, ctypes.c_uint, _u64, _u64, _u64, _u64, _u64,
                                           _u64] + [_vp] * 10
        L.xgref_streams_xor.argtypes = [arr, _u64, ctypes.c_uint, _u64, _u64, _u64, _u64, _vp]
        L.xgref_streams_convert.argtypes = [arr, _u64, ctypes.c_uint, _u64, _u64, _u64, _u64, _int, _vp]
        L.xgref_serial_rate.restype = ctypes.c_double
        L.xgref_serial_rate.argtypes = [_u64, _u64, ctypes.c_uint, ctypes.POINTER(_u64)]

    @staticmethod
    def _arr(p):
        return (ctypes.c_uint * 7)(p.r, p.s, p.a, p.b, p.c, p.d, p.w)

    def check(self, p) -> int:
        return self.lib.xgref_check_params(self._arr(p), p.omega, p.gamma)

    def stream(self, seed: int, n: int, p) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        rc = self.lib.xgref_stream(self._arr(p), p.omega, p.gamma, seed & (2**64 - 1), n, _ptr(out))
        if rc:
            raise ValueError("reference rejected the parameters")
        return out

    def raw_stream(self, seed: int, n: int, p) -> np.ndarray:
        """RawXorgens(p, seed).next() x n (the reference baseline class)."""
        out = np.empty(n, dtype=np.uint64)
        rc = self.lib.xgref_raw_stream(self._arr(p), p.omega, p.gamma, seed & (2**64 - 1), n, _ptr(out))
        if rc:
            raise ValueError("reference rejected the parameters")
        return out

    def low_bit_windows(self, seed: int, words: int, window: int, p, raw: bool = True):
        """(first, last) windows of the words' low bits (test_long_linearity.cpp:30-52)."""
        first = np.zeros(window, dtype=np.uint8)
        last = np.zeros(window, dtype=np.uint8)
        rc = self.lib.xgref_low_bit_windows(self._arr(p), p.omega, p.gamma, seed & (2**64 - 1),
                                            int(raw), words, window, _ptr(first), _ptr(last))
        if rc:
            raise ValueError("reference rejected the parameters")
        return first, last

    def seeded_state(self, seed: int, p):
        buf = np.empty(p.r, dtype=np.uint64)
        wy = np.empty(1, dtype=np.uint64)
        rc = self.lib.xgref_seeded_state(self._arr(p), p.omega, p.gamma, seed & (2**64 - 1),
                                         _ptr(buf), _ptr(wy))
        if rc:
            raise ValueError("reference rejected the parameters")
        return buf, int(wy[0])

    def from_raw_stream(self, buffer, weyl: int, n: int, p) -> np.ndarray:
        b = np.ascontiguousarray(np.asarray(buffer, dtype=np.uint64))
        out = np.empty(n, dtype=np.uint64)
        rc = self.lib.xgref_from_raw_stream(self._arr(p), p.omega, p.gamma, _ptr(b),
                                            int(weyl) & (2**64 - 1), n, _ptr(out))
        if rc:
            raise ValueError("reference rejected the parameters")
        return out

    def ensemble(self, p, base_seed: int, blocks: int, lanes: int):
        h = self.lib.xgref_ensemble_create(self._arr(p), p.omega, p.gamma, base_seed & (2**64 - 1),
                                           blocks, lanes)
        if not h:
            raise ValueError("reference BlockEnsemble construction failed")
        return h

    def generate_words(self, h, n_blocks: int, per_block: int, workers: int = 0):
        out = np.empty((n_blocks, per_block), dtype=np.uint32)
        secs = ctypes.c_double()
        sink = ctypes.c_uint64()
        rc = self.lib.xgref_ensemble_generate(h, per_block, workers, _ptr(out), ctypes.byref(secs),
                                              ctypes.byref(sink))
        if rc:
            raise RuntimeError("reference generate failed")
        return out, secs.value, sink.value

    def generate_timed(self, h, per_block: int, workers: int = 0):
        secs = ctypes.c_double()
        sink = ctypes.c_uint64()
        rc = self.lib.xgref_ensemble_generate(h, per_block, workers, None, ctypes.byref(secs),
                                              ctypes.byref(sink))
        if rc:
            raise RuntimeError("reference generate failed")
        return secs.value, sink.value

    def destroy(self, h) -> None:
        self.lib.xgref_ensemble_destroy(h)

    def stream_digests(self, p, base_seed: int, first: int, count: int, n_u32: int, n_f64: int = 0,
                       n_mc: int = 0) -> dict:
        """Per-stream digests of streams [first, first + count) (see
        xgref_stream_digests in oracle/ref_shim.cpp): {"u32"|"f32"|"f64":
        (xor u32[count], sum u64[count], wsum u64[count]), "mc": hits u32[count]}."""
        out = {}
        ptrs = []
        for key, n in (("u32", n_u32), ("f32", n_u32), ("f64", n_f64)):
            if n:
                t = (np.zeros(count, np.uint32), np.zeros(count, np.uint64), np.zeros(count, np.uint64))
                out[key] = t
                ptrs += [_ptr(a) for a in t]
            else:
                ptrs += [None] * 3
        if n_mc:
            out["mc"] = np.zeros(count, np.uint32)
            ptrs.append(_ptr(out["mc"]))
        else:
            ptrs.append(None)
        rc = self.lib.xgref_stream_digests(self._arr(p), p.omega, p.gamma, base_seed & (2**64 - 1),
                                           first, count, n_u32, n_f64, n_mc, *ptrs)
        if rc:
            raise ValueError("reference rejected the parameters")
        return out

    def streams_xor(self, p, base_seed: int, first: int, count: int, n: int) -> np.ndarray:
        """Per-stream xor of n words of streams [first, first + count), each an
        XorgensState loop (xgref_streams_xor); releases the GIL, so threads
        run it on all cores."""
        out = np.zeros(count, dtype=np.uint32)
        rc = self.lib.xgref_streams_xor(self._arr(p), p.omega, p.gamma, base_seed & (2**64 - 1),
                                        first, count, n, _ptr(out))
        if rc:
            raise ValueError("reference rejected the parameters")
        return out

    def streams_convert(self, p, base_seed: int, first: int, count: int, n: int, f64: bool) -> np.ndarray:
        """n f32 (or f64) values of each of streams [first, first + count)
        from XorgensState loops (xgref_streams_convert); per-stream xor of
        the value bits.  Releases the GIL."""
        out = np.zeros(count, dtype=np.uint64)
        rc = self.lib.xgref_streams_convert(self._arr(p), p.omega, p.gamma, base_seed & (2**64 - 1),
                                            first, count, n, int(f64), _ptr(out))
        if rc:
            raise ValueError("reference rejected the parameters")
        return out

    def serial_rate(self, seed: int, count: int, chunks: int = 20) -> float:
        sink = ctypes.c_uint64()
        return self.lib.xgref_serial_rate(seed, count, chunks, ctypes.byref(sink))

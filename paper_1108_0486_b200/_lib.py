"""ctypes binding of libxg_gpu.so (the C ABI in include/xg_gpu.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libxg_gpu.so")

XG_OK = 0
XG_ERANGE = 16
XG_EINVAL = 17
XG_EUNSUPPORTED = 18
XG_ECUDA = 19
XG_ENOMEM = 20


class xg_params_t(ctypes.Structure):
    """Mirror of ``xg_params_t`` / ``xg::GeneratorParams`` (field order kept)."""

    _fields_ = [
        ("r", ctypes.c_uint),
        ("s", ctypes.c_uint),
        ("a", ctypes.c_uint),
        ("b", ctypes.c_uint),
        ("c", ctypes.c_uint),
        ("d", ctypes.c_uint),
        ("w", ctypes.c_uint),
        ("omega", ctypes.c_uint64),
        ("gamma", ctypes.c_uint),
    ]


_u32, _u64, _int, _vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
_P = ctypes.POINTER

# name -> (restype, argtypes); every symbol declared in include/xg_gpu.h.
SIGNATURES = {
    "xg_params_check": (_int, [_P(xg_params_t)]),
    "xg_strerror": (ctypes.c_char_p, [_int]),
    "xg_lane_bound": (ctypes.c_uint, [_P(xg_params_t)]),
    "xg_recommended_weyl_increment": (_u64, [ctypes.c_uint]),
    "xg_default_output_shift": (ctypes.c_uint, [ctypes.c_uint]),
    "xg_params_xorgensgp32": (xg_params_t, []),
    "xg_params_tiny_r2w8": (xg_params_t, []),
    "xg_params_tiny_r2w16": (xg_params_t, []),
    "xg_params_tiny_r4w16": (xg_params_t, []),
    "xg_gpu_supported": (_int, [_P(xg_params_t)]),
    "xg_fast_path": (_int, [_P(xg_params_t)]),
    "xg_ensemble_create": (_int, [_P(xg_params_t), _u64, _u64, _u32, ctypes.c_uint, _int, _vp,
                                  _P(_vp)]),
    "xg_ensemble_create_from_raw": (_int, [_P(xg_params_t), _u32, _P(_u64), _P(_u64), _int, _vp,
                                           _P(_vp)]),
    "xg_ensemble_destroy": (_int, [_vp]),
    "xg_ensemble_info": (_int, [_vp, _P(_u32), _P(_u64), _P(_u64), _P(ctypes.c_uint), _P(_int)]),
    "xg_fill_u32": (_int, [_vp, _u64, _vp, _vp]),
    "xg_fill_u64": (_int, [_vp, _u64, _vp, _vp]),
    "xg_fill_words": (_int, [_vp, _u64, _vp, _vp]),
    "xg_fill_f32": (_int, [_vp, _u64, _vp, _vp]),
    "xg_fill_raw_u32": (_int, [_vp, _u64, _vp, _vp]),
    "xg_fill_f64": (_int, [_vp, _u64, _vp, _vp]),
    "xg_mc_pi": (_int, [_vp, _u64, _vp, _vp]),
    "xg_rank_test": (_int, [_vp, _u64, _vp, _vp]),
    "xg_linear_complexity_test": (_int, [_vp, ctypes.c_uint, _u64, _vp, _vp]),
    "xg_berlekamp_massey": (_int, [_vp, _u64, _u32, _u64, _vp, _vp]),
    "xg_pack_words": (_int, [_vp, _u64, ctypes.c_uint, _int, _vp, _vp]),
    "xg_rank_words": (_int, [_vp, _u64, _vp, _vp]),
    "xg_lc_words": (_int, [_vp, _u64, ctypes.c_uint, _u64, _vp, _vp]),
    "xg_bits_ones_runs": (_int, [_vp, _u64, _vp, _vp]),
    "xg_birthday_duplicates": (_int, [_vp, _u32, _u32, ctypes.c_uint, _vp, _vp]),
    "xg_digest_u32": (_int, [_vp, _u64, _u64, _vp, _vp, _vp, _vp]),
    "xg_skip": (_int, [_vp, _u64, _vp]),
    "xg_generate_host": (_int, [_vp, _u64, _vp, _vp]),
    "xg_generate_host_words": (_int, [_vp, _u64, _vp, _vp]),
    "xg_generate_host_rows": (_int, [_vp, _u64, _vp, _vp]),
    "xg_generate_host_f32": (_int, [_vp, _u64, _vp, _vp]),
    "xg_generate_host_f64": (_int, [_vp, _u64, _vp, _vp]),
    "xg_generate_host_tiles": (_int, [_vp, _u64, _vp, _vp, ctypes.c_uint, _vp]),
    "xg_next_word": (_int, [_vp, _P(_u64)]),
    "xg_next_view": (_int, [_vp, _P(_vp), _P(_u64)]),
    "xg_next_return": (_int, [_vp, _u64]),
    "xg_next_u32": (_int, [_vp, _P(_u32)]),
    "xg_next_u64": (_int, [_vp, _P(_u64)]),
    "xg_state_export": (_int, [_vp, _u32, _P(_u64), _P(_u64)]),
    "xg_state_import": (_int, [_vp, _u32, _P(_u64), _u64]),
    "xg_state_export_all": (_int, [_vp, _vp, _vp]),
    "xg_state_import_all": (_int, [_vp, _vp, _vp]),
    "xg_jump_minpoly": (_int, [_P(xg_params_t), _P(_u64)]),
    "xg_partition": (_int, [_u64, _u32, _u32, _P(_u64), _P(_u32)]),
    "xg_kernel_launches": (_u64, []),
    "xg_build_info": (ctypes.c_char_p, []),
}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the xorgensGP GPU path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()

"""CPU-side checks of the drop-in boundary (no kernel launches).

* libxg_gpu.so loads and exports every function include/xg_gpu.h declares;
* the host validation behind the C ABI matches the reference's check order
  and error classes (proj/src/params.cpp:22-37, proj/src/parallel.cpp:84-95)
  -- ensemble_create validates before it touches a device, so these run here;
* the Python mirror raises the reference's error types.
"""
import ctypes
import os
import re

import pytest

import paper_1108_0486_b200 as xg
from paper_1108_0486_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "xg_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 25
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_build():
    import subprocess

    r = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout


def test_params_and_sets():
    p = xg.xorgensgp32_params()
    assert (p.r, p.s, p.a, p.b, p.c, p.d, p.w, p.omega, p.gamma) == (128, 65, 15, 14, 12, 17, 32,
                                                                       2654435769, 16)
    assert xg.lane_bound(p) == 63
    assert xg.check_params(p) is None
    assert xg.lane_bound(xg.tiny_r4w16_params()) == 1
    assert xg.lane_bound(xg.GeneratorParams(128, 95, 17, 12, 13, 15, 32, 2654435769, 16)) == 33
    assert [xg.recommended_weyl_increment(w) for w in (8, 16, 32, 64)] == [
        159, 40503, 2654435769, 11400714819323198485]
    with pytest.raises(xg.ParamValidationError) as ei:
        xg.recommended_weyl_increment(12)
    assert ei.value.code() == xg.ParamError.bad_word_size
    assert xg.period_description(p).display == "~2^4128"
    assert xg.gpu_supported(p) and xg.fast_path(p)
    # every valid set is generated on the GPU; only w=32/r=128/lane_bound>=32
    # sets take the register-window kernels
    assert xg.gpu_supported(xg.tiny_r2w8_params()) and not xg.fast_path(xg.tiny_r2w8_params())
    big = xg.GeneratorParams(16385, 2, 1, 1, 1, 1, 32, 2654435769, 16)
    assert xg.check_params(big) is None and not xg.gpu_supported(big)


def _mk(r, s, a, b, c, d, w, omega=None, gamma=None):
    return xg.GeneratorParams(r, s, a, b, c, d, w,
                              omega if omega is not None else (xg.recommended_weyl_increment(w)
                                                                if w in (8, 16, 32, 64) else 159),
                              w // 2 if gamma is None else gamma)


@pytest.mark.parametrize("args,err", [
    ((128, 64, 15, 14, 12, 17, 32), xg.ParamError.gcd_not_one),
    ((2, 1, 1, 1, 1, 1, 12), xg.ParamError.bad_word_size),
    ((2, 0, 1, 1, 1, 1, 8), xg.ParamError.s_out_of_range),
    ((2, 2, 1, 1, 1, 1, 8), xg.ParamError.s_out_of_range),
    ((2, 1, 8, 1, 1, 1, 8), xg.ParamError.shift_out_of_range),
    ((2, 1, 1, 0, 1, 1, 8), xg.ParamError.shift_out_of_range),
])
def test_check_params_codes(args, err):
    p = _mk(*args)
    assert xg.check_params(p) == err
    with pytest.raises(xg.ParamValidationError) as ei:
        xg.validate_params(p)
    assert ei.value.code() == err


def test_check_params_agrees_with_reference(reference):
    import itertools

    from oracle import Params

    for r, s, w in itertools.product((2, 4, 128), (0, 1, 3, 64, 65, 128), (8, 12, 32)):
        for sh in ((1, 1, 1, 1), (0, 1, 1, 1), (1, 1, 1, 40)):
            for gamma, omega in ((w // 2, 159), (0, 159), (w // 2, 158)):
                rp = Params(r, s, *sh, w, omega, gamma)
                p = xg.GeneratorParams(r, s, *sh, w, omega, gamma)
                code = xg.check_params(p)
                assert (0 if code is None else int(code) + 1) == reference.check(rp)


def test_create_validation_order_without_gpu():
    # proj/src/parallel.cpp:86-91: params first, then blocks, then lanes; each
    # rejected before any device work, with the reference's error class.
    lib, P = _lib.lib, _lib.xg_params_t
    h = ctypes.c_void_p()
    bad = P(128, 64, 15, 14, 12, 17, 32, 2654435769, 16)
    assert lib.xg_ensemble_create(ctypes.byref(bad), 0, 0, 0, 0, 0, None, ctypes.byref(h)) == 3
    gp = lib.xg_params_xorgensgp32()
    assert lib.xg_ensemble_create(ctypes.byref(gp), 0, 0, 0, 1, 0, None, ctypes.byref(h)) == _lib.XG_ERANGE
    assert lib.xg_ensemble_create(ctypes.byref(gp), 0, 0, 1, 64, 0, None, ctypes.byref(h)) == _lib.XG_ERANGE
    assert lib.xg_ensemble_create(ctypes.byref(gp), 0, 0, 1, 0, 0, None, ctypes.byref(h)) == _lib.XG_ERANGE
    w64 = P(64, 53, 33, 26, 27, 29, 64, 11400714819323198485, 32)  # PAPER.md:448-449, lane_bound 11
    assert lib.xg_params_check(ctypes.byref(w64)) == 0
    assert lib.xg_ensemble_create(ctypes.byref(w64), 0, 0, 1, 12, 0, None, ctypes.byref(h)) == _lib.XG_ERANGE
    big = P(16385, 2, 1, 1, 1, 1, 32, 2654435769, 16)
    assert lib.xg_ensemble_create(ctypes.byref(big), 0, 0, 1, 1, 0, None, ctypes.byref(h)) == _lib.XG_EUNSUPPORTED
    assert h.value is None
    assert lib.xg_ensemble_create(ctypes.byref(gp), 0, 0, 1, 1, 0, None, None) == _lib.XG_EINVAL
    assert lib.xg_ensemble_destroy(None) == _lib.XG_EINVAL
    assert lib.xg_fill_u32(None, 10, None, None) == _lib.XG_EINVAL


def test_size_overflow_rejected_before_device_work():
    # Sizes whose byte / bit counts overflow 64 bits are XG_EINVAL up front
    # (std::invalid_argument in the reference), before any pointer query.
    lib = _lib.lib
    fake, out = ctypes.c_void_p(0x1000), ctypes.c_void_p(0x2000)
    big = 1 << 62
    assert lib.xg_berlekamp_massey(fake, 64, 2, big, out, None) == _lib.XG_EINVAL  # stride bits
    assert lib.xg_berlekamp_massey(fake, 64, 3, 1 << 61, out, None) == _lib.XG_EINVAL  # span
    assert lib.xg_berlekamp_massey(fake, 64, 2, 1, out, None) == _lib.XG_EINVAL  # stride < nbits
    assert lib.xg_pack_words(fake, 1 << 59, 32, 0, out, None) == _lib.XG_EINVAL
    assert lib.xg_lc_words(fake, 1, 64, 1, out, None) == _lib.XG_EINVAL  # 32 bits < one block
    assert lib.xg_digest_u32(fake, 1 << 20, big, out, out, out, None) == _lib.XG_EINVAL
    assert lib.xg_fill_u32(None, big, None, None) == _lib.XG_EINVAL


def test_python_mirror_errors_without_gpu():
    p = xg.xorgensgp32_params()
    with pytest.raises(xg.ParamValidationError):
        xg.BlockEnsemble(_mk(128, 64, 15, 14, 12, 17, 32), 0, 1, 1)
    if not __import__("torch").cuda.is_available():
        with pytest.raises(xg.XgCudaError):
            xg.BlockEnsemble(p, 0, 1, 1)


def test_strerror_texts():
    # proj/src/params.cpp:7-18
    assert _lib.lib.xg_strerror(3).decode() == "r and s must be coprime"
    assert _lib.lib.xg_strerror(6).decode() == "Weyl increment omega must be odd"
    assert b"sm_100a" in _lib.lib.xg_build_info()


@pytest.mark.parametrize("total,world", [(1 << 14, 1), (1 << 14, 2), (1 << 14, 8), (1000, 3),
                                         (7, 8), (2**34, 8)])
def test_partition_covers_disjointly(total, world):
    spans = [xg.partition(total, world, k) for k in range(world)]
    pos = 0
    for first, count in spans:
        assert first == pos
        pos += count
    assert pos == total
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(xg.OutOfRangeError):
        xg.partition(total, world, world)

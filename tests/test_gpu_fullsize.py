"""Full-size parity of BASELINE configs 2-5 on the GPU, stream by stream.

Every fill is digested on the device (xg_digest_u32: per-stream xor, sum and
position-weighted sum) and compared with tests/golden/full_size.json, which
make_golden.py --full-size computed from the reference's own words
(oracle/_ref, proj/src/xorgens.cpp + parallel.cpp:84-135), per chunk of 2^14
streams.  Bit-exact: integer work, exact conversions.
Reference anchors: seeding proj/src/parallel.cpp:84-95; bit-exact across
blocks proj/tests/acceptance.cpp:42-84; schedule independence
proj/tests/test_parallel.cpp:132-143 (chunks created with first_stream are
the slices a G-GPU job computes).
"""
import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1108_0486_b200 as xg  # noqa: E402
from paper_1108_0486_b200.digest import chunk_record, row_digests, slice_digest  # noqa: E402

GP32 = xg.xorgensgp32_params()
with open(os.path.join(os.path.dirname(__file__), "golden", "full_size.json")) as _f:
    FS = json.load(_f)
C = FS["chunk_streams"]
PER = FS["u32"]["per_stream"]


def test_config4_fill_2p34_one_ensemble():
    """Config 4 at N = 1 exactly as bench.py runs it: ONE ensemble of 2^18
    streams, one 2^34-word (64 GiB) fill, every stream digested."""
    free, _ = torch.cuda.mem_get_info()
    if free < (1 << 36) + (1 << 30):
        pytest.skip("needs 65 GiB of free device memory")
    e = xg.BlockEnsemble(GP32, 1, 16 * C, 63)
    out = e.fill_u32(PER)
    x, s, ws = row_digests(out)
    del out
    for c in range(16):
        sl = slice(c * C, (c + 1) * C)
        assert chunk_record(x[sl], s[sl], ws[sl], PER) == FS["u32"]["chunks"][c], c
    gx, gs, gws = slice_digest(x, s, ws, PER)
    a = FS["u32"]["all"]
    assert (f"{gx:08x}", f"{gs:016x}", f"{gws:016x}") == (a["xor"], a["sum"], a["wsum"])


def test_config4_chunks_as_slices():
    """The same 2^34 words as 16 slices of 2^14 streams (first_stream =
    c * 2^14, 4 GiB each): the partition a 16-GPU job runs; equal chunk by
    chunk, so any G in {1, 2, 4, 8, 16} reproduces the 1-GPU fill."""
    out = torch.empty((C, PER), dtype=torch.uint32, device="cuda")
    for c in range(16):
        e = xg.BlockEnsemble(GP32, 1, C, 63, first_stream=c * C)
        e.fill_u32(PER, out=out)
        assert chunk_record(*row_digests(out), PER) == FS["u32"]["chunks"][c], c


@pytest.mark.parametrize("chunk", range(8))
def test_config3_f32_f64_full_digest(chunk):
    """Config 3: 2^30 f32 and 2^30 f64 values from 2^14 fresh streams (chunk 0 =
    the 1-GPU config; chunk r = rank r of the weak-scaled fill), every value's
    bits digested."""
    e = xg.BlockEnsemble(GP32, 1, C, 63, first_stream=chunk * C)
    f = e.fill_f32(PER)
    assert chunk_record(*row_digests(f), PER) == FS["f32"]["chunks"][chunk]
    del f
    e = xg.BlockEnsemble(GP32, 1, C, 63, first_stream=chunk * C)
    d = e.fill_f64(PER)
    assert chunk_record(*row_digests(d), 2 * PER) == FS["f64"]["chunks"][chunk]


def test_config5_mc_exact_2p32_samples():
    """Config 5's stream set (2^17 streams, base_seed 1): the exact hit count
    of 2^32 samples (2^15 per stream), then per chunk of 2^14 streams (the
    slices of N = 2, 4, 8)."""
    spp = FS["mc"]["samples_per_stream"]
    e = xg.BlockEnsemble(GP32, 1, 8 * C, 63)
    assert int(e.mc_pi(spp).item()) == FS["mc"]["total_hits_2p32"]
    for c in range(8):
        e = xg.BlockEnsemble(GP32, 1, C, 63, first_stream=c * C)
        assert int(e.mc_pi(spp).item()) == FS["mc"]["chunk_hits"][c], c


def test_mc_chunked_calls_compose():
    """mc_pi(a) then mc_pi(b) equals mc_pi(a + b) at scale (2^17 streams)."""
    spp = FS["mc"]["samples_per_stream"]
    e = xg.BlockEnsemble(GP32, 1, 8 * C, 63)
    h = e.mc_pi(spp // 4)
    e.mc_pi(3 * spp // 4, hits=h)
    assert int(h.item()) == FS["mc"]["total_hits_2p32"]


def test_digest_kernel_matches_numpy():
    """xg_digest_u32 against numpy on ragged and misaligned rows."""
    g = torch.Generator(device="cpu").manual_seed(5)
    for rows, per in ((1, 1), (3, 7), (5, 1000), (17, 4096), (2, 65537)):
        host = torch.randint(0, 2**32, (rows, per + 1), generator=g, dtype=torch.int64).numpy()
        host = host.astype(np.uint32)
        dev = torch.from_numpy(host.view(np.int32)).cuda()
        for t in (dev[:, :per].contiguous(), dev.reshape(-1)[1:1 + rows * per].reshape(rows, per)):
            x, s, ws = row_digests(t)
            ref = t.cpu().numpy().view(np.uint32).astype(np.uint64)
            k = np.arange(1, per + 1, dtype=np.uint64)
            assert np.array_equal(x, np.bitwise_xor.reduce(ref.astype(np.uint32), axis=1))
            assert np.array_equal(s, ref.sum(axis=1, dtype=np.uint64))
            with np.errstate(over="ignore"):
                assert np.array_equal(ws, (ref * k).sum(axis=1, dtype=np.uint64))

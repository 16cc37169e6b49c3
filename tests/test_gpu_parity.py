"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle,
the reference goldens and size-independent properties.  Bit-exact everywhere
(integer work; the float conversions are exact by construction)."""
import numpy as np
import pytest

from helpers import u32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1108_0486_b200 as xg  # noqa: E402
from oracle import Params  # noqa: E402

GP32 = xg.xorgensgp32_params()
KAT_SEED0 = ["a2c5f91b", "bd5797de", "cac8bc67", "7ba44aee", "11254d96", "198b2ab0", "656ea882",
             "9a94ce3e", "45568ed8", "1a4d6e4b", "bdcd2db4", "4bb14332", "74e6e085", "4cafd1e2",
             "04dbdceb", "07ba0f22"]  # proj/tests/test_xorgens.cpp:165-170


def np_u32(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def test_kat_seed0_and_golden_seed42():
    e = xg.BlockEnsemble(GP32, 0, 1, 63)
    assert np.array_equal(np_u32(e.fill_u32(16))[0], u32(KAT_SEED0))
    e = xg.BlockEnsemble(GP32, 42, 1, 63)
    assert [f"{v:08x}" for v in np_u32(e.fill_u32(4))[0]] == ["a61e8308", "8469633b", "80f8af0d",
                                                               "57f95c64"]


def test_golden_streams(golden):
    for seed, words in golden["streams"].items():
        e = xg.BlockEnsemble(GP32, int(seed), 1, 63)
        assert np.array_equal(np_u32(e.fill_u32(len(words)))[0], u32(words)), seed


def test_golden_seeded_state(golden):
    e = xg.BlockEnsemble(GP32, 1, 1, 63)
    buf, wy = e.block_state(0)
    g = golden["seeded_state_seed1"]
    assert np.array_equal(np.array(buf, dtype=np.uint32), u32(g["buffer"]))
    assert wy == int(g["weyl"], 16)


def test_golden_generate_and_continuation(golden):
    for g in golden["generate"]:
        e = xg.BlockEnsemble(GP32, g["base_seed"], g["blocks"], g["lanes"])
        first = np_u32(e.fill_u32(g["per_block"]))
        second = e.generate(g["per_block"])  # host path continues the same streams
        assert np.array_equal(first, np.stack([u32(r) for r in g["first"]]))
        assert np.array_equal(second, np.stack([u32(r) for r in g["second"]]))


@pytest.mark.parametrize("idx", [0, 1])
def test_golden_alt_params_runtime_kernels(golden, idx):
    entry = golden["alt_params"][idx]
    p = xg.GeneratorParams(*entry["params"])
    assert xg.gpu_supported(p)
    for seed, words in entry["streams"].items():
        e = xg.BlockEnsemble(p, int(seed), 1, 32)
        a = np_u32(e.fill_u32(250))[0]
        b = np_u32(e.fill_u32(len(words) - 250))[0]
        assert np.array_equal(np.concatenate([a, b]), u32(words))


@pytest.mark.parametrize("streams", [1, 7, 8, 9, 257])
@pytest.mark.parametrize("per", [1, 17, 31, 32, 33, 127, 128, 129, 256, 640, 1000, 2048, 4101])
def test_fill_u32_vs_oracle(oracle, streams, per):
    base = 0x1234_5678_9ABC + streams * 1000 + per
    e = xg.BlockEnsemble(GP32, base, streams, 63)
    o = oracle.ensemble(base, streams)
    for _ in range(2):  # second call checks continuation from a ragged end
        assert np.array_equal(np_u32(e.fill_u32(per)), o.fill_u32(per))


def test_fill_random_call_sequence(oracle):
    rng = np.random.default_rng(11)
    e = xg.BlockEnsemble(GP32, 99, 33, 63)
    o = oracle.ensemble(99, 33)
    for _ in range(12):
        kind = rng.integers(0, 5)
        n = int(rng.integers(0, 700))
        if kind == 0:
            assert np.array_equal(np_u32(e.fill_u32(n)), o.fill_u32(n))
        elif kind == 1:
            got = np_u32(e.fill_f32(n))
            assert np.array_equal(got.view(np.uint32), o.fill_f32(n).view(np.uint32))
        elif kind == 2:
            got = np_u32(e.fill_f64(n))
            assert np.array_equal(got.view(np.uint64), o.fill_f64(n).view(np.uint64))
        elif kind == 3:
            n -= n % 32
            hits = e.mc_pi(n)
            assert int(hits.item()) == int(o.mc_hits(n).sum())
        else:
            e.skip(n)
            o.fill_u32(n)
    assert np.array_equal(np_u32(e.fill_u32(300)), o.fill_u32(300))


def test_partitioned_slices_equal_single_fill(oracle):
    total, per = 100, 777
    full = np_u32(xg.BlockEnsemble(GP32, 5, total, 63).fill_u32(per))
    for world in (2, 3, 8):
        parts = []
        for rank in range(world):
            first, count = xg.partition(total, world, rank)
            parts.append(np_u32(xg.BlockEnsemble(GP32, 5, count, 63, first_stream=first).fill_u32(per)))
        assert np.array_equal(np.concatenate(parts), full)


def test_seed_wrap():
    e = xg.BlockEnsemble(GP32, 2**64 - 1, 2, 63)
    w = np_u32(e.fill_u32(40))
    assert np.array_equal(w[1], np_u32(xg.BlockEnsemble(GP32, 0, 1, 63).fill_u32(40))[0])


@pytest.mark.parametrize("per", [1, 2, 31, 32, 33, 63, 64, 65, 1001])
def test_conversions_vs_oracle(oracle, per):
    e = xg.BlockEnsemble(GP32, 77, 5, 63)
    o = oracle.ensemble(77, 5)
    f = np_u32(e.fill_f32(per))
    assert np.array_equal(f.view(np.uint32), o.fill_f32(per).view(np.uint32))
    d = np_u32(e.fill_f64(per))
    assert np.array_equal(d.view(np.uint64), o.fill_f64(per).view(np.uint64))
    u = np_u32(e.fill_u64(per))
    w = o.fill_u32(2 * per).astype(np.uint64)
    assert np.array_equal(u, w[:, 0::2] | (w[:, 1::2] << np.uint64(32)))
    assert (f >= 0).all() and (f < 1).all() and (d >= 0).all() and (d < 1).all()


def test_golden_conversions(golden):
    g = golden["conversions_seed42"]
    assert np.array_equal(np_u32(xg.BlockEnsemble(GP32, 42, 1, 63).fill_f32(256))[0].view(np.uint32),
                          u32(g["f32_bits"]))
    d = np_u32(xg.BlockEnsemble(GP32, 42, 1, 63).fill_f64(128))[0]
    assert [f"{v:016x}" for v in d.view(np.uint64)] == g["f64_bits"]
    u = np_u32(xg.BlockEnsemble(GP32, 42, 1, 63).fill_u64(128))[0]
    assert [f"{int(v):016x}" for v in u] == g["u64"]
    h = xg.BlockEnsemble(GP32, 42, 1, 63).mc_pi(128)
    assert int(h.item()) == g["mc_hits_128_samples"]


@pytest.mark.parametrize("samples", [32, 64, 96, 1024, 32 * 1001, 65536 + 32])
def test_mc_pi_exact_vs_oracle(oracle, samples):
    e = xg.BlockEnsemble(GP32, 3, 19, 63)
    o = oracle.ensemble(3, 19)
    hits = e.mc_pi(samples)
    hits = e.mc_pi(samples, hits=hits)  # accumulates, continues streams
    assert int(hits.item()) == int(o.mc_hits(samples).sum() + o.mc_hits(samples).sum())


def test_mc_pi_block_rule_and_continuation(oracle):
    """Samples are consecutive word pairs (w[2m], w[2m+1]); a call must be
    a multiple of 32 samples; MC and fills interleave on the same streams."""
    e = xg.BlockEnsemble(GP32, 21, 3, 63)
    with pytest.raises(ValueError):
        e.mc_pi(33)
    e.fill_u32(17)                      # leave the streams at a ragged position
    words = oracle.ensemble(21, 3)
    words.fill_u32(17)
    w = words.fill_u32(64 * 5)          # the words MC will consume
    want = sum(oracle.mc_hits(w[g]) for g in range(3))
    assert int(e.mc_pi(160).item()) == want
    assert np.array_equal(np_u32(e.fill_u32(50)), words.fill_u32(50))


def test_from_raw_and_state_roundtrip(oracle, golden):
    g = golden["from_raw"]
    buf = u32(g["buffer"]).astype(np.uint64)
    st = xg.XorgensState.from_raw(GP32, buf.tolist(), int(g["weyl"], 16))
    words = [st.next_word() for _ in range(len(g["stream"]))]
    assert np.array_equal(np.array(words, dtype=np.uint32), u32(g["stream"]))
    # export after an odd number of words equals the oracle's logical buffer
    e = xg.BlockEnsemble(GP32, 8, 3, 63)
    e.fill_u32(333)
    o = oracle.ensemble(8, 3)
    o.fill_u32(333)
    for i in range(3):
        b, w = e.block_state(i)
        assert np.array_equal(np.array(b, dtype=np.uint64), o.logical_buffer(i))
        assert w == o.weyl(i)
    # import stream 0's state into stream 2: they then agree
    b0, w0 = e.block_state(0)
    e.set_block_state(2, b0, w0)
    out = np_u32(e.fill_u32(500))
    assert np.array_equal(out[0], out[2])
    assert not np.array_equal(out[0], out[1])


def test_next_word_interleaves_with_fills(oracle):
    st = xg.XorgensState(GP32, 1234)
    ref = oracle.stream(1234, 40000)
    got = [st.next_word() for _ in range(1000)]
    got += np_u32(st.ensemble.fill_u32(3000))[0].tolist()
    got += [st.next_word() for _ in range(20000)]       # crosses a refill boundary
    v = st.next_u64()
    got += [v & 0xFFFFFFFF, v >> 32]
    got += np_u32(st.ensemble.fill_u32(1000))[0].tolist()
    assert np.array_equal(np.array(got, dtype=np.uint32), ref[:len(got)])
    b, w = st.logical_buffer(), st.weyl_value()
    o = oracle.ensemble(1234, 1)
    o.fill_u32(len(got))
    assert np.array_equal(np.array(b, dtype=np.uint64), o.logical_buffer(0)) and w == o.weyl(0)


def test_batch_step_and_source(oracle):
    st = xg.XorgensState(GP32, 5)
    got = []
    for lanes in (1, 32, 63, 7):
        got += xg.batch_step(st, lanes)
    assert np.array_equal(np.array(got, dtype=np.uint32), oracle.stream(5, len(got)))
    with pytest.raises(xg.OutOfRangeError):
        xg.batch_step(st, 64)
    with pytest.raises(xg.OutOfRangeError):
        xg.batch_step(st, 0)
    src = xg.XorgensSource(GP32, 42)
    assert [src.next() for _ in range(4)] == [0xa61e8308, 0x8469633b, 0x80f8af0d, 0x57f95c64]
    assert src.word_bits() == 32


def test_empty_and_errors():
    e = xg.BlockEnsemble(GP32, 0, 2, 1)
    assert e.generate(0).shape == (2, 0)
    with pytest.raises(xg.OutOfRangeError):
        xg.BlockEnsemble(GP32, 0, 0, 1)
    with pytest.raises(xg.OutOfRangeError):
        xg.BlockEnsemble(GP32, 0, 1, 64)
    with pytest.raises(xg.UnsupportedParamsError):  # conventions defined on w = 32 words
        xg.BlockEnsemble(xg.tiny_r4w16_params(), 0, 1, 1).fill_f32(10)
    with pytest.raises(ValueError):
        e.fill_u32(10, out=torch.empty(3, dtype=torch.uint32, device="cuda"))
    with pytest.raises(xg.OutOfRangeError):
        e.block_state(2)


def test_block_independence(oracle):
    # proj/tests/test_parallel.cpp:155-167
    a = xg.BlockEnsemble(GP32, 55, 3, 63)
    b = xg.BlockEnsemble(GP32, 55, 3, 63)
    buf, w = a.block_state(1)
    o = oracle.from_raw(np.array(buf, dtype=np.uint64)[None, :], [w])
    o.fill_u32(100)
    a.set_block_state(1, o.logical_buffer(0).tolist(), o.weyl(0))
    ra, rb = np_u32(a.fill_u32(200)), np_u32(b.fill_u32(200))
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[2], rb[2])
    assert not np.array_equal(ra[1], rb[1])


@pytest.mark.slow
def test_config2_full_size_checksum(golden, oracle):
    """BASELINE config 2: 2^30 words, P = 2^14 streams x 2^16, base_seed 1 --
    xor and block-major weighted sum against the reference-derived golden,
    plus sampled streams word-for-word against the oracle."""
    g = golden["config2"]
    P, n = g["streams"], g["per_stream"]
    e = xg.BlockEnsemble(GP32, g["base_seed"], P, 63)
    out = e.fill_u32(n)
    host = np_u32(out).reshape(-1)
    del out
    per_stream_xor = np.bitwise_xor.reduce(host.reshape(P, n), axis=1).astype(np.uint32)
    gx = int(np.bitwise_xor.reduce(per_stream_xor))
    gs = 0
    chunk = 1 << 24
    for start in range(0, host.size, chunk):
        w = host[start:start + chunk].astype(np.uint64)
        pos = np.arange(start + 1, start + w.size + 1, dtype=np.uint64)
        gs = (gs + int(np.sum(w * pos, dtype=np.uint64))) % 2**64
    assert f"{gx:08x}" == g["xor"]
    assert f"{gs:016x}" == g["wsum"]
    import hashlib
    assert hashlib.sha256(per_stream_xor.tobytes()).hexdigest() == g["per_stream_xor_sha"]
    for s in (0, 1, 4095, P - 1):
        assert np.array_equal(host[s * n:(s + 1) * n], oracle.stream(g["base_seed"] + s, n))


def test_config1_single_stream(golden):
    """BASELINE config 1 on the GPU: ONE stream, seed 1, 10^8 words (one warp,
    pair-lane kernel) -- xor, sum_k w_k (k+1) mod 2^64 and the last word
    against the reference-derived golden (tests/golden/ref_vectors.json)."""
    g = golden["config1"]
    e = xg.BlockEnsemble(GP32, g["seed"], 1, 63)
    host = np_u32(e.fill_u32(g["n"]))[0]
    assert f"{int(np.bitwise_xor.reduce(host)):08x}" == g["xor"]
    ws = 0
    chunk = 1 << 24
    for start in range(0, host.size, chunk):
        w = host[start:start + chunk].astype(np.uint64)
        pos = np.arange(start + 1, start + w.size + 1, dtype=np.uint64)
        ws = (ws + int(np.sum(w * pos, dtype=np.uint64))) % 2**64
    assert f"{ws:016x}" == g["sum"]
    assert f"{int(host[-1]):08x}" == g["last"]


@pytest.mark.slow
def test_full_size_float_properties(oracle):
    """2^30 f32 and f64 values: range, mean, and sampled streams bit-exact."""
    P, n = 1 << 14, 1 << 16
    e = xg.BlockEnsemble(GP32, 1, P, 63)
    f = e.fill_f32(n)
    assert float(f.min()) >= 0.0 and float(f.max()) < 1.0
    assert abs(float(f.double().mean()) - 0.5) < 1e-4
    o = oracle.ensemble(1, 2)
    assert np.array_equal(np_u32(f[:2]).view(np.uint32), o.fill_f32(n).view(np.uint32))
    del f
    d = e.fill_f64(n // 2)
    assert float(d.min()) >= 0.0 and float(d.max()) < 1.0
    assert abs(float(d.mean()) - 0.5) < 1e-4
    assert np.array_equal(np_u32(d[:2]).view(np.uint64), o.fill_f64(n // 2).view(np.uint64))


def test_cpp_dropin_against_reference():
    """tests/cpp/dropin_test.cpp: the reference C++ API (its own sources) next
    to xg::gpu on the same calls; built by oracle/Makefile where the reference
    tree exists and shipped as oracle/_ref/dropin_test."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("dropin_test not built (needs the reference tree at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def test_raw_stream_vs_golden_and_oracle(oracle, golden):
    """xg_fill_raw_u32 = RawXorgens::next (Weyl ablated); the Weyl accumulator
    is untouched, so raw and full fills interleave exactly like the reference
    classes sharing one XorgensState."""
    for seed, words in golden["raw_streams"].items():
        e = xg.BlockEnsemble(GP32, int(seed), 1, 63)
        assert np.array_equal(np_u32(e.fill_raw_u32(len(words)))[0], u32(words))
    e = xg.BlockEnsemble(GP32, 11, 9, 63)
    o = oracle.ensemble(11, 9)
    for n in (100, 129, 4096):
        assert np.array_equal(np_u32(e.fill_raw_u32(n)), o.fill_raw_u32(n))
        assert np.array_equal(np_u32(e.fill_u32(n)), o.fill_u32(n))
    for i in range(9):
        b, w = e.block_state(i)
        assert w == o.weyl(i) and np.array_equal(np.array(b, dtype=np.uint64), o.logical_buffer(i))


# ---- runtime-parameter kernels (any w=32, r=128 set with lane_bound >= 32) ----

RT_SETS = [
    (128, 95, 17, 12, 13, 15, 32, 2654435769, 16),   # J=1, delta=1 (proj/tests/test_params.cpp:65)
    (128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11),  # J=2, delta=31
    (128, 63, 9, 23, 5, 27, 32, 0x9E3779B9, 5),       # J=2, delta=1
    (128, 65, 15, 14, 12, 17, 32, 2654435761, 16),    # gp32 shape, different omega -> runtime path
]


@pytest.mark.parametrize("ps", RT_SETS)
def test_runtime_params_all_modes(oracle, reference, ps):
    p = xg.GeneratorParams(*ps)
    op = Params(*ps)
    assert xg.gpu_supported(p)
    e = xg.BlockEnsemble(p, 77, 11, 32)
    o = oracle.ensemble(77, 11, op)
    assert np.array_equal(np_u32(e.fill_u32(1000)), o.fill_u32(1000))
    assert np.array_equal(np_u32(e.fill_f32(257)).view(np.uint32), o.fill_f32(257).view(np.uint32))
    assert np.array_equal(np_u32(e.fill_f64(129)).view(np.uint64), o.fill_f64(129).view(np.uint64))
    assert int(e.mc_pi(320).item()) == int(o.mc_hits(320).sum())
    assert np.array_equal(np_u32(e.fill_raw_u32(300)), o.fill_raw_u32(300))
    assert np.array_equal(np_u32(e.fill_u32(64)), o.fill_u32(64))
    # and the reference sources themselves, stream 0
    assert np.array_equal(np_u32(xg.BlockEnsemble(p, 5, 1, 32).fill_u32(2000))[0],
                          reference.stream(5, 2000, op).astype(np.uint32))


def test_many_streams_seeding_sampled(oracle):
    """2^20 streams: seeding + a fill, sampled streams word-for-word."""
    P, n = 1 << 20, 256
    e = xg.BlockEnsemble(GP32, 12345, P, 63)
    out = e.fill_u32(n)
    rng = np.random.default_rng(3)
    for g in [0, 1, P - 1, *rng.integers(0, P, 20).tolist()]:
        assert np.array_equal(np_u32(out[g]), oracle.stream(12345 + g, n)), g


def test_generate_host_chunked_matches_device_fill(oracle):
    """xg_generate_host streams P x per through two 2^26-word staging slots
    (several chunks here) and must equal a device fill of a twin ensemble."""
    P, per = 4096, 1 << 15
    a = xg.BlockEnsemble(GP32, 9, P, 63)
    b = xg.BlockEnsemble(GP32, 9, P, 63)
    host = a.generate(per)
    dev = np_u32(b.fill_u32(per))
    assert np.array_equal(host, dev)
    for g in (0, 2047, 2048, P - 1):
        assert np.array_equal(host[g], oracle.stream(9 + g, per))
    assert np.array_equal(a.generate(100), np_u32(b.fill_u32(100)))


def test_independent_handles_on_separate_streams(oracle):
    """Handles are single-owner but independent: two ensembles filling on two
    CUDA streams concurrently give the same words as the oracle."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a = xg.BlockEnsemble(GP32, 100, 64, 63)
    b = xg.BlockEnsemble(GP32, 200, 64, 63)
    oa = torch.empty((64, 4096), dtype=torch.uint32, device="cuda")
    ob = torch.empty((64, 4096), dtype=torch.uint32, device="cuda")
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            a.fill_u32(4096, out=oa, stream=s1)
        with torch.cuda.stream(s2):
            b.fill_u32(4096, out=ob, stream=s2)
    torch.cuda.synchronize()
    ea, eb = oracle.ensemble(100, 64), oracle.ensemble(200, 64)
    for _ in range(2):
        ea.fill_u32(4096)
        eb.fill_u32(4096)
    assert np.array_equal(np_u32(oa), ea.fill_u32(4096))
    assert np.array_equal(np_u32(ob), eb.fill_u32(4096))


def test_kernel_launch_accounting():
    e = xg.BlockEnsemble(GP32, 1, 16, 63)
    n0 = xg.kernel_launches()
    e.fill_u32(100)
    e.fill_f32(100)
    e.mc_pi(64)
    torch.cuda.synchronize()
    assert xg.kernel_launches() - n0 == 3


def test_checkpoint_resume(oracle, tmp_path):
    """Whole-ensemble checkpoint (xg_state_export_all / import_all): a resumed
    ensemble continues every stream exactly."""
    e = xg.BlockEnsemble(GP32, 31, 100, 63)
    e.fill_u32(777)
    path = str(tmp_path / "ckpt.npz")
    e.save(path)
    a = np_u32(e.fill_u32(1000))
    r = xg.BlockEnsemble.load(path, 63)
    assert np.array_equal(a, np_u32(r.fill_u32(1000)))
    o = oracle.ensemble(31, 100)
    o.fill_u32(777)
    assert np.array_equal(a, o.fill_u32(1000))
    with pytest.raises(ValueError):
        xg.BlockEnsemble(GP32, 31, 99, 63).load_state_dict(e.state_dict())
    # a state_dict round trip through a different ensemble object
    sd = e.state_dict()
    f = xg.BlockEnsemble(GP32, 0, 100, 63)
    f.load_state_dict(sd)
    assert np.array_equal(np_u32(f.fill_u32(64)), np_u32(e.fill_u32(64)))


def test_cuda_graph_capture_replays_continue_streams(oracle):
    """Fills are asynchronous, host-sync-free launches with the state in device
    memory, so they capture into a CUDA graph; each replay continues the
    streams (the launch-bound small-fill case)."""
    e = xg.BlockEnsemble(GP32, 5, 256, 63)
    out = torch.empty((256, 1024), dtype=torch.uint32, device="cuda")
    hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        e.fill_u32(1024, out=out)       # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        e.fill_u32(1024, out=out)
        e.mc_pi(64, hits=hits)
    o = oracle.ensemble(5, 256)
    o.fill_u32(1024)
    want_hits = 0
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(np_u32(out), o.fill_u32(1024))
        want_hits += int(o.mc_hits(64).sum())
        assert int(hits.item()) == want_hits


def test_generate_host_streams_longer_than_a_slot(oracle):
    """per_stream > 2^26 words: tiles of 2048 streams advanced in word chunks,
    copied 2D into the block-major host layout (continuation inside a call)."""
    P, per = 3, (1 << 26) + 1000
    e = xg.BlockEnsemble(GP32, 77, P, 63)
    host = e.generate(per)
    for g in range(P):
        x, s = oracle.ensemble(77 + g, 1).checksums(per)
        w = host[g].astype(np.uint64)
        assert int(np.bitwise_xor.reduce(host[g])) == int(x[0])
        assert int(np.sum(w * np.arange(1, per + 1, dtype=np.uint64), dtype=np.uint64)) == int(s[0])
    assert np.array_equal(e.generate(64), oracle.ensemble(77, P).fill_u32(per + 64)[:, per:])



# ---- general-parameter kernels (every set the reference accepts) ------------

GENERIC_SETS = [
    ("tiny_r2w8", (2, 1, 1, 1, 5, 7, 8, 159, 4)),
    ("tiny_r2w16", (2, 1, 1, 1, 6, 11, 16, 40503, 8)),
    ("tiny_r4w16", (4, 3, 1, 2, 5, 8, 16, 40503, 8)),
    ("w64_paper", (64, 53, 33, 26, 27, 29, 64, 11400714819323198485, 32)),
    ("r128_lb3", (128, 125, 15, 14, 12, 17, 32, 2654435769, 16)),           # lane_bound 3
    ("r64_w32", (64, 37, 13, 7, 11, 19, 32, 2654435769, 16)),               # lane_bound 27
    ("r1024", (1024, 511, 9, 23, 5, 27, 32, 2654435769, 16)),               # 8 KiB state per stream
]


@pytest.mark.parametrize("name,ps", GENERIC_SETS, ids=[n for n, _ in GENERIC_SETS])
def test_generic_params_vs_oracle_and_reference(oracle, reference, name, ps):
    p = xg.GeneratorParams(*ps)
    op = Params(*ps)
    assert xg.gpu_supported(p) and not xg.fast_path(p)
    lanes = xg.lane_bound(p)
    e = xg.BlockEnsemble(p, 2**64 - 2, 5, lanes)          # seeds wrap through 0
    o = oracle.ensemble(2**64 - 2, 5, op)
    for n in (1, 33, 700):
        assert np.array_equal(np_u32(e.fill_words(n)), o.fill_words(n)), n
    if p.w <= 32:
        assert np.array_equal(np_u32(e.fill_u32(100)), o.fill_words(100).astype(np.uint32))
        assert np.array_equal(np_u32(e.fill_raw_u32(50)), o.fill_raw_u32(50))
        assert np.array_equal(e.generate(77), o.fill_words(77).astype(np.uint32))
    else:
        assert np.array_equal(e.generate(77), o.fill_words(77))
    for i in (0, 4):
        b, w = e.block_state(i)
        assert np.array_equal(np.array(b, dtype=np.uint64), o.logical_buffer(i)) and w == o.weyl(i)
    # the reference sources themselves: one stream, and next_word served from refills
    st = xg.XorgensState(p, 123)
    ref = reference.stream(123, 3000, op)
    got = [st.next_word() for _ in range(1000)]
    got += np_u32(st.ensemble.fill_words(2000))[0].tolist()
    assert np.array_equal(np.array(got, dtype=np.uint64), ref)
    with pytest.raises(xg.UnsupportedParamsError):
        e.mc_pi(32)


@pytest.mark.parametrize("streams", [1, 5, 33])
@pytest.mark.parametrize("matrices", [1, 2, 3, 5, 38, 101])
def test_rank_test_counts_vs_oracle(oracle, streams, matrices):
    """Fused matrix-rank bins (xg_rank_test) equal the oracle's counting loop
    (tests.cpp:93-109) on the same streams, from ragged positions, and the
    streams continue exactly afterwards."""
    base = 9000 + streams * 100 + matrices
    e = xg.BlockEnsemble(GP32, base, streams, 63)
    o = oracle.ensemble(base, streams)
    e.fill_u32(17)
    o.fill_u32(17)
    got = np_u32(e.rank_test(matrices)).astype(np.uint64)
    assert np.array_equal(got, o.rank_counts(matrices).sum(axis=0))
    assert np.array_equal(np_u32(e.fill_u32(40)), o.fill_u32(40))


def test_rank_test_runtime_params_and_unsupported(oracle):
    p1 = xg.GeneratorParams(128, 95, 17, 12, 13, 15, 32, 2654435769, 16)  # J = 1: pair kernel
    e = xg.BlockEnsemble(p1, 3, 9, 32)
    o = oracle.ensemble(3, 9, oracle.params(128, 95, 17, 12, 13, 15, 32, 2654435769, 16))
    assert np.array_equal(np_u32(e.rank_test(77)).astype(np.uint64), o.rank_counts(77).sum(axis=0))
    p2 = xg.GeneratorParams(128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11)  # J = 2
    with pytest.raises(Exception):
        xg.BlockEnsemble(p2, 3, 2, 32).rank_test(4)
    with pytest.raises(Exception):
        xg.BlockEnsemble(xg.tiny_r4w16_params(), 3, 2, 1).rank_test(4)


def test_rank_test_statistic_equals_reference_on_gpu_words():
    """The statistic from the GPU bins equals the reference's own
    matrix_rank_test run over the same GPU-generated words."""
    from oracle import Battery
    try:
        b = Battery()
    except FileNotFoundError as ex:  # pragma: no cover
        pytest.skip(str(ex))
    m = 5000
    words = np_u32(xg.BlockEnsemble(GP32, 77, 1, 63).fill_u32(32 * m))[0]
    counts = xg.BlockEnsemble(GP32, 77, 1, 63).rank_test(m)
    chi2, p = xg.matrix_rank_statistic(counts)
    rchi2, rp = b.matrix_rank(words, m)
    assert chi2 == rchi2 and abs(p - rp) <= 1e-12 * max(1.0, rp)


def test_rank_test_large_ensemble():
    """2^14 streams x 2^10 matrices (2^29 words): bins sum to the matrix count
    and the reference statistic is unremarkable."""
    P, m = 1 << 14, 1 << 10
    c = np_u32(xg.BlockEnsemble(GP32, 1, P, 63).rank_test(m))
    assert int(c.sum()) == P * m
    chi2, p = xg.matrix_rank_statistic(c)
    assert 1e-6 < p <= 1.0, (c, chi2, p)


@pytest.mark.parametrize("K,nb", [(1, 50), (7, 65), (31, 33), (32, 40), (33, 97), (100, 64),
                                  (500, 70), (1000, 45), (1023, 38), (1024, 40), (2000, 39),
                                  (4099, 40)])
def test_linear_complexity_histogram_vs_reference(K, nb):
    """GPU Berlekamp-Massey histogram (xg_linear_complexity_test) equals the
    reference's own berlekamp_massey (gf2.cpp:62-110) block by block over the
    same words (3 streams, blocks straddling words, ragged last word), and
    the streams continue after exactly ceil(K * nb / 32) words."""
    from oracle import Battery
    try:
        b = Battery()
    except FileNotFoundError as ex:  # pragma: no cover
        pytest.skip(str(ex))
    P = 3
    nwords = (K * nb + 31) // 32
    words = np_u32(xg.BlockEnsemble(GP32, 555 + K, P, 63).fill_u32(nwords + 7))
    e = xg.BlockEnsemble(GP32, 555 + K, P, 63)
    got = np_u32(e.linear_complexity_test(K, nb)).astype(np.uint64)
    want = sum(b.lc_histogram(words[g, :nwords], K, nb) for g in range(P))
    assert np.array_equal(got, want)
    assert np.array_equal(np_u32(e.fill_u32(7)), words[:, nwords:nwords + 7])


def test_linear_complexity_statistic_on_gpu_equals_reference():
    from oracle import Battery
    try:
        b = Battery()
    except FileNotFoundError as ex:  # pragma: no cover
        pytest.skip(str(ex))
    K, nb = 1000, 2000
    words = np_u32(xg.BlockEnsemble(GP32, 31, 1, 63).fill_u32((K * nb + 31) // 32))[0]
    hist = xg.BlockEnsemble(GP32, 31, 1, 63).linear_complexity_test(K, nb)
    chi2, p = xg.linear_complexity_statistic(hist, K)
    rchi2, rp = b.linear_complexity(words, K, nb)
    assert chi2 == rchi2 and abs(p - rp) <= 1e-12 * max(1.0, rp)


def test_linear_complexity_chunked_and_errors():
    """More blocks than one chunk holds (2^14 streams x 4100 blocks of 1000
    bits: chunk boundaries at multiples of 32 blocks) -- all blocks counted,
    the statistic unremarkable; argument errors."""
    P, K, nb = 1 << 14, 1000, 4100
    e = xg.BlockEnsemble(GP32, 1, P, 63)
    h = np_u32(e.linear_complexity_test(K, nb))
    assert int(h.sum()) == P * nb
    chi2, p = xg.linear_complexity_statistic(h, K)
    assert 1e-6 < p <= 1.0, (chi2, p)
    with pytest.raises(Exception):
        e.linear_complexity_test((1 << 18) + 1, 1)
    with pytest.raises(Exception):
        e.linear_complexity_test(0, 1)
    with pytest.raises(Exception):
        xg.BlockEnsemble(xg.tiny_r4w16_params(), 3, 2, 1).linear_complexity_test(100, 4)


def test_cuda_graph_capture_of_a_capped_fill(oracle):
    """A large-ensemble u32 fill (the occupancy-capped launch: 4-stream CTAs,
    reserved shared memory) captured into a CUDA graph on a fresh ensemble
    with no warm-up launch: the launch path makes no non-stream driver call,
    and every replay continues the streams."""
    P, n = 8192, 256
    e = xg.BlockEnsemble(GP32, 11, P, 63)
    out = torch.empty((P, n), dtype=torch.uint32, device="cuda")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        e.fill_u32(n, out=out)
    o = oracle.ensemble(11, P)
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(np_u32(out), o.fill_u32(n))


def test_long_linearity_on_gpu(golden):
    """proj/tests/test_long_linearity.cpp:71-99 (an opt-in long test in the
    reference) on the GPU: the low bits of the Weyl-ablated stream, seed 1,
    over 2^30 words -- the first and the last 2^14-bit windows, the stream
    skipped 2^30 - 2^15 words in between on the device -- have linear
    complexity exactly 4096 (the state size) and the last window's bits equal
    the reference's bit for bit; the Weyl-combined stream's first window has
    complexity 8192.  Complexities by the reference's berlekamp_massey."""
    import hashlib

    from oracle import Battery
    try:
        b = Battery()
    except FileNotFoundError as ex:  # pragma: no cover
        pytest.skip(str(ex))
    g = golden["long_linearity"]
    win, words = g["window"], g["raw_words"]
    e = xg.BlockEnsemble(GP32, 1, 1, 63)
    first = (np_u32(e.fill_raw_u32(win))[0] & 1).astype(np.uint8)
    e.skip(words - 2 * win)
    last = (np_u32(e.fill_raw_u32(win))[0] & 1).astype(np.uint8)
    assert hashlib.sha256(first.tobytes()).hexdigest() == g["raw_seed1_first_bits_sha256"]
    assert hashlib.sha256(last.tobytes()).hexdigest() == g["raw_seed1_last_bits_sha256"]
    assert b.berlekamp_massey(first) == g["raw_seed1_first"] == 4096
    assert b.berlekamp_massey(last) == g["raw_seed1_last"] == 4096
    weyl = (np_u32(xg.BlockEnsemble(GP32, 1, 1, 63).fill_u32(win))[0] & 1).astype(np.uint8)
    assert b.berlekamp_massey(weyl) == g["weyl_seed1_first"] == 8192
    # the same three complexities by the GPU's own Berlekamp-Massey
    packed = np.stack([np.packbits(x).view(">u4").astype(np.uint32) for x in (first, last, weyl)])
    dev = torch.from_numpy(packed.view(np.int32)).cuda()
    assert np_u32(xg.berlekamp_massey(dev, win)).tolist() == [4096, 4096, 8192]


@pytest.mark.parametrize("nbits", [1, 2, 31, 32, 33, 64, 999, 1000, 4096, 16384, 40001])
def test_gpu_berlekamp_massey_vs_reference(nbits):
    """xg_berlekamp_massey (shared-memory polynomials, one warp per sequence)
    equals the reference's berlekamp_massey (gf2.cpp:62-110) on random,
    LFSR-generated (low complexity) and zero sequences."""
    from oracle import Battery
    try:
        b = Battery()
    except FileNotFoundError as ex:  # pragma: no cover
        pytest.skip(str(ex))
    rng = np.random.default_rng(nbits)
    seqs = [rng.integers(0, 2, size=nbits, dtype=np.uint8) for _ in range(3)]
    lfsr = list(rng.integers(0, 2, size=min(nbits, 40), dtype=np.uint8))
    taps = [int(t) for t in rng.choice(np.arange(1, 41), size=4, replace=False)]
    while len(lfsr) < nbits:
        i = len(lfsr)
        lfsr.append(np.uint8(np.bitwise_xor.reduce([lfsr[i - t] for t in taps if i - t >= 0])))
    seqs.append(np.array(lfsr[:nbits], dtype=np.uint8))
    seqs.append(np.zeros(nbits, dtype=np.uint8))
    words = (nbits + 31) // 32 + 1
    packed = np.zeros((len(seqs), words), dtype=np.uint32)
    for i, sq in enumerate(seqs):
        pb = np.packbits(np.concatenate([sq, np.zeros(32 * words - nbits, dtype=np.uint8)]))
        packed[i] = pb.view(">u4").astype(np.uint32)
    dev = torch.from_numpy(packed.view(np.int32)).cuda()
    got = np_u32(xg.berlekamp_massey(dev, nbits)).tolist()
    assert got == [b.berlekamp_massey(sq) for sq in seqs]


def test_next_view_and_return_continue_exactly(oracle):
    """xg_next_view hands out pinned refill words (double-buffered slots of
    2^16); xg_next_return gives unread ones back; fills, next_word and the
    state export then continue right after the last word used."""
    import ctypes

    L = xg._lib.lib
    st = xg.XorgensState(GP32, 99)
    h = st.ensemble.handle
    ref = oracle.stream(99, 400000)
    got = []
    ptr, cnt = ctypes.c_void_p(), ctypes.c_uint64()
    for take in (5, 65531, 70000, 1, 140000):
        left = take
        while left:
            assert L.xg_next_view(h, ctypes.byref(ptr), ctypes.byref(cnt)) == 0
            n = min(left, cnt.value)
            got += np.ctypeslib.as_array((ctypes.c_uint64 * cnt.value).from_address(ptr.value))[:n].tolist()
            assert L.xg_next_return(h, cnt.value - n) == 0
            left -= n
        got.append(st.next_word())
        got += np_u32(st.ensemble.fill_u32(777))[0].tolist()
    assert np.array_equal(np.array(got, dtype=np.uint32), ref[:len(got)])
    assert L.xg_next_return(h, 1) == xg._lib.XG_ERANGE  # nothing held after the fill
    b, w = st.logical_buffer(), st.weyl_value()
    o = oracle.ensemble(99, 1)
    o.fill_u32(len(got))
    assert np.array_equal(np.array(b, dtype=np.uint64), o.logical_buffer(0)) and w == o.weyl(0)


def test_next_word_many_slots_w64_and_tiny(reference):
    """The ring for the general-parameter path: w = 64 (8-byte slots) and a
    tiny w = 8 set, against the reference sources, across slot boundaries."""
    w64 = xg.GeneratorParams(64, 53, 33, 26, 27, 29, 64, 0x9E3779B97F4A7C15, 32)
    for p in (w64, xg.tiny_r2w8_params()):
        st = xg.XorgensState(p, 3)
        got = [st.next_word() for _ in range(140000)]
        pr = Params(p.r, p.s, p.a, p.b, p.c, p.d, p.w, p.omega, p.gamma)
        assert np.array_equal(np.array(got, dtype=np.uint64), reference.stream(3, 140000, pr))


def test_generate_host_rows_tiles_and_rows(oracle):
    """xg_generate_host_rows (the C++ generate() path): caller-owned uint64
    rows, u32 over PCIe widened by host threads; multi-tile shapes (a stream
    longer than one 256 MiB staging slot; many streams per tile) equal the
    device fill of a twin ensemble, and calls continue the streams."""
    import ctypes

    L = xg._lib.lib
    for P, per in ((3, (1 << 26) + 77), (5000, 6000), (1, 1)):
        a = xg.BlockEnsemble(GP32, 17, P, 63)
        b = xg.BlockEnsemble(GP32, 17, P, 63)
        for _ in range(2):
            rows = [np.full(per, 0xDEADBEEFDEADBEEF, dtype=np.uint64) for _ in range(P)]
            arr = (ctypes.c_void_p * P)(*[r.ctypes.data for r in rows])
            assert L.xg_generate_host_rows(a.handle, per, arr, None) == 0
            dev = np_u32(b.fill_u32(per))
            for g in (0, P // 2, P - 1):
                assert np.array_equal(rows[g], dev[g].astype(np.uint64)), (P, per, g)
            del dev
    assert L.xg_generate_host_rows(a.handle, 4, None, None) == xg._lib.XG_EINVAL


def test_hostbench_runs_reference_methods_over_dropin():
    """xg_hostbench (the reference's measure_throughput and
    measure_ensemble_throughput over xg::gpu) runs and reports rates."""
    import json
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_1108_0486_b200", "lib", "xg_hostbench")
    r = subprocess.run([exe, str(10**6), "3", "64", str(1 << 20)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    assert d["measure_throughput"]["rn_per_s"]["mean"] > 0
    assert d["measure_ensemble_throughput"]["rn_per_s"]["mean"] > 0


def test_generate_host_tiles_callback_order_and_content(oracle):
    """xg_generate_host_tiles (what xg::gpu::BlockEnsemble::generate uses):
    every (stream, word) range arrives exactly once, a stream's tiles in word
    order, with the stream's words; elements of 4 bytes for w = 32."""
    import ctypes

    L = xg._lib.lib
    P, per = 3, (1 << 26) + 99   # longer than one staging slot: several tiles per stream
    e = xg.BlockEnsemble(GP32, 8, P, 63)
    seen = {g: [] for g in range(P)}
    ref = oracle.ensemble(8, P)
    want = ref.fill_u32(per)
    bad = []
    FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                          ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint)

    def cb(ctx, s0, w0, ns, nw, tile, eb, part, parts):
        if part != 0:
            return
        if eb != 4:
            bad.append(eb)
        t = np.ctypeslib.as_array((ctypes.c_uint32 * (ns * nw)).from_address(tile)).reshape(ns, nw)
        for i in range(ns):
            seen[s0 + i].append(w0)
            if not np.array_equal(t[i], want[s0 + i, w0:w0 + nw]):
                bad.append((s0 + i, w0))

    f = FN(cb)
    assert L.xg_generate_host_tiles(e.handle, per, f, None, 2, None) == 0
    assert not bad
    for g in range(P):
        assert seen[g] == sorted(seen[g]) and seen[g][0] == 0 and len(seen[g]) > 1


def test_generate_host_f32_f64_equal_device_fills(oracle):
    """xg_generate_host_f32/f64 (the e2e path of config 3): the same values
    as the device fills, block-major in host memory, continuing the streams;
    odd lengths and streams longer than a staging slot."""
    for P, per in ((5, 1001), (3, 1000), (2, (1 << 26) + 3)):
        a = xg.BlockEnsemble(GP32, 21, P, 63)
        b = xg.BlockEnsemble(GP32, 21, P, 63)
        for _ in range(2):
            h32 = np.empty((P, per), dtype=np.float32)
            a.generate_f32_into_host(per, h32)
            assert np.array_equal(h32.view(np.uint32), np_u32(b.fill_f32(per)).view(np.uint32)), (P, per)
        h64 = np.empty((P, per // 2), dtype=np.float64)
        a.generate_f64_into_host(per // 2, h64)
        assert np.array_equal(h64.view(np.uint64), np_u32(b.fill_f64(per // 2)).view(np.uint64))
    o = oracle.ensemble(21, 5)
    c = xg.BlockEnsemble(GP32, 21, 5, 63)
    h = np.empty((5, 777), dtype=np.float64)
    c.generate_f64_into_host(777, h)
    assert np.array_equal(h.view(np.uint64), o.fill_f64(777).view(np.uint64))


def test_host_and_device_buffers_are_checked_before_the_call():
    """The C ABI takes bare pointers; the Python mirror checks every caller
    buffer (size, element width, host/device placement) before calling it."""
    e = xg.BlockEnsemble(GP32, 3, 4, 63)
    with pytest.raises(ValueError):
        e.generate_into_host(100, np.empty((4, 99), dtype=np.uint32))      # too small
    with pytest.raises(ValueError):
        e.generate_into_host(100, np.empty((4, 100), dtype=np.uint64))     # wrong width
    with pytest.raises(ValueError):
        e.generate_f64_into_host(10, np.empty((4, 10), dtype=np.float32))  # wrong width
    with pytest.raises(ValueError):
        e.generate_into_host(8, torch.empty((4, 8), dtype=torch.uint32, device="cuda"))  # not host
    with pytest.raises(ValueError):
        e.fill_u32(8, out=torch.empty((4, 7), dtype=torch.uint32, device="cuda"))
    with pytest.raises(ValueError):
        e.mc_pi(32, hits=torch.zeros(1, dtype=torch.int32, device="cuda"))
    # nothing was consumed by the rejected calls
    o = xg.BlockEnsemble(GP32, 3, 4, 63)
    h = torch.empty((4, 100), dtype=torch.uint32).pin_memory()
    e.generate_into_host(100, h)
    assert np.array_equal(h.numpy(), np_u32(o.fill_u32(100)))

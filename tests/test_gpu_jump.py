"""GPU parity of the jump-ahead path (csrc/xg_jump.cuh): one stream of a
register-window set filled with >= 2^20 words is cut into segments whose start
states are computed as s G^(kJ) over GF(2) and generated in parallel.  Every
test compares with the oracle's serial stream (or, past what the oracle can
generate, with an independent route to the same state), word for word."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1108_0486_b200 as xg  # noqa: E402
from oracle import Params  # noqa: E402

GP32 = xg.xorgensgp32_params()
M = 1 << 20  # the jump path's threshold (kJumpMin in csrc/xg_gpu.cu)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def one(seed, p=GP32):
    return xg.BlockEnsemble(p, seed, 1, xg.lane_bound(p))


@pytest.mark.parametrize("seed", [1, 0, (1 << 64) - 1, 987654321])
@pytest.mark.parametrize("n", [M, M + 12345, 5 * M + 64, 37 * M + 7])
def test_jump_fill_equals_serial_stream(oracle, seed, n):
    out = host(one(seed).fill_u32(n))[0]
    assert np.array_equal(out, oracle.stream(seed, n))


def test_jump_continuation_and_state(oracle):
    """jump / direct / jump / direct calls continue one stream exactly, and
    the exported state after them is the reference's."""
    e = one(31)
    sizes = [M + 1, 999, 3 * M, 100, 2 * M + 128]
    got = np.concatenate([host(e.fill_u32(n))[0] for n in sizes])
    o = oracle.ensemble(31, 1)
    want = np.concatenate([o.fill_u32(n)[0] for n in sizes])
    assert np.array_equal(got, want)
    buf, wy = e.block_state(0)
    assert wy == o.weyl(0) and np.array_equal(np.array(buf, dtype=np.uint64), o.logical_buffer(0))


def test_jump_every_mode(oracle):
    """f32 / f64 / u64 / zero-extended words / raw / MC / rank on one stream,
    each call continuing the previous one, against the oracle's ensemble."""
    e = one(5)
    o = oracle.ensemble(5, 1)
    f = host(e.fill_f32(M + 3))
    assert np.array_equal(f.view(np.uint32), o.fill_f32(M + 3).view(np.uint32))
    d = host(e.fill_f64(M + 5))
    assert np.array_equal(d.view(np.uint64), o.fill_f64(M + 5).view(np.uint64))
    u = host(e.fill_u64(M))  # 2^21 words, lo = first
    w = o.fill_u32(2 * M).astype(np.uint64)
    assert np.array_equal(u.view(np.uint64), w[:, 0::2] | (w[:, 1::2] << np.uint64(32)))
    wd = host(e.fill_words(M + 7))
    assert np.array_equal(wd.view(np.uint64), o.fill_words(M + 7))
    r = host(e.fill_raw_u32(2 * M + 11))
    assert np.array_equal(r, o.fill_raw_u32(2 * M + 11))
    assert int(e.mc_pi(M + 32 * 5).item()) == int(o.mc_hits(M + 32 * 5).sum())
    assert np.array_equal(host(e.rank_test(M // 16 + 3)), o.rank_counts(M // 16 + 3).sum(axis=0))
    assert np.array_equal(host(e.fill_u32(777)), o.fill_u32(777))
    buf, wy = e.block_state(0)
    assert wy == o.weyl(0) and np.array_equal(np.array(buf, dtype=np.uint64), o.logical_buffer(0))


@pytest.mark.parametrize("n", [M, M + 777, 9 * M + 4096])
def test_jump_skip_equals_serial_stream(oracle, n):
    e = one(17)
    e.skip(n)
    assert np.array_equal(host(e.fill_u32(1000))[0], oracle.stream(17, n + 1000)[n:])


def test_jump_skip_far_is_consistent():
    """Past what the oracle can generate: skip(2^40) = skip(2^39) twice =
    skip(2^40 - 2^21) + a jump fill of 2^21 words; then the same words."""
    a, b, c = one(3), one(3), one(3)
    a.skip(1 << 40)
    b.skip(1 << 39)
    b.skip(1 << 39)
    c.skip((1 << 40) - 2 * M)
    c.fill_u32(2 * M)
    wa, wb, wc = (host(x.fill_u32(4096))[0] for x in (a, b, c))
    assert np.array_equal(wa, wb) and np.array_equal(wa, wc)
    sa, sb = a.block_state(0), b.block_state(0)
    assert sa == sb
    # and the Weyl accumulator moved by exactly 2^40 + 4096 increments
    d = one(3)
    _, w0 = d.block_state(0)
    assert sa[1] == (w0 + ((1 << 40) + 4096) * GP32.omega) % (1 << 32)


def test_jump_matches_the_multistream_kernels(oracle):
    """An ensemble of 65 streams takes the direct path (one warp per stream):
    its stream 0 must equal the one-stream (jump) fill of the same seed."""
    n = (1 << 21) + 384
    a = host(one(1234).fill_u32(n))[0]
    b = host(xg.BlockEnsemble(GP32, 1234, 65, 63).fill_u32(n))[0]
    assert np.array_equal(a, b)
    assert np.array_equal(a[:M], oracle.stream(1234, M))


def test_jump_few_streams_each_jumped(oracle):
    """Up to 64 streams with >= 2^20 words each are jumped stream by stream:
    block-major rows, every mode's row offsets, continuation."""
    P, n = 3, M + 4099
    e = xg.BlockEnsemble(GP32, 40, P, 63)
    o = oracle.ensemble(40, P)
    assert np.array_equal(host(e.fill_u32(n)), o.fill_u32(n))
    assert np.array_equal(host(e.fill_f64(M + 1)).view(np.uint64), o.fill_f64(M + 1).view(np.uint64))
    assert int(e.mc_pi(M).item()) == int(o.mc_hits(M).sum())
    e.skip(2 * M + 7)
    o.fill_u32(2 * M + 7)
    assert np.array_equal(host(e.fill_u32(100)), o.fill_u32(100))
    g = e.generate(2 * M)
    assert np.array_equal(g, o.fill_u32(2 * M))


@pytest.mark.parametrize("ps", [
    (128, 95, 17, 12, 13, 15, 32, 2654435769, 16),   # J=1 runtime set
    (128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11),  # J=2 (word-lane kernel)
    (128, 65, 15, 14, 12, 17, 32, 2654435761, 16),    # gp32 shape, other omega
])
def test_jump_runtime_parameter_sets(oracle, ps):
    p = xg.GeneratorParams(*ps)
    n = 2 * M + 33
    assert np.array_equal(host(one(77, p).fill_u32(n))[0], oracle.stream(77, n, Params(*ps)))


def test_jump_host_paths_and_next_word(oracle):
    """generate() into host memory, then next_word, on one stream: the jump
    path serves the host copies and next_word continues after them."""
    s = xg.XorgensState(GP32, 8)
    e = s.ensemble
    n = 3 * M + 5
    want = oracle.stream(8, n + 2 * M + 10)
    assert np.array_equal(e.generate(n)[0], want[:n])
    assert np.array_equal(e.generate(2 * M)[0], want[n:n + 2 * M])
    words = [s.next_word() for _ in range(10)]
    assert np.array_equal(np.array(words, dtype=np.uint32), want[n + 2 * M:])
    e.skip(M + 3)  # a jump skip after next_word hands back the unread refill
    assert np.array_equal(host(e.fill_u32(64))[0],
                          oracle.stream(8, n + 2 * M + 10 + M + 3 + 64)[-64:])


def test_jump_on_a_side_torch_stream(oracle):
    """The caller's stream orders the jump products, the segment fill and the
    short last segment (side stream joined back)."""
    st = torch.cuda.Stream()
    e = one(99)
    out = torch.empty((1, 4 * M + 321), dtype=torch.uint32, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        e.fill_u32(4 * M + 321, out=out, stream=st)
        out2 = out.clone()
    st.synchronize()
    assert np.array_equal(out2.cpu().numpy()[0], oracle.stream(99, 4 * M + 321))


def test_bench_stream1_parity_and_rate():
    """The bench's config-1 workload checks the jump-ahead stream against the
    reference golden (tests/golden/ref_vectors.json) in the run."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    res = bench.parity_check("stream1", 1, 0, 0)
    assert res["checked"] and res["ok"], res


def test_jump_skip_many_streams(oracle):
    """More than 64 streams skipping >= 2^22 words jump as a batch (rows times
    G^(2^i) in chunks of 1024): sampled streams against the oracle, and a
    2^30 skip of 2000 streams against one-stream skips (other kernels:
    four-Russians rows vs the dense single-row product)."""
    P, n = 100, (1 << 22) + 3
    e = xg.BlockEnsemble(GP32, 600, P, 63)
    e.skip(n)
    got = host(e.fill_u32(1000))
    for g in (0, 50, P - 1):
        assert np.array_equal(got[g], oracle.stream(600 + g, n + 1000)[n:]), g
    P, n = 2000, 1 << 30
    e = xg.BlockEnsemble(GP32, 9000, P, 63)
    e.skip(n)
    got = host(e.fill_u32(256))
    for g in (0, 1023, 1024, P - 1):
        s = one(9000 + g)
        s.skip(n)
        assert np.array_equal(got[g], host(s.fill_u32(256))[0]), g
    assert e.block_state(P - 1)[1] == (one(9000 + P - 1).block_state(0)[1] + (n + 256) * GP32.omega) % (1 << 32)


def test_jump_from_two_host_threads(oracle):
    """Two one-stream handles of the same parameter set on two host threads
    and two CUDA streams share the process-wide jump tables: each gets the
    reference's words (fills and long skips, so the powers grow meanwhile)."""
    import threading

    out, errs = {}, []

    def work(seed):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                e = one(seed)
                a = e.fill_u32(3 * M + 11, stream=st)
                e.skip((1 << 33) + seed, stream=st)
                b = e.fill_u32(512, stream=st)
                st.synchronize()
                out[seed] = (a.cpu().numpy()[0], b.cpu().numpy()[0])
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)

    th = [threading.Thread(target=work, args=(s,)) for s in (70, 71)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for seed in (70, 71):
        assert np.array_equal(out[seed][0], oracle.stream(seed, 3 * M + 11))
        ref = one(seed)
        ref.skip(3 * M + 11)
        ref.skip((1 << 33) + seed)
        assert np.array_equal(out[seed][1], host(ref.fill_u32(512))[0])


@pytest.mark.parametrize("P,n", [(100, 1 << 21), (512, 1 << 20), (65, 1 << 22)])
def test_jump_many_streams_power_of_two(oracle, P, n):
    """65 .. 512 streams with a power-of-two length: every stream cut into Q
    segments (doubling over q for all streams at once), one fill of P Q
    segments -- block-major rows, continuation, f64 and MC modes."""
    e = xg.BlockEnsemble(GP32, 300, P, 63)
    o = oracle.ensemble(300, P)
    assert np.array_equal(host(e.fill_u32(n)), o.fill_u32(n))
    assert np.array_equal(host(e.fill_u32(1000)), o.fill_u32(1000))  # state continued
    if P == 100:
        assert np.array_equal(host(e.fill_f64(n // 2)).view(np.uint64), o.fill_f64(n // 2).view(np.uint64))
        assert int(e.mc_pi(n // 2).item()) == int(o.mc_hits(n // 2).sum())
        assert np.array_equal(host(e.fill_raw_u32(n)), o.fill_raw_u32(n))
    for g in (0, P - 1):
        buf, wy = e.block_state(g)
        assert wy == o.weyl(g) and np.array_equal(np.array(buf, dtype=np.uint64), o.logical_buffer(g))


def test_jump_host_generate_across_staging_tiles(oracle):
    """One stream longer than a 2^26-word staging slot: generate() tiles it
    (each tile a jump fill continuing the previous one, copies overlapping
    generation) -- the whole stream is the reference's."""
    n = (1 << 26) + 1000
    e = one(4242)
    g = e.generate(n)
    assert np.array_equal(g[0], oracle.stream(4242, n))
    host_rows = [np.zeros(3 * M + 7, dtype=np.uint64)]
    import ctypes

    arr = (ctypes.c_void_p * 1)(host_rows[0].ctypes.data)
    assert xg._lib.lib.xg_generate_host_rows(e.handle, 3 * M + 7, arr, None) == 0
    assert np.array_equal(host_rows[0], oracle.stream(4242, n + 3 * M + 7)[n:].astype(np.uint64))


@pytest.mark.parametrize("P,n", [(100, (1 << 21) + 777), (65, (1 << 20) + 1), (7, 3 * M + 64), (300, 906752),
                                 (2, (1 << 18) + 3), (600, (1 << 18) + 64)])
def test_jump_many_streams_any_length(oracle, P, n):
    """2 .. 700 streams of any length >= 2^18: Q segments of 2^j words per
    stream in one fill (output rows in groups of Q, one stream row apart --
    the fill kernels' row-group addressing) plus the per-stream remainders on
    the side stream; odd lengths send the fills to the word-lane kernel."""
    e = xg.BlockEnsemble(GP32, 500 + P, P, 63)
    o = oracle.ensemble(500 + P, P)
    assert np.array_equal(host(e.fill_u32(n)), o.fill_u32(n))
    assert np.array_equal(host(e.fill_f64(n // 2)).view(np.uint64), o.fill_f64(n // 2).view(np.uint64))
    k = 32 * (n // 64)
    assert int(e.mc_pi(k).item()) == int(o.mc_hits(k).sum())
    assert np.array_equal(host(e.fill_u32(333)), o.fill_u32(333))
    for g in (0, P - 1):
        buf, wy = e.block_state(g)
        assert wy == o.weyl(g) and np.array_equal(np.array(buf, dtype=np.uint64), o.logical_buffer(g))

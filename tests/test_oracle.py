"""Pins the CPU oracle (oracle/xg_oracle.c) before it is trusted as the checker.

Sources of truth, in order: the reference's own known-answer vectors
(proj/tests/test_xorgens.cpp:129-137,163-173, proj/tests/golden/
gen_gp32_seed42_count4.hex), the golden fixtures generated from the reference
itself (tests/golden/ref_vectors.json via oracle/_ref), and -- when it is
built -- oracle/_ref called live.  Mirrors the reference's hot-path unit tests
(proj/tests/test_xorgens.cpp, test_parallel.cpp, test_seeding.cpp,
test_params.cpp).
"""
import ctypes

import numpy as np
import pytest

from helpers import u32
from oracle import OracleEnsemble, Params

KAT_SEED0 = ["a2c5f91b", "bd5797de", "cac8bc67", "7ba44aee", "11254d96", "198b2ab0", "656ea882",
             "9a94ce3e", "45568ed8", "1a4d6e4b", "bdcd2db4", "4bb14332", "74e6e085", "4cafd1e2",
             "04dbdceb", "07ba0f22"]  # proj/tests/test_xorgens.cpp:165-170
KAT_SEED42 = ["a61e8308", "8469633b", "80f8af0d", "57f95c64"]  # proj/tests/golden/gen_gp32_seed42_count4.hex


def test_reference_kat_seed0(oracle):
    assert np.array_equal(oracle.stream(0, 16), u32(KAT_SEED0))


def test_reference_golden_seed42(oracle):
    assert np.array_equal(oracle.stream(42, 4), u32(KAT_SEED42))


def test_weyl_sequence(oracle):
    # proj/tests/test_xorgens.cpp:129-137: from weyl 0, w=32 -> 2654435769, 1013904242, 3668340011
    p = oracle.gp32()
    st = ctypes.create_string_buffer(oracle.state_size)
    buf = np.zeros(128, dtype=np.uint64)
    buf[0] = 1
    oracle.lib.xgo_from_raw(st, ctypes.byref(p), buf.ctypes.data_as(ctypes.c_void_p), 0)
    oracle.lib.xgo_weyl_next.restype = ctypes.c_uint64
    oracle.lib.xgo_weyl_next.argtypes = [ctypes.c_void_p]
    got = [oracle.lib.xgo_weyl_next(st) for _ in range(3)]
    assert got == [2654435769, 1013904242, 3668340011]


def test_golden_streams(oracle, golden):
    for seed, words in golden["streams"].items():
        assert np.array_equal(oracle.stream(int(seed), len(words)), u32(words)), seed


def test_golden_seeded_state(oracle, golden):
    e = oracle.ensemble(1, 1)
    g = golden["seeded_state_seed1"]
    assert np.array_equal(e.logical_buffer(0).astype(np.uint32), u32(g["buffer"]))
    assert e.weyl(0) == int(g["weyl"], 16)


def test_golden_alt_params(oracle, golden):
    for entry in golden["alt_params"]:
        p = Params(*entry["params"])
        assert oracle.check(p) == entry["check"] == 0
        for seed, words in entry["streams"].items():
            assert np.array_equal(oracle.stream(int(seed), len(words), p), u32(words))


def test_golden_generate_block_major_and_continuation(oracle, golden):
    # proj/src/parallel.cpp:84-135, proj/tests/test_parallel.cpp:114-153
    for g in golden["generate"]:
        e = oracle.ensemble(g["base_seed"], g["blocks"])
        first = e.fill_u32(g["per_block"])
        second = e.fill_u32(g["per_block"])
        assert np.array_equal(first, np.stack([u32(r) for r in g["first"]]))
        assert np.array_equal(second, np.stack([u32(r) for r in g["second"]]))


def test_golden_from_raw(oracle, golden):
    g = golden["from_raw"]
    buf = u32(g["buffer"]).astype(np.uint64)
    e = oracle.from_raw(buf[None, :], [int(g["weyl"], 16)])
    assert np.array_equal(e.fill_u32(len(g["stream"]))[0], u32(g["stream"]))


def test_golden_conversions(oracle, golden):
    g = golden["conversions_seed42"]
    w = oracle.stream(42, 256)
    f32 = oracle.ensemble(42, 1).fill_f32(256)[0]
    assert np.array_equal(f32.view(np.uint32), u32(g["f32_bits"]))
    assert np.array_equal(oracle.f32(w).view(np.uint32), u32(g["f32_bits"]))
    f64 = oracle.ensemble(42, 1).fill_f64(128)[0]
    assert [f"{v:016x}" for v in f64.view(np.uint64)] == g["f64_bits"]
    assert int(oracle.ensemble(42, 1).mc_hits(128)[0]) == g["mc_hits_128_samples"]
    # scalar conventions agree with the vector forms
    lib = oracle.lib
    for i in range(0, 256, 2):
        assert lib.xgo_u32pair_to_u64(int(w[i]), int(w[i + 1])) == int(g["u64"][i // 2], 16)
        assert lib.xgo_u32pair_to_f64(int(w[i]), int(w[i + 1])) == f64[i // 2]


def test_config1_checksum(oracle, golden):
    # BASELINE config 1: seed 1, 10^8 words.
    g = golden["config1"]
    e = oracle.ensemble(1, 1)
    x, s = e.checksums(g["n"])
    assert f"{int(x[0]):08x}" == g["xor"]
    assert f"{int(s[0]):016x}" == g["sum"]


def test_config2_checksum(oracle, golden):
    # BASELINE config 2: P = 2^14 streams x 2^16 words from base_seed 1.
    g = golden["config2"]
    P, n = g["streams"], g["per_stream"]
    e = oracle.ensemble(g["base_seed"], P)
    x, s = e.checksums(n)
    gx = int(np.bitwise_xor.reduce(x))
    # block-major weighted sum: sum_k w_gk (g*n + k + 1) = s_g + g*n*sum_k w_gk
    e2 = oracle.ensemble(g["base_seed"], P)
    words_sum = np.zeros(P, dtype=np.uint64)
    chunk = 1024
    for g0 in range(0, P, chunk):
        sub = OracleEnsemble(oracle, oracle.gp32(), g["base_seed"], chunk, first_stream=g0)
        words_sum[g0:g0 + chunk] = sub.fill_u32(n).astype(np.uint64).sum(axis=1, dtype=np.uint64)
    del e2
    gs = int(np.sum(s + np.arange(P, dtype=np.uint64) * np.uint64(n) * words_sum, dtype=np.uint64))
    assert f"{gx:08x}" == g["xor"]
    assert f"{gs:016x}" == g["wsum"]
    assert [f"{int(v):08x}" for v in x[:16]] == g["per_stream_xor_first16"]


def test_batch_step_equals_serial_all_lane_counts(oracle):
    # proj/tests/test_parallel.cpp:33-48
    for p in (oracle.gp32(), oracle.lib.xgo_tiny_r4w16_params()):
        bound = oracle.lib.xgo_lane_bound(ctypes.byref(p))
        serial = oracle.ensemble(99, 1, p).next_words(0, 4096)
        for lanes in range(1, bound + 1, 7 if bound > 8 else 1):
            e = oracle.ensemble(99, 1, p)
            got = []
            out = np.zeros(lanes, dtype=np.uint64)
            while len(got) < 4096:
                assert oracle.lib.xgo_batch_step(e._state(0), lanes, out.ctypes.data_as(ctypes.c_void_p)) == 0
                got.extend(out.tolist())
            assert np.array_equal(np.array(got[:4096], dtype=np.uint64), serial), lanes


def test_lane_bound_and_hazard(oracle):
    # proj/tests/test_parallel.cpp:50-89, proj/tests/acceptance.cpp:88-108
    p = oracle.gp32()
    assert oracle.lib.xgo_lane_bound(ctypes.byref(p)) == 63
    e = oracle.ensemble(0, 1)
    out = np.zeros(128, dtype=np.uint64)
    ptr = out.ctypes.data_as(ctypes.c_void_p)
    assert oracle.lib.xgo_batch_step(e._state(0), 0, ptr) == -1
    assert oracle.lib.xgo_batch_step(e._state(0), 64, ptr) == -1
    # unsynchronised schedule is exact up to the bound ...
    serial = oracle.ensemble(321, 1).next_words(0, 63 * 8)
    h = oracle.ensemble(321, 1)
    got = []
    for _ in range(8):
        oracle.lib.xgo_unsynchronized_batch(h._state(0), 63, ptr)
        got.extend(out[:63].tolist())
    assert np.array_equal(np.array(got, dtype=np.uint64), serial)
    # ... and breaks one lane past it
    differs = False
    for seed in range(4):
        h = oracle.ensemble(seed, 1)
        oracle.lib.xgo_unsynchronized_batch(h._state(0), 64, ptr)
        differs |= not np.array_equal(out[:64], oracle.ensemble(seed, 1).next_words(0, 64))
    assert differs


def test_consecutive_seeds_and_wrap(oracle):
    # proj/src/parallel.cpp:93-94 (uint64 wrap of base_seed + i)
    e = oracle.ensemble(2**64 - 1, 2)
    words = e.fill_u32(32)
    assert np.array_equal(words[0], oracle.stream(2**64 - 1, 32))
    assert np.array_equal(words[1], oracle.stream(0, 32))


def test_schedule_independence(oracle):
    # proj/tests/test_parallel.cpp:132-143 (threads)
    ref = None
    for threads in (1, 2, 3, 8, 64):
        e = oracle.ensemble(42, 8)
        e.o.threads = threads
        got = e.fill_u32(500)
        if ref is None:
            ref = got
        assert np.array_equal(got, ref)
    oracle.threads = __import__("os").cpu_count() or 1


PARAM_CASES = [
    ((128, 65, 15, 14, 12, 17, 32), 0),
    ((128, 64, 15, 14, 12, 17, 32), 3),   # gcd
    ((2, 1, 1, 1, 1, 1, 8), 0),
    ((2, 1, 1, 1, 1, 1, 12), 1),          # bad w (checked first)
    ((2, 0, 1, 1, 1, 1, 8), 2),
    ((2, 2, 1, 1, 1, 1, 8), 2),
    ((2, 1, 8, 1, 1, 1, 8), 4),
    ((2, 1, 1, 0, 1, 1, 8), 4),
    ((0, 0, 0, 0, 0, 0, 7), 1),
    ((4, 2, 0, 0, 0, 0, 16), 3),          # gcd checked before shifts
]


@pytest.mark.parametrize("rsabcdw,code", PARAM_CASES)
def test_param_error_codes(oracle, rsabcdw, code):
    # proj/tests/test_params.cpp:20-61 and the check order of proj/src/params.cpp:22-37
    p = oracle.params(*rsabcdw, omega=159 if rsabcdw[6] == 12 else None)
    assert oracle.check(p) == code


def test_param_gamma_and_omega_codes(oracle):
    p = oracle.params(2, 1, 1, 1, 1, 1, 8, omega=158)
    assert oracle.check(p) == 6
    p = oracle.params(2, 1, 1, 1, 1, 1, 8, gamma=8)
    assert oracle.check(p) == 5


def test_oracle_matches_live_reference(oracle, reference):
    # the restatement against the reference sources themselves
    rng = np.random.default_rng(7)
    for seed in [0, 1, 2**64 - 1, *rng.integers(0, 2**63, 5).tolist()]:
        assert np.array_equal(oracle.stream(seed, 5000), reference.stream(seed, 5000, oracle.gp32()).astype(np.uint32))
    for t in (oracle.lib.xgo_tiny_r2w8_params(), oracle.lib.xgo_tiny_r2w16_params(),
              oracle.lib.xgo_tiny_r4w16_params()):
        e = oracle.ensemble(5, 1, t)
        assert np.array_equal(e.next_words(0, 3000), reference.stream(5, 3000, t))
    for rs, _ in PARAM_CASES:
        p = oracle.params(*rs, omega=159 if rs[6] == 12 else None)
        assert oracle.check(p) == reference.check(p)


def test_golden_raw_streams(oracle, golden):
    # RawXorgens (proj/include/xg/baselines.hpp:60-71): seeding as XorgensState,
    # then step_linear only.
    for seed, words in golden["raw_streams"].items():
        e = oracle.ensemble(int(seed), 1)
        assert np.array_equal(e.fill_raw_u32(len(words))[0], u32(words)), seed


def _xs(x, l, r):
    t = (x ^ (x << np.uint32(l))) & np.uint32(0xFFFFFFFF)
    return t ^ (t >> np.uint32(r))


def _shfl(vals, src):
    return vals[src]


@pytest.mark.parametrize("s", [65, 67, 79, 93, 95])
def test_pair_lane_schedule_equals_serial(oracle, s):
    """The pair-lane kernel's schedule (paper_1108_0486_b200/csrc/xg_pairs.cuh),
    simulated lane by lane with its exact shuffle sources and giver selects:
    lane l holds pairs A = (W[2l], W[2l+1]) and B = (W[64+2l], W[65+2l]), and
    a double step makes the 64 words N[2l], N[2l+1] from the pre-step window.
    Must equal the serial linear recurrence (RawXorgens::next,
    proj/include/xg/baselines.hpp:60-71) for every r = 128 set with
    r - s < 64 (s = 65 is xorgensgp32: one shuffle, the other operand own)."""
    p = oracle.params(128, s, 15, 14, 12, 17, 32) if s == 65 else oracle.params(128, s, 11, 7, 9, 19, 32)
    assert oracle.check(p) == 0
    q = 128 - s  # 33..63: the J = 1 sets (r - s = 32 + delta)
    m = 16 + (q - 32 - 1) // 2  # make_pair_lane: q = 2m + 1
    assert q == 2 * m + 1
    e = oracle.ensemble(5, 1, p)
    W = e.logical_buffer(0).astype(np.uint32)
    want = e.fill_raw_u32(64 * 9)[0]
    lane = np.arange(32)
    A = np.stack([W[2 * lane], W[2 * lane + 1]], axis=1)
    B = np.stack([W[64 + 2 * lane], W[65 + 2 * lane]], axis=1)
    got = []
    for _ in range(9):
        if s == 65:  # GP32 specialisation: give = lane == 31 ? A.y : B.y from lane l-1
            give = np.where(lane == 31, A[:, 1], B[:, 1])
            ty = _shfl(give, (lane + 31) & 31)
            tx = B[:, 0]
        else:  # runtime sets: two shuffles
            ty = _shfl(np.where(lane >= m, A[:, 1], B[:, 1]), (lane + m) & 31)
            tx = _shfl(np.where(lane >= m + 1, A[:, 0], B[:, 0]), (lane + m + 1) & 31)
        N = np.stack([_xs(A[:, 0], p.a, p.b) ^ _xs(ty, p.c, p.d),
                      _xs(A[:, 1], p.a, p.b) ^ _xs(tx, p.c, p.d)], axis=1).astype(np.uint32)
        got.append(N.reshape(-1))  # lane l's pair = words 2l, 2l+1 of the step
        A, B = B, N
    assert np.array_equal(np.concatenate(got), want)


def _battery_or_skip():
    from oracle import Battery
    try:
        return Battery()
    except FileNotFoundError as e:  # pragma: no cover - needs the reference tree
        pytest.skip(str(e))


def test_gf2_rank32_matches_reference():
    """The oracle's 32 x 32 GF(2) rank against the reference's own gf2_rank
    (proj/src/stattests/gf2.cpp, compiled into oracle/_ref) on random,
    duplicated-row, low-rank and zero matrices."""
    from oracle import Oracle
    o, b = Oracle(), _battery_or_skip()
    rng = np.random.default_rng(11)
    for t in range(3000):
        rows = rng.integers(0, 2**32, size=32, dtype=np.uint64).astype(np.uint32)
        kind = t % 6
        if kind == 1:
            rows[rng.integers(0, 32)] = rows[rng.integers(0, 32)]
        elif kind == 2:
            rows &= np.uint32(0xFFFF0000)
        elif kind == 3:
            basis = rows[:int(rng.integers(1, 32))]
            rows = np.array([np.bitwise_xor.reduce(basis[rng.integers(0, 2, size=basis.size) == 1])
                             if basis.size else 0 for _ in range(32)], dtype=np.uint32)
        elif kind == 4:
            rows[:] = 0
        elif kind == 5:
            rows = (np.uint32(1) << np.arange(32, dtype=np.uint32)).astype(np.uint32)
        want = b.gf2_rank32(rows)
        assert int(o.lib.xgo_gf2_rank32(rows.ctypes.data)) == want, t
    assert b.gf2_rank32(np.zeros(32, dtype=np.uint32)) == 0


def test_rank_counts_give_the_reference_statistic():
    """Bins from the oracle's counting loop, turned into the statistic by the
    Python mirror's matrix_rank_statistic, equal the reference's
    matrix_rank_test (proj/src/stattests/tests.cpp:81-126) on the same words:
    chi-square bit for bit, p-value to 1e-12."""
    import paper_1108_0486_b200 as xg
    from oracle import Oracle
    b = _battery_or_skip()
    o = Oracle()
    for seed, m in ((1, 38), (42, 1000), (7, 4321)):
        words = o.ensemble(seed, 1).fill_u32(32 * m)[0]
        counts = o.ensemble(seed, 1).rank_counts(m)[0]
        assert int(counts.sum()) == m
        chi2, p = xg.matrix_rank_statistic(counts)
        rchi2, rp = b.matrix_rank(words, m)
        assert chi2 == rchi2
        assert abs(p - rp) <= 1e-12 * max(1.0, rp)


def test_linear_complexity_statistic_equals_reference():
    """The reference's per-block Berlekamp-Massey (gf2.cpp:62-110) histogram,
    binned by the Python mirror's linear_complexity_statistic, gives the
    reference's linear_complexity_test (tests.cpp:128-178) statistic bit for
    bit and its p-value to 1e-12, on oracle words, for even and odd K."""
    import paper_1108_0486_b200 as xg
    from oracle import Oracle
    b = _battery_or_skip()
    o = Oracle()
    for seed, K, nb in ((1, 1000, 200), (5, 500, 300), (9, 129, 400), (3, 128, 1000)):
        w = o.ensemble(seed, 1).fill_u32((K * nb + 31) // 32)[0]
        hist = b.lc_histogram(w, K, nb)
        assert int(hist.sum()) == nb
        chi2, p = xg.linear_complexity_statistic(hist, K)
        rchi2, rp = b.linear_complexity(w, K, nb)
        assert chi2 == rchi2
        assert abs(p - rp) <= 1e-12 * max(1.0, rp)


def test_berlekamp_massey_known_sequences():
    """The reference's own KATs (proj/tests/acceptance.cpp:369-382): the
    v13 sequence has complexity 4, alternating 24 bits complexity 2."""
    b = _battery_or_skip()
    assert b.berlekamp_massey(np.array([1, 1, 0, 1, 0, 1, 1, 1, 1, 0, 0, 0, 1], dtype=np.uint8)) == 4
    assert b.berlekamp_massey(np.array([0, 1] * 12, dtype=np.uint8)) == 2
    lfsr = [1, 0, 0, 0, 0, 0, 0, 0]
    while len(lfsr) < 24:
        i = len(lfsr)
        lfsr.append(lfsr[i - 8] ^ lfsr[i - 4] ^ lfsr[i - 3] ^ lfsr[i - 2])
    assert b.berlekamp_massey(np.array(lfsr, dtype=np.uint8)) == 8
    assert b.berlekamp_massey(np.zeros(64, dtype=np.uint8)) == 0
    assert b.berlekamp_massey(np.array([0] * 63 + [1], dtype=np.uint8)) == 64


def _row_digests_np(words: np.ndarray):
    """Per-row (xor, sum, sum e_k (k+1)) of a 2-D uint32 array (mod 2^64)."""
    w = words.astype(np.uint64)
    k = np.arange(1, words.shape[1] + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return (np.bitwise_xor.reduce(words, axis=1).astype(np.uint32),
                w.sum(axis=1, dtype=np.uint64), (w * k).sum(axis=1, dtype=np.uint64))


@pytest.fixture(scope="module")
def full_size():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "full_size.json")) as f:
        return json.load(f)


def test_full_size_golden_consistent_with_config2(golden, full_size):
    """Chunk 0 of the 2^34-word golden is the 2^30-word config-2 fill."""
    c0 = full_size["u32"]["chunks"][0]
    assert c0["xor"] == golden["config2"]["xor"] and c0["wsum"] == golden["config2"]["wsum"]
    assert len(full_size["u32"]["chunks"]) == 16 and len(full_size["mc"]["chunk_hits"]) == 8
    hits = full_size["mc"]["total_hits_2p32"]
    assert hits == sum(full_size["mc"]["chunk_hits"])
    assert abs(4.0 * hits / 2**32 - np.pi) < 6 * 1.6e-6 * 2**4  # sigma(pi_hat) at 2^32 samples ~ 2.5e-5


def test_full_size_golden_pinned_by_restatement(oracle, full_size):
    """The full-size goldens come from the reference's own words
    (make_golden.py --full-size); the C restatement reproduces the last u32
    chunk (streams 15*2^14 ...: 2^30 words, config 4) and the last MC chunk
    (2^14 streams x 2^15 samples) exactly."""
    from paper_1108_0486_b200.digest import chunk_record

    C, per = full_size["chunk_streams"], full_size["u32"]["per_stream"]
    piece = 1024
    parts = []
    for g0 in range(15 * C, 16 * C, piece):
        sub = OracleEnsemble(oracle, oracle.gp32(), 1, piece, first_stream=g0)
        parts.append(_row_digests_np(sub.fill_u32(per)))
    rec = chunk_record(*(np.concatenate([p[i] for p in parts]) for i in range(3)), per)
    assert rec == full_size["u32"]["chunks"][15]
    spp = full_size["mc"]["samples_per_stream"]
    sub = OracleEnsemble(oracle, oracle.gp32(), 1, C, first_stream=7 * C)
    assert int(sub.mc_hits(spp).sum()) == full_size["mc"]["chunk_hits"][7]

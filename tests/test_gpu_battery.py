"""The reference's battery run on the GPU (paper_1108_0486_b200/battery.py)
equals the reference's own run_battery (proj/src/stattests/battery.cpp:72-130,
compiled into oracle/_ref/libxgref_battery.so) over the same stream: every
test's statistic and p-value bit for bit, every verdict -- for the quick and
the default configuration."""
import json
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1108_0486_b200 as xg  # noqa: E402
from paper_1108_0486_b200.battery import BatteryConfig, run_battery_gpu  # noqa: E402


def _battery():
    from oracle import Battery
    try:
        return Battery()
    except FileNotFoundError as e:  # pragma: no cover
        pytest.skip(str(e))


def _words_consumed(cfg):
    return ((cfg.monobit_bits + 31) // 32 + (cfg.runs_bits + 31) // 32 + 32 * cfg.rank_matrices +
            (cfg.lc_block_length * cfg.lc_blocks + 31) // 32 +
            cfg.birthday_draws * cfg.birthday_rounds)


@pytest.mark.parametrize("quick,seed", [(True, 1), (True, 42), (False, 7)])
def test_gpu_battery_equals_reference(quick, seed):
    b = _battery()
    cfg = BatteryConfig.quick() if quick else BatteryConfig.defaults()
    p = xg.xorgensgp32_params()
    t0 = time.perf_counter()
    rep = run_battery_gpu(p, seed, cfg)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    words = xg.BlockEnsemble(p, seed, 1, 63).fill_u32(_words_consumed(cfg)).cpu().numpy()[0]
    t0 = time.perf_counter()
    verdict, js = b.run(words, quick=quick, label="xorgensgp32")
    t_ref = time.perf_counter() - t0
    ref = json.loads(js)
    assert rep["overall"] == ref["overall"] == verdict
    assert [t["name"] for t in rep["tests"]] == [t["name"] for t in ref["tests"]]
    for mine, theirs in zip(rep["tests"], ref["tests"]):
        assert mine["n"] == theirs["n"], mine["name"]
        assert mine["statistic"] == theirs["statistic"], mine["name"]
        assert mine["p"] == theirs["p"], mine["name"]
        assert mine["verdict"] == theirs["verdict"], mine["name"]
    print(f"battery {'quick' if quick else 'default'}: GPU {t_gpu:.3f} s, reference {t_ref:.3f} s")


def test_ones_runs_and_birthday_kernels_direct():
    """The counting kernels on buffers with ragged bit counts."""
    rng = np.random.default_rng(3)
    w = rng.integers(0, 2**32, size=1000, dtype=np.uint64).astype(np.uint32)
    bits = np.unpackbits(w.byteswap().view(np.uint8)).astype(np.int64)
    dev = torch.from_numpy(w.view(np.int32)).cuda()
    for n in (1, 31, 32, 33, 100, 999, 31999, 32000):
        out = torch.zeros(2, dtype=torch.int64, device="cuda")
        xg._lib.lib.xg_bits_ones_runs(dev.data_ptr(), n, out.data_ptr(), None)
        ones, trans = out.tolist()
        assert ones == int(bits[:n].sum())
        assert trans == int(np.count_nonzero(bits[1:n] != bits[:n - 1]))
    for nd, t in ((2, 32), (100, 20), (4096, 32), (8192, 30), (5000, 31)):
        rounds = 3
        v = rng.integers(0, 2**32, size=nd * rounds, dtype=np.uint64)
        dup = 0
        for r in v.reshape(rounds, nd):
            sp = np.sort(np.diff(np.sort(r >> np.uint64(32 - t))))
            dup += int(np.count_nonzero(sp[1:] == sp[:-1]))
        d = torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda()
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        assert xg._lib.lib.xg_birthday_duplicates(d.data_ptr(), nd, rounds, t, out.data_ptr(), None) == 0
        assert int(out.item()) == dup, (nd, t)


def test_battery_runs_every_w32_set_and_the_raw_stream():
    """A w = 32 set the fused rank test cannot take (r - s >= 64, J = 2) and
    the Weyl-ablated stream run the whole battery: the matrix-rank test over
    stored words (xg_rank_words), the linear complexity test over stored raw
    words (xg_lc_words).  Reports equal the reference's run_battery over the
    same words."""
    from paper_1108_0486_b200.battery import BatteryConfig, run_battery_gpu

    b = _battery()
    cfg = BatteryConfig.quick()
    j2 = xg.GeneratorParams(128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11)
    for p, raw in ((j2, False), (xg.xorgensgp32_params(), True)):
        rep = run_battery_gpu(p, 5, cfg, raw=raw)
        e = xg.BlockEnsemble(p, 5, 1, xg.lane_bound(p))
        n = _words_consumed(cfg)
        words = (e.fill_raw_u32(n) if raw else e.fill_u32(n)).cpu().numpy()[0]
        verdict, js = b.run(words, quick=True, label="x")
        ref = json.loads(js)
        assert rep["overall"] == ref["overall"] == verdict
        for mine, theirs in zip(rep["tests"], ref["tests"]):
            assert (mine["statistic"], mine["p"], mine["verdict"]) == \
                   (theirs["statistic"], theirs["p"], theirs["verdict"]), (raw, mine["name"])


def test_rank_and_lc_over_word_buffers():
    """xg_rank_words / xg_lc_words against the reference's own gf2_rank and
    berlekamp_massey on random words (odd matrix counts, blocks straddling
    words, K above the register path's 1023)."""
    from oracle import Battery

    b = _battery()
    rng = np.random.default_rng(11)
    w = rng.integers(0, 2**32, size=32 * 41, dtype=np.uint64).astype(np.uint32)
    dev = torch.from_numpy(w.view(np.int32)).cuda()
    for m in (1, 2, 7, 41):
        out = torch.zeros(3, dtype=torch.int64, device="cuda")
        assert xg._lib.lib.xg_rank_words(dev.data_ptr(), m, out.data_ptr(), None) == 0
        ranks = [b.gf2_rank32(w[32 * k:32 * k + 32]) for k in range(m)]
        want = [sum(r == 32 for r in ranks), sum(r == 31 for r in ranks), sum(r < 31 for r in ranks)]
        assert out.tolist() == want, m
    for k, nb in ((128, 9), (1000, 3), (1023, 2), (2000, 2)):
        hist = torch.zeros(k + 1, dtype=torch.int64, device="cuda")
        assert xg._lib.lib.xg_lc_words(dev.data_ptr(), dev.numel(), k, nb, hist.data_ptr(), None) == 0
        assert np.array_equal(hist.cpu().numpy(), b.lc_histogram(w, k, nb).astype(np.int64)), k
    hist = torch.zeros(2001, dtype=torch.int64, device="cuda")
    assert xg._lib.lib.xg_lc_words(dev.data_ptr(), 10, 2000, 1, hist.data_ptr(), None) == \
        xg._lib.XG_EINVAL


def test_handle_less_calls_reject_host_pointers():
    """The calls without a handle take their device from the input pointer;
    a host pointer is XG_EINVAL, not a fault."""
    host = np.zeros(64, dtype=np.uint32)
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    assert xg._lib.lib.xg_bits_ones_runs(host.ctypes.data, 64, out.data_ptr(), None) == xg._lib.XG_EINVAL


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_battery_on_a_non_current_device(reference):  # pragma: no cover - 1-GPU boxes
    from paper_1108_0486_b200.battery import BatteryConfig, run_battery_gpu

    torch.cuda.set_device(0)
    a = run_battery_gpu(xg.xorgensgp32_params(), 3, BatteryConfig.quick(), device=1)
    b = run_battery_gpu(xg.xorgensgp32_params(), 3, BatteryConfig.quick(), device=0)
    assert a == b


def _words_consumed_w(cfg, w):
    """Words a run_battery consumes from a w-bit source (BitSource reads w
    bits per word; each test starts a fresh BitSource)."""
    per = lambda bits: (bits + w - 1) // w  # noqa: E731
    n = 0
    if cfg.run_monobit:
        n += per(cfg.monobit_bits)
    if cfg.run_runs:
        n += per(cfg.runs_bits)
    if cfg.run_matrix_rank:
        n += per(1024 * cfg.rank_matrices)
    if cfg.run_linear_complexity:
        n += per(cfg.lc_block_length * cfg.lc_blocks)
    if cfg.run_birthday:
        n += cfg.birthday_draws * cfg.birthday_rounds
    return n


def _cfg_text(cfg):
    b = lambda v: "true" if v else "false"  # noqa: E731
    return (f"monobit.enabled = {b(cfg.run_monobit)}\nmonobit.bits = {cfg.monobit_bits}\n"
            f"runs.enabled = {b(cfg.run_runs)}\nruns.bits = {cfg.runs_bits}\n"
            f"matrix_rank.enabled = {b(cfg.run_matrix_rank)}\nmatrix_rank.matrices = {cfg.rank_matrices}\n"
            f"linear_complexity.enabled = {b(cfg.run_linear_complexity)}\n"
            f"linear_complexity.block_length = {cfg.lc_block_length}\n"
            f"linear_complexity.blocks = {cfg.lc_blocks}\n"
            f"birthday.enabled = {b(cfg.run_birthday)}\nbirthday.draws = {cfg.birthday_draws}\n"
            f"birthday.bits = {cfg.birthday_bits}\nbirthday.rounds = {cfg.birthday_rounds}\n")


@pytest.mark.parametrize("tiny,raw,quick", [("r2w8", True, False), ("r4w16", False, True),
                                            ("r2w16", True, True)])
def test_battery_on_8_and_16_bit_sets_equals_reference(reference, tiny, raw, quick):
    """The 8- and 16-bit verification sets read w bits per word (BitSource):
    packed into the 32-bit bit stream on the GPU (xg_pack_words), the report
    equals the reference's run_battery over the same w-bit words.  r2w8 raw
    is the reference's own negative control (acceptance.cpp:253-265)."""
    from oracle import Params

    b = _battery()
    p = getattr(xg, f"tiny_{tiny}_params")()
    cfg = BatteryConfig.quick() if quick else BatteryConfig.defaults()
    cfg.run_birthday = False  # t_bits = 32 cannot apply to w < 32 words (tests.cpp:179-180)
    rep = run_battery_gpu(p, 1, cfg, raw=raw)
    pr = Params(p.r, p.s, p.a, p.b, p.c, p.d, p.w, p.omega, p.gamma)
    n = _words_consumed_w(cfg, p.w)
    words = (reference.raw_stream(1, n, pr) if raw else reference.stream(1, n, pr))
    verdict, js = b.run_config(words, p.w, _cfg_text(cfg))
    ref = json.loads(js)
    assert rep["overall"] == ref["overall"] == verdict
    for mine, theirs in zip(rep["tests"], ref["tests"]):
        assert (mine["name"], mine["n"], mine["statistic"], mine["p"], mine["verdict"]) == \
               (theirs["name"], theirs["n"], theirs["statistic"], theirs["p"], theirs["verdict"])


def test_quality_split_on_gpu():
    """acceptance.cpp:241-270 (criterion 4) with the counting on the GPU:
    xorgensgp32 passes the default battery; the Weyl-ablated tiny r2w8
    (birthday disabled) fails, caught by linear complexity or matrix rank
    with p < 1e-10."""
    good = run_battery_gpu(xg.xorgensgp32_params(), 1, BatteryConfig.defaults())
    assert good["overall"] == "pass"
    cfg = BatteryConfig.defaults()
    cfg.run_birthday = False
    bad = run_battery_gpu(xg.tiny_r2w8_params(), 1, cfg, raw=True)
    assert bad["overall"] == "fail"
    assert any(t["name"] in ("linear_complexity", "matrix_rank") and t["verdict"] == "fail"
               and t["p"] < 1e-10 for t in bad["tests"])

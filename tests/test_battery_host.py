"""Host side of the GPU battery (paper_1108_0486_b200/battery.py,
pvalues.py) without a GPU: the device's integer results (ones, runs, rank
bins, complexity histogram, birthday duplicates) are computed here from
oracle words with numpy and the reference's own gf2_rank / berlekamp_massey,
and the statistics, p-values and verdicts built from them must equal the
reference's run_battery report over the same words (battery.cpp:72-130)."""
import json
import math

import numpy as np
import pytest

from oracle import Oracle


def _battery():
    from oracle import Battery
    try:
        return Battery()
    except FileNotFoundError as e:  # pragma: no cover - needs the reference tree
        pytest.skip(str(e))


def _bits(words):
    return np.unpackbits(np.ascontiguousarray(words, dtype=np.uint32).byteswap().view(np.uint8))


def test_host_statistics_equal_reference_report():
    import paper_1108_0486_b200.battery as xb
    from paper_1108_0486_b200 import linear_complexity_statistic, matrix_rank_statistic
    from paper_1108_0486_b200.pvalues import poisson_upper_tail

    b = _battery()
    cfg = xb.BatteryConfig.quick()
    o = Oracle()
    seed = 20261017
    nw = {"mono": (cfg.monobit_bits + 31) // 32, "runs": (cfg.runs_bits + 31) // 32,
          "rank": 32 * cfg.rank_matrices,
          "lc": (cfg.lc_block_length * cfg.lc_blocks + 31) // 32,
          "bd": cfg.birthday_draws * cfg.birthday_rounds}
    words = o.ensemble(seed, 1).fill_u32(sum(nw.values()))[0]
    verdict, js = b.run(words, quick=True, label="x")
    ref = {t["name"]: t for t in json.loads(js)["tests"]}
    pos = 0

    def take(k):
        nonlocal pos
        w = words[pos:pos + nw[k]]
        pos += nw[k]
        return w

    bits = _bits(take("mono"))[:cfg.monobit_bits]
    n = cfg.monobit_bits
    abs_s = abs(float(2 * int(bits.sum()) - n))
    assert ref["monobit"]["statistic"] == abs_s / math.sqrt(float(n))
    assert ref["monobit"]["p"] == math.erfc(abs_s / math.sqrt(2.0 * float(n)))

    bits = _bits(take("runs"))[:cfg.runs_bits].astype(np.int64)
    runs = 1 + int(np.count_nonzero(bits[1:] != bits[:-1]))
    assert ref["runs"]["statistic"] == float(runs)

    rw = take("rank").reshape(-1, 32)
    counts = [0, 0, 0]
    for m in rw:
        r = b.gf2_rank32(m)
        counts[0 if r == 32 else (1 if r == 31 else 2)] += 1
    chi2, p = matrix_rank_statistic(counts)
    assert ref["matrix_rank"]["statistic"] == chi2 and ref["matrix_rank"]["p"] == p

    hist = b.lc_histogram(take("lc"), cfg.lc_block_length, cfg.lc_blocks)
    chi2, p = linear_complexity_statistic(hist, cfg.lc_block_length)
    assert ref["linear_complexity"]["statistic"] == chi2 and ref["linear_complexity"]["p"] == p

    bd = take("bd").reshape(cfg.birthday_rounds, cfg.birthday_draws).astype(np.uint64)
    dup = 0
    for r in bd:
        sp = np.sort(np.diff(np.sort(r)))
        dup += int(np.count_nonzero(sp[1:] == sp[:-1]))
    lam = float(cfg.birthday_draws) ** 3 / math.pow(2.0, cfg.birthday_bits + 2.0)
    assert ref["birthday_spacings"]["statistic"] == float(dup)
    assert ref["birthday_spacings"]["p"] == poisson_upper_tail(dup, lam * cfg.birthday_rounds)
    assert verdict in ("pass", "suspect")

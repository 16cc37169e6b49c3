"""The GPU backend of the reference CLI (paper_1108_0486_b200/lib/xgen), checked
the way the reference checks its own xgen (proj/tests/test_cli.cpp): golden
stream file, block-major concatenation of consecutive seeds, lane invariance,
exit codes, the params table.  Exit-code cases that fail before any device
work run on CPU; stream cases need the GPU."""
import os
import subprocess

import numpy as np
import pytest

from helpers import u32

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
XGEN = os.path.join(ROOT, "paper_1108_0486_b200", "lib", "xgen")
GOLDEN_SEED42 = "a61e8308\n8469633b\n80f8af0d\n57f95c64\n"  # proj/tests/golden/gen_gp32_seed42_count4.hex


def run(*args, timeout=300):
    r = subprocess.run([XGEN, *args], capture_output=True, timeout=timeout)
    return r.returncode, r.stdout


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def test_binary_built():
    assert os.access(XGEN, os.X_OK)


@pytest.mark.parametrize("args,code", [
    (("gen", "-g", "nosuchgen", "--count", "4"), 64),          # test_cli.cpp:95
    (("params", "nosuchgen"), 64),                              # :96
    (("gen", "-g", "xorgensgp32", "--count", "64", "--lanes", "64"), 65),  # :97
    # lanes 0 with blocks > 1: BlockEnsemble throws out_of_range (parallel.cpp:90-91)
    (("gen", "-g", "xorgensgp32", "--count", "64", "--blocks", "2", "--lanes", "0"), 65),
    (("gen", "-g", "xorgensgp32", "--count", "7", "--blocks", "2"), 67),   # :98
    (("gen", "-g", "xorgens-raw", "--count", "4", "--blocks", "2"), 67),   # :99 (non-Weyl id)
    (("gen", "-g", "xorgensgp32", "--count", "4", "--format", "bogus"), 67),  # :100
    (("gen", "-g", "xorgensgp32"), 67),                         # --count is required
    (("frobnicate",), 67),
])
def test_exit_codes(args, code):
    assert run(*args)[0] == code


def test_params_table():
    # proj/tests/test_cli.cpp:104-115
    rc, out = run("params", "xorgensgp32")
    assert rc == 0
    for line in ("r,s:          128,65", "a,b,c,d:      15,14,12,17", "word bits:    32",
                 "gamma:        16", "omega:        2654435769", "lane bound:   63",
                 "state words:  129", "~2^4128"):
        assert line.encode() in out, line
    rc, out = run("params", "xorgens-raw")
    assert rc == 0 and b"2^4096-1" in out and b"gamma" not in out


gpu = pytest.mark.gpu


@gpu
def test_gen_golden_stream():
    # proj/tests/test_cli.cpp:59-63
    rc, out = run("gen", "--generator", "xorgensgp32", "--seed", "42", "--count", "4",
                  "--format", "hex")
    assert rc == 0 and out.decode() == GOLDEN_SEED42


@gpu
def test_gen_block_major_and_lanes():
    # proj/tests/test_cli.cpp:79-92
    _, combined = run("gen", "-g", "xorgensgp32", "--seed", "42", "--count", "8", "--blocks", "2",
                      "--format", "u32-lines")
    _, first = run("gen", "-g", "xorgensgp32", "--seed", "42", "--count", "4", "--format", "u32-lines")
    _, second = run("gen", "-g", "xorgensgp32", "--seed", "43", "--count", "4", "--format", "u32-lines")
    assert combined == first + second
    _, serial = run("gen", "-g", "xorgensgp32", "--seed", "5", "--count", "256", "--format", "hex")
    rc, laned = run("gen", "-g", "xorgensgp32", "--seed", "5", "--count", "256", "--lanes", "63",
                    "--format", "hex")
    assert rc == 0 and laned == serial
    rc, empty = run("gen", "-g", "xorgensgp32", "--seed", "1", "--count", "0")
    assert rc == 0 and empty == b""


@gpu
def test_gen_raw_le_matches_oracle(oracle, golden, tmp_path):
    # raw-le bytes == little-endian uint32 buffer; 3 blocks, ragged size
    path = tmp_path / "out.bin"
    rc, _ = run("gen", "--seed", "2", "--count", str(3 * 1001), "--blocks", "3", "--format",
                "raw-le", "-o", str(path))
    assert rc == 0
    got = np.fromfile(path, dtype="<u4").reshape(3, 1001)
    assert np.array_equal(got, oracle.ensemble(2, 3).fill_u32(1001))
    rc, raw = run("gen", "-g", "xorgens-raw", "--seed", "42", "--count", "300", "--format", "hex")
    assert rc == 0 and raw.decode().split() == golden["raw_streams"]["42"]


@gpu
def test_gen_long_single_block_chunks(oracle, tmp_path):
    # longer than the 2^25-word staging buffer: produced in continuation chunks
    n = (1 << 26) + 777
    path = tmp_path / "long.bin"
    rc, _ = run("gen", "--seed", "9", "--count", str(n), "--format", "raw-le", "-o", str(path),
                timeout=600)
    assert rc == 0
    got = np.fromfile(path, dtype="<u4")
    assert got.size == n
    assert np.array_equal(got, oracle.stream(9, n))


@gpu
def test_bench_reports():
    rc, out = run("bench", "--count", "16777216", "--blocks", "4096", "--trials", "3")
    assert rc == 0 and b"RN/s" in out
    rc, out = run("bench", "--count", "16777216", "--blocks", "4096", "--trials", "3", "--json")
    assert rc == 0 and b'"mean"' in out


@gpu
@pytest.mark.parametrize("gid,ps,weyl", [
    ("tiny:r2w8", (2, 1, 1, 1, 5, 7, 8, 159, 4), True),
    ("tiny:r4w16", (4, 3, 1, 2, 5, 8, 16, 40503, 8), True),
    ("tiny-raw:r2w16", (2, 1, 1, 1, 6, 11, 16, 40503, 8), False),
])
def test_gen_tiny_generators(oracle, gid, ps, weyl, tmp_path):
    """Every xorgens registry id (proj/src/registry.cpp:27-42): w/4 hex digits,
    w/8 raw-le bytes per word, on the general-parameter kernels."""
    from oracle import Params

    o = oracle.ensemble(11, 1, Params(*ps))
    want = o.fill_words(500)[0] if weyl else o.fill_raw_u32(500)[0].astype(np.uint64)
    rc, out = run("gen", "-g", gid, "--seed", "11", "--count", "500", "--format", "hex")
    assert rc == 0
    lines = out.decode().split()
    assert all(len(x) == ps[6] // 4 for x in lines)
    assert [int(x, 16) for x in lines] == want.tolist()
    path = tmp_path / "t.bin"
    rc, _ = run("gen", "-g", gid, "--seed", "11", "--count", "500", "--format", "raw-le", "-o", str(path))
    assert rc == 0
    dt = {8: "<u1", 16: "<u2"}[ps[6]]
    assert np.array_equal(np.fromfile(path, dtype=dt).astype(np.uint64), want)


# ---- `xgen test` (proj/tools/xgen.cpp:132-191; exit-by-verdict goldens
# proj/tests/test_cli.cpp:117-176) -------------------------------------------

QUICK_CFG = """# the reference's BatteryConfig::quick (battery.cpp:11-20) as a config file
monobit.bits = 1000000
runs.bits = 1000000
matrix_rank.matrices = 1000
linear_complexity.block_length = 500
linear_complexity.blocks = 200
birthday.rounds = 8
"""


def test_test_exit_codes_before_device_work(tmp_path):
    """Argument / config / file errors exit as the reference's xgen does,
    before any device work (CPU)."""
    cfg = tmp_path / "q.cfg"
    cfg.write_text(QUICK_CFG)
    bad = tmp_path / "bad.cfg"
    bad.write_text("monobit.bits 12\n")
    unknown = tmp_path / "unknown.cfg"
    unknown.write_text("nosuch.key = 1\n")
    assert run("test", "-g", "nosuchgen")[0] == 64
    assert run("test", "--config", str(tmp_path / "missing.cfg"))[0] == 66
    assert run("test", "--config", str(bad))[0] == 67
    assert run("test", "--config", str(unknown))[0] == 67
    assert run("test", "--input", str(tmp_path / "missing.bin"), "--config", str(cfg))[0] == 66
    assert run("test", "--bogus-flag")[0] == 67


def _ref_report(words, quick=True):
    from oracle import Battery

    try:
        b = Battery()
    except FileNotFoundError as e:  # pragma: no cover
        pytest.skip(str(e))
    verdict, js = b.run(words, quick=quick, label="ref")
    import json

    return verdict, json.loads(js)


def _same_tests(mine, ref):
    assert mine["overall"] == ref["overall"]
    assert mine["num_tests"] == ref["num_tests"]
    for a, b in zip(mine["tests"], ref["tests"]):
        assert (a["name"], a["n"], a["statistic"], a["p"], a["verdict"]) == \
               (b["name"], b["n"], b["statistic"], b["p"], b["verdict"]), a["name"]


@gpu
def test_test_generator_report_equals_reference(oracle, tmp_path):
    """`xgen test -g xorgensgp32` (GPU battery) reports exactly what the
    reference's run_battery reports over the same stream; exit 0 on pass."""
    import json

    cfg = tmp_path / "q.cfg"
    cfg.write_text(QUICK_CFG)
    out = tmp_path / "rep.json"
    rc, _ = run("test", "-g", "xorgensgp32", "--seed", "3", "--config", str(cfg), "-o", str(out))
    mine = json.loads(out.read_text())
    words = oracle.stream(3, 200000)
    verdict, ref = _ref_report(words)
    _same_tests(mine, ref)
    assert mine["generator"] == "xorgensgp32" and mine["seed"] == 3
    assert rc == {"pass": 0, "suspect": 2, "fail": 3}.get(ref["overall"], 0)


@gpu
def test_test_raw_stream_report_equals_reference(golden, tmp_path):
    """`xgen test -g xorgens-raw` (RawXorgens, the Weyl-ablated stream):
    rank and linear complexity counted over stored raw words
    (xg_rank_words / xg_lc_words); the report equals the reference's
    run_battery over the same words.  (With 4096 bits of state the raw
    stream passes these sizes -- its bit stream's linear complexity bound,
    32 x 4096, sits at K/2 even for the largest blocks; the reference's own
    negative control is the 16-bit-state tiny-raw:r2w8, acceptance.cpp:253-265.)"""
    import json

    from oracle import Reference

    cfg = tmp_path / "q.cfg"
    cfg.write_text(QUICK_CFG)
    rc, out = run("test", "-g", "xorgens-raw", "--seed", "1", "--config", str(cfg))
    mine = json.loads(out)
    try:
        ref_words = Reference().raw_stream(1, 140000, _gp32())
    except FileNotFoundError as e:  # pragma: no cover
        pytest.skip(str(e))
    _, ref = _ref_report(ref_words.astype(np.uint32))
    _same_tests(mine, ref)
    assert mine["params"].endswith("(no Weyl stage)")
    assert rc == {"pass": 0, "suspect": 2, "fail": 3}.get(ref["overall"], 0)


def _gp32():
    from oracle import Params

    return Params(128, 65, 15, 14, 12, 17, 32, 2654435769, 16)


@gpu
def test_test_input_file_equals_reference(oracle, tmp_path):
    """`xgen test --input words.bin`: raw-le words consumed in the
    reference's order (FileWordSource); report equal to the reference's over
    the same words; a file too short for the configuration exits 66."""
    import json

    cfg = tmp_path / "q.cfg"
    cfg.write_text(QUICK_CFG)
    words = oracle.stream(77, 140000)
    path = tmp_path / "w.bin"
    words.astype("<u4").tofile(path)
    rc, out = run("test", "--input", str(path), "--config", str(cfg))
    mine = json.loads(out)
    _, ref = _ref_report(words)
    _same_tests(mine, ref)
    assert mine["generator"] == "file:" + str(path) and mine["seed"] == 0
    short = tmp_path / "s.bin"
    words[:50000].astype("<u4").tofile(short)
    assert run("test", "--input", str(short), "--config", str(cfg))[0] == 66


@gpu
def test_test_tiny_raw_negative_control_exits_3(tmp_path):
    """`xgen test -g tiny-raw:r2w8` (8-bit words, no Weyl stage): the
    reference's negative control fails the battery -- exit 3."""
    import json

    cfg = tmp_path / "nb.cfg"
    cfg.write_text(QUICK_CFG + "birthday.enabled = false\n")
    rc, out = run("test", "-g", "tiny-raw:r2w8", "--seed", "1", "--config", str(cfg))
    rep = json.loads(out)
    assert rc == 3 and rep["overall"] == "fail"
    assert rep["params"] == "(r,s,a,b,c,d)=(2,1,1,1,5,7) w=8 (no Weyl stage)"
    # default config: birthday's 32-bit draws cannot apply to 8-bit words -> 67
    assert run("test", "-g", "tiny:r2w8")[0] == 67

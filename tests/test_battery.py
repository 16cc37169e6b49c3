"""The reference's own statistical battery (proj/src/stattests/*, compiled
unmodified into oracle/_ref/libxgref_battery.so) as a consumer of the
stream: SURVEY.md section 8f rank 3.  GPU words are bit-identical to the
reference's, so the GPU reports must equal the CPU ones p-value for
p-value, and pass (PAPER.md:650-678 reports no TestU01 failures)."""
import os

import numpy as np
import pytest

from oracle import BATTERY_SO

pytestmark = pytest.mark.skipif(not os.path.exists(BATTERY_SO),
                                reason="reference battery not built (needs the reference tree)")


@pytest.fixture(scope="module")
def battery():
    from oracle import Battery

    return Battery()


def test_battery_discriminates(battery, oracle):
    # quick config (BatteryConfig::quick, proj/src/stattests/battery.cpp:11-20)
    assert battery.run(oracle.stream(1, 1 << 20), quick=True)[0] == "pass"
    assert battery.run(np.arange(1 << 20, dtype=np.uint32), quick=True)[0] == "fail"


@pytest.mark.gpu
def test_gpu_streams_pass_the_reference_battery(battery, oracle):
    import torch

    import paper_1108_0486_b200 as xg

    p = xg.xorgensgp32_params()
    # one stream (seed 1), 2^24 words = the default battery's appetite (~1.6e7 words)
    one = xg.BlockEnsemble(p, 1, 1, 63).fill_u32(1 << 24)
    torch.cuda.synchronize()
    v, report = battery.run(one.cpu().numpy(), quick=False, label="xorgensgp32")
    assert v == "pass", report
    assert report == battery.run(oracle.stream(1, 1 << 24), quick=False, label="xorgensgp32")[1]
    # block-major ensemble output (256 consecutive seeds x 2^16 words)
    ens = xg.BlockEnsemble(p, 1000, 256, 63).fill_u32(1 << 16)
    torch.cuda.synchronize()
    v, report = battery.run(ens.cpu().numpy(), quick=False, label="ensemble")
    assert v == "pass", report

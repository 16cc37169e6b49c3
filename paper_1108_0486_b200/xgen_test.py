"""`xgen test` on the GPU: the reference CLI's battery subcommand
(proj/tools/xgen.cpp:132-191) over the GPU battery (battery.py).

    python -m paper_1108_0486_b200.xgen_test [-g ID] [--seed S] [--config PATH]
                                             [--input PATH] [-o PATH]

(`lib/xgen test ...` execs this module.)  Same flags, same JSON report
layout as the reference's to_json (battery.cpp:114-130: keys sorted as
nlohmann::json sorts them, two-space indent) and the same exit codes: 0 pass
(or not applicable), 2 suspect, 3 fail, 64 unknown generator, 66 I/O (config
or input unreadable, input exhausted), 67 bad arguments / bad config.
Generators: every xorgens id of the reference registry (xorgensgp32,
xorgens-raw, tiny:r2w8 / r2w16 / r4w16 and their tiny-raw: forms -- the
8- and 16-bit sets read w bits per word, as BitSource does); --input reads
raw-le 32-bit words ("file:<path>", seed 0), copied to the device once.
"""
from __future__ import annotations

import json
import sys

import numpy as np

EXIT_OK, EXIT_SUSPECT, EXIT_FAIL = 0, 2, 3
EXIT_UNKNOWN_GENERATOR, EXIT_IO, EXIT_BAD_ARGS = 64, 66, 67

# the xorgens ids of the registry (proj/src/registry.cpp:27-42): (params factory, raw)
def _generators():
    from . import xorgens as x

    return {"xorgensgp32": (x.xorgensgp32_params, False), "xorgens-raw": (x.xorgensgp32_params, True),
            "tiny:r2w8": (x.tiny_r2w8_params, False), "tiny:r2w16": (x.tiny_r2w16_params, False),
            "tiny:r4w16": (x.tiny_r4w16_params, False), "tiny-raw:r2w8": (x.tiny_r2w8_params, True),
            "tiny-raw:r2w16": (x.tiny_r2w16_params, True), "tiny-raw:r4w16": (x.tiny_r4w16_params, True)}


def params_display(p, raw: bool) -> str:
    """proj/tools/xgen.cpp:116-129."""
    s = f"(r,s,a,b,c,d)=({p.r},{p.s},{p.a},{p.b},{p.c},{p.d}) w={p.w}"
    return s + (" (no Weyl stage)" if raw else f" gamma={p.gamma} omega={p.omega}")


def _err(msg: str, code: int) -> int:
    sys.stderr.write(f"xgen: {msg}\n")
    return code


def _parse(argv):
    a = {"generator": "xorgensgp32", "seed": 0, "config": "", "input": "", "output": ""}
    i = 0
    names = {"--generator": "generator", "-g": "generator", "--seed": "seed", "--config": "config",
             "--input": "input", "--output": "output", "-o": "output"}
    while i < len(argv):
        arg = argv[i]
        key, val = (arg.split("=", 1) + [None])[:2] if arg.startswith("--") and "=" in arg else (arg, None)
        if key not in names:
            raise ValueError(f"unknown option {arg}")
        if val is None:
            i += 1
            if i >= len(argv):
                raise ValueError(f"{key} needs a value")
            val = argv[i]
        a[names[key]] = val
        i += 1
    try:
        a["seed"] = int(a["seed"], 0) if isinstance(a["seed"], str) else a["seed"]
    except ValueError:
        raise ValueError("--seed must be an unsigned 64-bit integer") from None
    if not 0 <= a["seed"] < 2**64:
        raise ValueError("--seed must be an unsigned 64-bit integer")
    return a


def to_json(report: dict, generator: str, params: str) -> str:
    """battery.cpp:114-130 through nlohmann::json (std::map keys: sorted)."""
    j = {"generator": generator, "params": params, "seed": report["seed"],
         "num_tests": report["num_tests"], "overall": report["overall"],
         "tests": [{"name": t["name"], "n": t["n"], "statistic": t["statistic"], "p": t["p"],
                    "verdict": t["verdict"]} for t in report["tests"]]}
    return json.dumps(j, indent=2, sort_keys=True)


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    try:
        a = _parse(argv)
    except ValueError as e:
        return _err(str(e), EXIT_BAD_ARGS)
    from .battery import BatteryConfig, BatteryInputError, run_battery_gpu, run_battery_on_words

    cfg = BatteryConfig.defaults()
    if a["config"]:
        try:
            with open(a["config"]) as f:
                text = f.read()
        except OSError:
            return _err(f"cannot open battery config: {a['config']}", EXIT_IO)
        try:
            cfg = BatteryConfig.parse(text)
        except ValueError as e:
            return _err(f"bad battery config: {e}", EXIT_BAD_ARGS)
    try:
        if a["input"]:
            try:
                data = np.fromfile(a["input"], dtype="<u4")
            except OSError:
                return _err(f"cannot open input file: {a['input']}", EXIT_IO)
            import torch

            words = torch.from_numpy(data.view(np.int32)).cuda()
            report = run_battery_on_words(words, cfg, seed=0)
            gen_id, params = "file:" + a["input"], "32-bit little-endian words"
        else:
            gens = _generators()
            if a["generator"] not in gens:
                return _err(f"unknown generator: {a['generator']}", EXIT_UNKNOWN_GENERATOR)
            factory, raw = gens[a["generator"]]
            p = factory()
            report = run_battery_gpu(p, a["seed"], cfg, raw=raw)
            gen_id, params = a["generator"], params_display(p, raw)
    except BatteryInputError as e:
        return _err(str(e), EXIT_IO)
    except ValueError as e:
        return _err(str(e), EXIT_BAD_ARGS)
    text = to_json(report, gen_id, params) + "\n"
    if a["output"] and a["output"] != "-":
        try:
            with open(a["output"], "w") as f:
                f.write(text)
        except OSError:
            return _err(f"cannot open output file: {a['output']}", EXIT_IO)
    else:
        sys.stdout.write(text)
        sys.stdout.flush()
    return {"fail": EXIT_FAIL, "suspect": EXIT_SUSPECT}.get(report["overall"], EXIT_OK)


if __name__ == "__main__":
    sys.exit(main())

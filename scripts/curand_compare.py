#!/usr/bin/env python3
"""Context only (paper Table 1 on B200): device throughput of cuRAND's
XORWOW / MTGP32 / Philox / MT19937 generating 2^30 uint32 into HBM, next to
the xorgensGP fill of the same size, all timed the same way (CUDA events,
best/mean of K launches after warm-up, output > L2).  cuRAND is a library
call, not part of this framework; the numbers only place xorgensGP among the
generators the paper compared against.

usage: python scripts/curand_compare.py [--steps 50]
"""
import argparse
import ctypes
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RNG = {"xorwow": 101, "mrg32k3a": 121, "mtgp32": 141, "mt19937": 142, "philox4_32_10": 161}


def load_curand():
    cands = glob.glob("/usr/local/cuda/lib64/libcurand.so*")
    try:
        import nvidia.curand

        cands += glob.glob(os.path.join(os.path.dirname(nvidia.curand.__file__), "lib", "libcurand.so*"))
    except Exception:
        pass
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError:
            continue
    raise OSError("libcurand not found")


def time_fn(fn, stream, steps, warmup):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_1108_0486_b200 as xg

    n = 1 << 30
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    res = {}
    cr = load_curand()
    for name, rt in RNG.items():
        gen = ctypes.c_void_p()
        if cr.curandCreateGenerator(ctypes.byref(gen), rt) != 0:
            res[name] = "unavailable"
            continue
        cr.curandSetStream(gen, ctypes.c_void_p(stream.cuda_stream))
        cr.curandSetPseudoRandomGeneratorSeed(gen, ctypes.c_uint64(1))
        fn = lambda: cr.curandGenerate(gen, ctypes.c_void_p(out.data_ptr()), ctypes.c_size_t(n))  # noqa: E731
        ms = time_fn(fn, stream, args.steps, args.warmup)
        res[name] = {"RN/s_best": n / (min(ms) / 1e3), "RN/s_mean": n / (statistics.mean(ms) / 1e3),
                     "ms_mean": statistics.mean(ms)}
        cr.curandDestroyGenerator(gen)
    ens = xg.BlockEnsemble(xg.xorgensgp32_params(), 1, 1 << 14, 63)
    buf = out.view(torch.uint32).view(1 << 14, 1 << 16)
    ms = time_fn(lambda: ens.fill_u32(1 << 16, out=buf), stream, args.steps, args.warmup)
    res["xorgensgp32 (this repo)"] = {"RN/s_best": n / (min(ms) / 1e3),
                                      "RN/s_mean": n / (statistics.mean(ms) / 1e3),
                                      "ms_mean": statistics.mean(ms)}
    print(json.dumps({"n_words": n, "results": res}, indent=1))


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Generates tests/golden/ref_vectors.json from the REFERENCE ITSELF.

Every word below comes out of oracle/_ref/libxgref.so, i.e. the reference's
own proj/src/{params,xorgens,parallel}.cpp compiled unmodified (see
oracle/Makefile).  The float / uint64 / Monte Carlo entries apply the
conventions of DESIGN.md section 3 (numpy, exact) to reference words, since
the reference has no conversions of its own.

Run in the container that has /root/reference:  python tests/golden/make_golden.py
(``--full-size`` regenerates only tests/golden/full_size.json, the per-chunk
digests of the full-size configs 2-5: about a minute on 8 cores).
"""
from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Oracle, Params, Reference  # noqa: E402

M64 = (1 << 64) - 1


def hexs(a):
    return [f"{int(v):08x}" for v in a]


def stream_checksums(ref: Reference, p, seed: int, n: int):
    w = ref.stream(seed, n, p).astype(np.uint64)
    x = int(np.bitwise_xor.reduce(w)) & 0xFFFFFFFF
    s = int(np.sum(w * np.arange(1, n + 1, dtype=np.uint64), dtype=np.uint64))
    return x, s, int(w[-1])


def full_size(ref: Reference, gp32) -> dict:
    """Digests of the full-size workloads, base_seed 1, from the reference's
    own words (xgref_stream_digests), per chunk of 2^14 consecutive streams:
      u32: streams [0, 2^18) x 2^16 words -- config 4 (2^34 words) and, chunk by
           chunk, config 2 (chunk 0 = the 2^30-word fill; chunk r = rank r of
           the weak-scaled config 2 at N <= 16);
      f32 / f64: streams [0, 2^17) x 2^16 values (f64: 2^17 words) -- config 3
           per chunk (rank r of the weak-scaled fills at N <= 8);
      mc: streams [0, 2^17) x 2^15 samples -- exact hit counts for 2^32 samples
           (config 5's stream set), per chunk so any N in {1, 2, 4, 8} checks its
           slice.
    A chunk record is paper_1108_0486_b200.digest.chunk_record of the
    per-stream (xor, sum, wsum): xor / sum / wsum of the chunk's block-major
    concatenation and the sha256 of the per-stream records."""
    from paper_1108_0486_b200.digest import chunk_record

    C, per = 1 << 14, 1 << 16
    n_u32_chunks, n_conv_chunks = 16, 8
    piece = 256

    def work(first):
        conv = first < n_conv_chunks * C
        return first, ref.stream_digests(gp32, 1, first, piece, per, per if conv else 0,
                                         (per // 2) if conv else 0)

    res = {}
    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        for first, d in ex.map(work, range(0, n_u32_chunks * C, piece)):
            res[first] = d
    out = {"base_seed": 1, "chunk_streams": C, "params": "xorgensgp32",
           "source": "oracle/_ref/libxgref.so xgref_stream_digests (reference next_word)"}

    def cat(key, i, chunk):
        parts = [res[f][key] for f in range(chunk * C, (chunk + 1) * C, piece)]
        if key == "mc":
            return np.concatenate(parts)
        return tuple(np.concatenate([p[i] for p in parts]) for i in range(3))

    out["u32"] = {"per_stream": per, "chunks": [chunk_record(*cat("u32", 0, c), per)
                                                for c in range(n_u32_chunks)]}
    out["f32"] = {"per_stream": per, "chunks": [chunk_record(*cat("f32", 0, c), per)
                                                for c in range(n_conv_chunks)]}
    out["f64"] = {"per_stream": per, "u32_per_stream": 2 * per,
                  "chunks": [chunk_record(*cat("f64", 0, c), 2 * per) for c in range(n_conv_chunks)]}
    out["mc"] = {"samples_per_stream": per // 2,
                 "chunk_hits": [int(cat("mc", 0, c).sum()) for c in range(n_conv_chunks)]}
    # whole 2^34-word fill (config 4), block-major over all 2^18 streams
    from paper_1108_0486_b200.digest import slice_digest
    xs = np.concatenate([res[f]["u32"][0] for f in sorted(res)])
    ss = np.concatenate([res[f]["u32"][1] for f in sorted(res)])
    wss = np.concatenate([res[f]["u32"][2] for f in sorted(res)])
    gx, gs, gws = slice_digest(xs, ss, wss, per)
    out["u32"]["all"] = {"streams": len(xs), "xor": f"{gx:08x}", "sum": f"{gs:016x}",
                         "wsum": f"{gws:016x}"}
    out["mc"]["total_hits_2p32"] = int(sum(out["mc"]["chunk_hits"]))
    return out


def main() -> None:
    ref = Reference()
    if "--full-size" in sys.argv:
        fs = full_size(ref, Oracle().gp32())
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "full_size.json")
        with open(path, "w") as f:
            json.dump(fs, f, indent=1)
        print("wrote", path, fs["u32"]["chunks"][0], fs["mc"]["total_hits_2p32"])
        return
    o = Oracle()
    gp32 = o.gp32()
    out = {"generator": "xorgensgp32 (128,65,15,14,12,17) w=32",
           "source": "oracle/_ref/libxgref.so = reference proj/src/{params,xorgens,parallel}.cpp"}

    # 1. per-seed stream prefixes (incl. the reference KAT seeds 0 and 42)
    seeds = [0, 1, 2, 3, 42, 1000, 1001, 2**63, M64]
    out["streams"] = {str(s): hexs(ref.stream(s, 300, gp32)) for s in seeds}

    # 1b. the Weyl-ablated baseline (RawXorgens, registry id "xorgens-raw")
    out["raw_streams"] = {str(s): hexs(ref.raw_stream(s, 300, gp32)) for s in (0, 42, M64)}

    # 2. seeded state of seed 1 (logical buffer oldest first + weyl)
    buf, wy = ref.seeded_state(1, gp32)
    out["seeded_state_seed1"] = {"buffer": hexs(buf), "weyl": f"{wy:08x}"}

    # 3. other parameter sets the GPU path accepts (w=32, r=128, lane_bound>=32)
    alt = Params(128, 95, 17, 12, 13, 15, 32, 2654435769, 16)   # lane_bound 33 (test_params.cpp:65)
    alt2 = Params(128, 33, 11, 7, 9, 19, 32, 0x6A09E667 | 1, 11)
    out["alt_params"] = []
    for p in (alt, alt2):
        out["alt_params"].append({
            "params": [p.r, p.s, p.a, p.b, p.c, p.d, p.w, p.omega, p.gamma],
            "check": ref.check(p),
            "streams": {str(s): hexs(ref.stream(s, 600, p)) for s in (5, 6, 7)}})

    # 4. BlockEnsemble::generate, block-major, awkward sizes (test_parallel.cpp:145-153)
    gens = []
    for base, blocks, lanes, per in ((7, 3, 63, 1), (7, 3, 63, 17), (7, 3, 63, 1000), (M64, 2, 63, 64),
                                     (42, 8, 32, 600)):
        h = ref.ensemble(gp32, base, blocks, lanes)
        words, _, _ = ref.generate_words(h, blocks, per)
        words2, _, _ = ref.generate_words(h, blocks, per)  # continuation
        ref.destroy(h)
        gens.append({"base_seed": base, "blocks": blocks, "lanes": lanes, "per_block": per,
                     "first": [hexs(r) for r in words], "second": [hexs(r) for r in words2]})
    out["generate"] = gens

    # 5. from_raw streams
    rng = np.random.default_rng(2024)
    raw = rng.integers(0, 2**32, size=128, dtype=np.uint64)
    out["from_raw"] = {"buffer": hexs(raw), "weyl": "deadbeef",
                       "stream": hexs(ref.from_raw_stream(raw, 0xDEADBEEF, 400, gp32))}

    # 6. conversions on reference words
    w = ref.stream(42, 256, gp32).astype(np.uint64)
    f32 = ((w.astype(np.uint32) >> 8).astype(np.float32) * np.float32(2.0 ** -24))
    u64 = w[0::2] | (w[1::2] << np.uint64(32))
    f64 = (u64 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    xy = w.astype(np.uint32).view(np.int32).astype(np.int64).reshape(-1, 2)  # (w[2m], w[2m+1])
    x = xy[:, 0]
    y = xy[:, 1]
    hits = int(np.count_nonzero((x * x).astype(np.uint64) + (y * y).astype(np.uint64)
                                < np.uint64(1 << 62)))
    out["conversions_seed42"] = {"f32_bits": [f"{v:08x}" for v in f32.view(np.uint32)],
                                 "u64": [f"{int(v):016x}" for v in u64],
                                 "f64_bits": [f"{v:016x}" for v in f64.view(np.uint64)],
                                 "mc_hits_128_samples": hits}

    # 7. BASELINE config 1: seed 1, 10^8 words
    x1, s1, last1 = stream_checksums(ref, gp32, 1, 10**8)
    out["config1"] = {"seed": 1, "n": 10**8, "xor": f"{x1:08x}", "sum": f"{s1 % 2**64:016x}",
                      "last": f"{last1:08x}"}

    # 8. BASELINE config 2: base_seed 1, P = 2^14 streams x 2^16 words, block-major,
    #    xor and sum_pos word*(pos+1) mod 2^64 with pos = g*2^16 + k; per-stream xor.
    P, n = 1 << 14, 1 << 16

    def one(g):
        wg = ref.stream(1 + g, n, gp32).astype(np.uint64)
        pos = np.arange(g * n + 1, g * n + n + 1, dtype=np.uint64)
        return (int(np.bitwise_xor.reduce(wg)), int(np.sum(wg * pos, dtype=np.uint64)))

    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        res = list(ex.map(one, range(P)))
    gx = 0
    gs = 0
    for xv, sv in res:
        gx ^= xv
        gs = (gs + sv) % 2**64
    per_stream_xor = np.array([r[0] for r in res], dtype=np.uint32)
    out["config2"] = {"base_seed": 1, "streams": P, "per_stream": n, "xor": f"{gx:08x}",
                      "wsum": f"{gs:016x}",
                      "per_stream_xor_sha": __import__("hashlib").sha256(per_stream_xor.tobytes()).hexdigest(),
                      "per_stream_xor_first16": hexs(per_stream_xor[:16])}

    # 9. proj/tests/test_long_linearity.cpp:71-99: low-bit windows of 2^14 bits,
    #    linear complexity by the reference's berlekamp_massey.  Raw xorgens
    #    seed 1 over 2^30 words (first and last window), Weyl-combined seed 1
    #    over its first 2^14 words.
    from oracle import Battery
    bat = Battery()
    win = 1 << 14
    rf, rl = ref.low_bit_windows(1, 1 << 30, win, gp32, raw=True)
    wf, _ = ref.low_bit_windows(1, win, win, gp32, raw=False)
    import hashlib
    out["long_linearity"] = {"window": win, "raw_words": 1 << 30,
                             "raw_seed1_first": bat.berlekamp_massey(rf),
                             "raw_seed1_last": bat.berlekamp_massey(rl),
                             "weyl_seed1_first": bat.berlekamp_massey(wf),
                             "raw_seed1_last_bits_sha256": hashlib.sha256(rl.tobytes()).hexdigest(),
                             "raw_seed1_first_bits_sha256": hashlib.sha256(rf.tobytes()).hexdigest()}

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, "config1", out["config1"], "config2", out["config2"]["xor"],
          out["config2"]["wsum"])


if __name__ == "__main__":
    main()

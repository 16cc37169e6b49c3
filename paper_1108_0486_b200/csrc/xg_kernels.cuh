// xg_kernels.cuh -- sm_100a device code for the xorgensGP generation path:
// the seeding kernel (K1), shared helpers, and the WORD-PER-LANE fill kernel.
// The default fill kernel is the pair-lane kernel in xg_pairs.cuh; the one
// here runs the J = 2 parameter sets and output rows the pair stores cannot
// address (odd lengths / 4-byte aligned rows).
//
// Design: ONE WARP PER STREAM, the r = 128 word window in
// registers.  Lane l holds logical window words W[l], W[32+l], W[64+l],
// W[96+l] (oldest first), i.e. four registers R[0..3].  One warp step makes
// the next 32 words of the stream at once -- 32 <= lane_bound = min(s, r-s)
// = 63, so every operand is older than the step (the gather/commit argument of
// proj/src/parallel.cpp:8-42):
//
//   x_{i+l} = T(W[l], a, b) ^ T(W[(r-s)+l], c, d)          (xorgens.hpp:39-47)
//
// W[l] is the lane's own R[0].  W[(r-s)+l] ((r-s) = 32*J + delta) belongs to
// another lane: the fill reads it from a per-warp shared-memory ring that
// mirrors the window (one STS of the new block + one LDS per step); the seeding
// kernel takes it from lane (l+delta)&31's register J or J+1 with one select +
// one shuffle.  The new word replaces R[0] and the window rotates by renaming
// registers (4-step unroll), so there are no moves.  The Weyl term of lane l in
// step k is weyl + (32k + l + 1)*omega (closed form, parallel.cpp:33-39), and
// the output is ((w ^ (w >> gamma)) + x) mod 2^32 (xorgens.hpp:58-62).
//
// Each warp step emits one contiguous, 128-byte aligned line of the
// block-major output (out[g*per_stream + k], parallel.cpp:97-135), stored with
// one coalesced evict-first STG.32 per step.  (Round-1 placement experiments --
// IMAD.HI right shifts, SHF.L left shifts, bulk-copy stores -- were measured
// slower and removed; profiles/ab_r1/README_round1.md keeps the A/B table.)
#pragma once

#include <cstdint>

namespace xgk {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarpsPerBlock = 8;  // 256 threads: 8 streams per CTA
constexpr int kThreads = 32 * kWarpsPerBlock;
constexpr unsigned kR = 128;       // GPU path: r = 128 (four registers per lane)

// xorgensgp32 (proj/src/params.cpp:83): (r,s,a,b,c,d) = (128,65,15,14,12,17),
// w = 32, omega = 2654435769, gamma = 16.  Compile-time so every shift is an
// immediate (the paper bakes parameters in).
struct GP32 {
    static constexpr int J = 1;              // (r - s) / 32 = 63 / 32
    static constexpr unsigned delta = 31;    // (r - s) % 32
    static constexpr unsigned a = 15, b = 14, c = 12, d = 17, gamma = 16;
    static constexpr uint32_t omega = 2654435769u;
};

// Any other valid w = 32, r = 128 set with lane_bound >= 32: r - s is odd
// (gcd(128, s) = 1), so J is 1 or 2 and delta is in 1..31.
template <int J_>
struct RtParams {
    static constexpr int J = J_;
    unsigned delta, a, b, c, d, gamma;
    uint32_t omega;
};

// kRaw: the linear recurrence alone (RawXorgens::next = step_linear,
// proj/include/xg/baselines.hpp:60-71, registry id "xorgens-raw"): emits x_i
// and leaves the Weyl accumulator untouched.
// kWide: each word zero-extended to uint64 -- the element type of the
// reference's generate() result (proj/include/xg/parallel.hpp:46-47).
// kRank: fused GF(2) matrix-rank test (pair-lane kernel only): every 32
// consecutive words are a 32 x 32 matrix, rows = words (bits MSB first, as the
// reference's BitSource reads them), ranks binned {32, 31, <= 30}.
enum Mode : int { kU32 = 0, kF32 = 1, kF64 = 2, kMC = 3, kSkip = 4, kRaw = 5, kWide = 6, kRank = 7 };

// Per-warp loop invariants.
struct Lane {
    unsigned src;      // shuffle source lane for the s-tap (seeding kernel)
    bool gives_J;      // this lane provides register J (else J+1) to the s-tap shuffle
    // Shared-memory s-tap (fill kernel): the block produced at step T (mod 8)
    // lives in slot T of an 8-slot, 256-word ring, with slot 0 mirrored at
    // words 256..287 so a read never wraps.  At step T the window's block j
    // was produced at step T-4+j, so W[32J + delta + l] is ring word
    // A_T + delta + l with the compile-time A_T = 32(T-4+J) mod 256.
    uint32_t* ring_w;  // ring + lane (stores)
    uint32_t* ring_r;  // ring + delta + lane (s-tap loads)
    uint32_t* stage;   // f64 / MC: 2 x 128-word pair staging
};

// One warp step on the register window.  T is the step index mod 8; the
// register rotation uses T mod 4: logical block j of the window lives in
// R[(T + j) & 3].  xorshift_transform (proj/include/xg/xorgens.hpp:13-18)
// twice, then xor.  RING: s-tap from the shared-memory ring (fills), else by
// select + shuffle (seeding, where no ring is set up).
template <int T, bool RING, class P>
__device__ __forceinline__ uint32_t warp_step(uint32_t (&R)[4], const P& p, const Lane& ln) {
    constexpr int i0 = T & 3;
    constexpr int iJ = (T + P::J) & 3;
    constexpr int iJ1 = (T + P::J + 1) & 3;
    uint32_t y;
    if constexpr (RING) {
        constexpr int kA = (32 * (T - 4 + P::J)) & 255;
        y = ln.ring_r[kA];
    } else {
        const uint32_t give = ln.gives_J ? R[iJ] : R[iJ1];
        y = __shfl_sync(kFull, give, ln.src);
    }
    const uint32_t x = R[i0];
    const uint32_t t1 = x ^ (x << p.a);
    const uint32_t t2 = y ^ (y << p.c);
    const uint32_t v = t1 ^ (t1 >> p.b) ^ t2 ^ (t2 >> p.d);
    R[i0] = v;  // newest block; the old block 0 is no longer needed
    if constexpr (RING) {
        ln.ring_w[32 * (T & 7)] = v;
        if constexpr ((T & 7) == 0) ln.ring_w[256] = v;  // mirror of slot 0
        // Hazards: a slot is rewritten 8 steps after it was written and read
        // at most 3 steps after (WAR: always separated by a sync).  The s-tap
        // reads blocks produced 2 and 3 steps earlier when J = 1 (xorgensgp32),
        // 1 and 2 steps earlier when J = 2, so publishing every second step
        // (J = 1) or every step (J = 2) covers RAW.  compute-sanitizer
        // racecheck reports no hazards.
        if constexpr (P::J != 1 || (T & 1) == 1) __syncwarp();
    }
    return v;
}

// Output stage (xorgens.hpp:58-62): ((w ^ (w >> gamma)) + x) mod 2^32.
template <class P>
__device__ __forceinline__ uint32_t weyl_out(uint32_t w, uint32_t v, const P& p) {
    return (w ^ (w >> p.gamma)) + v;
}

// Uniform float: (u >> 8) * 2^-24, exact.  The
// conversion of a 24-bit integer is exact in every rounding mode; the _rd
// form compiles to I2F.U32.RM (XU pipe) instead of I2FP (ALU pipe), which is
// the busiest pipe of this kernel.  (Reading the half-word and the byte
// straight out of the register with I2F.U16 R.H1 + I2F.U8 R.B1 and one FFMA
// saves the shift but is 1 % slower: profiles/ab_r1/README_round1.md, r1za.)
__device__ __forceinline__ float u32_to_f32(uint32_t u) {
    return __uint2float_rd(u >> 8) * 0x1p-24f;
}

// Uniform double from raw (lo, hi): clearing the low 11 bits leaves a value
// (u64 >> 11) << 11 with at most 53 significant bits, so the u64 -> f64
// conversion is exact and so is the scaling by 2^-64.
__device__ __forceinline__ double raw_pair_to_f64(uint32_t lo, uint32_t hi) {
    const uint64_t u = (static_cast<uint64_t>(hi) << 32) | (lo & ~0x7ffu);
    return __ull2double_rz(u) * 0x1p-64;
}

// Monte Carlo predicate.  A sample is a pair of CONSECUTIVE words
// (w[2m], w[2m+1]) of the stream -- in the pair-lane
// kernel (xg_pairs.cuh) exactly the pair a lane holds.  Each word, read as a
// signed 32-bit integer, is a coordinate in [-2^31, 2^31); the sample hits
// the disc iff x^2 + y^2 < 2^62 (exact).  Returns 1 for a hit.  Per sample
// ptxas emits IMAD.WIDE + IMAD.HI (the high word of x^2 + y^2), one VIADD and
// a LEA.HI that accumulates the sign bit -- no shifts, no selects.  (Folding
// the -2^62 into IMAD.WIDE's 64-bit addend saves the VIADD -- 245 instead of
// 253 instructions per 512 words -- but an IMAD.WIDE with a register-pair
// addend co-issues worse: 1.707e12 against 1.784e12 RN/s, measured A/B in
// profiles/s2b_mc_ab.txt.)
__device__ __forceinline__ uint32_t mc_hit(uint32_t a, uint32_t b) {
    const int64_t x = static_cast<int32_t>(a), y = static_cast<int32_t>(b);
    // x^2 + y^2 <= 2^63 fits in uint64; hit iff its high word is < 2^30,
    // i.e. iff (high word - 2^30), in [-2^30, 2^30], has its sign bit set.
    const uint64_t q = static_cast<uint64_t>(x * x) + static_cast<uint64_t>(y * y);
    return (static_cast<uint32_t>(q >> 32) - 0x40000000u) >> 31;
}

// SplitMix64 draw k (1-based) from `seed` in closed form: the chain of
// proj/include/xg/mix.hpp:9-14 has state seed + k * 0x9e3779b97f4a7c15 at draw k.
__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ Lane make_lane(unsigned delta) {
    Lane ln;
    const unsigned lane = threadIdx.x & 31u;
    ln.src = (lane + delta) & 31u;
    ln.gives_J = lane >= delta;
    ln.ring_w = nullptr;
    ln.ring_r = nullptr;
    ln.stage = nullptr;
    return ln;
}

// K1: XorgensState(params, seed) for stream g (proj/src/xorgens.cpp:19-32):
// r SplitMix draws (lane-parallel, closed form), weyl = draw r+1, zero guard
// (warp vote), then 4r = 512 discarded outputs = 16 warp steps.  The discarded
// outputs do not feed back, so the warm-up runs the linear part only and
// advances the Weyl accumulator in closed form.
template <class P>
__global__ void __launch_bounds__(kThreads)
seed_kernel(P p, uint32_t* __restrict__ win, uint32_t* __restrict__ weyl,
            uint32_t nstreams, uint64_t seed0) {
    const unsigned lane = threadIdx.x & 31;
    const uint32_t g = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (g >= nstreams) return;
    const uint64_t seed = seed0 + g;  // base_seed + i, uint64 wrap (parallel.cpp:93-94)
    uint32_t R[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) R[j] = static_cast<uint32_t>(splitmix_draw(seed, 32u * j + lane + 1));
    const uint32_t w0 = static_cast<uint32_t>(splitmix_draw(seed, kR + 1));
    const bool any = __any_sync(kFull, (R[0] | R[1] | R[2] | R[3]) != 0u);
    if (!any && lane == 0) R[0] = 0x7f4a7c15u;  // 0x9e3779b97f4a7c15 & mask (xorgens.cpp:28-29)
    const Lane ln = make_lane(p.delta);
#pragma unroll 1
    for (int it = 0; it < 4; ++it) {  // 16 steps = 4r words
        warp_step<0, false>(R, p, ln);
        warp_step<1, false>(R, p, ln);
        warp_step<2, false>(R, p, ln);
        warp_step<3, false>(R, p, ln);
    }
    uint32_t* w = win + static_cast<size_t>(g) * kR;
#pragma unroll
    for (int j = 0; j < 4; ++j) w[32 * j + lane] = R[j];
    if (lane == 0) weyl[g] = w0 + 4u * kR * p.omega;
}

template <int MODE>
__device__ __forceinline__ void* advance(void* o, int n) {
    if constexpr (MODE == kF64) return static_cast<double*>(o) + n;
    else if constexpr (MODE == kWide) return static_cast<unsigned long long*>(o) + n;
    else if constexpr (MODE == kU32 || MODE == kF32 || MODE == kRaw) return static_cast<uint32_t*>(o) + n;
    else return o;
}

// Four warp steps (one full register rotation) = 128 words of the stream.
// PH is the body's parity: its steps are T = 4*PH .. 4*PH+3 (mod 8) of the
// shared-memory ring, and it selects the f64 / MC stage buffer.  Emits at
// cursor o (single-word modes: o[0], o[32], o[64], o[96]; pair modes: o[0],
// o[32]); the tail variant masks by `limit` (values of this body still wanted).
template <int MODE, bool TAIL, int PH, class P>
__device__ __forceinline__ void body4(uint32_t (&R)[4], const P& p, const Lane& ln, uint32_t& wl,
                                      uint32_t w_step, void* o, uint32_t& hits, unsigned limit) {
    constexpr bool kW = MODE != kRaw;  // Weyl output stage applied
    const uint32_t v0 = warp_step<4 * PH + 0, true>(R, p, ln);
    const uint32_t o0 = kW ? weyl_out(wl, v0, p) : v0;
    const uint32_t v1 = warp_step<4 * PH + 1, true>(R, p, ln);
    const uint32_t o1 = kW ? weyl_out(wl + w_step, v1, p) : v1;
    const uint32_t v2 = warp_step<4 * PH + 2, true>(R, p, ln);
    const uint32_t o2 = kW ? weyl_out(wl + 2u * w_step, v2, p) : v2;
    const uint32_t v3 = warp_step<4 * PH + 3, true>(R, p, ln);
    const uint32_t o3 = kW ? weyl_out(wl + 3u * w_step, v3, p) : v3;
    wl += 4u * w_step;
    const unsigned lane = threadIdx.x & 31u;
    if constexpr (MODE == kU32 || MODE == kF32 || MODE == kRaw) {
        uint32_t* u = static_cast<uint32_t*>(o);
        const uint32_t ov[4] = {o0, o1, o2, o3};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (!TAIL || lane + 32u * j < limit) {
                if constexpr (MODE == kU32 || MODE == kRaw) __stcs(u + 32 * j, ov[j]);
                else __stcs(reinterpret_cast<float*>(u) + 32 * j, u32_to_f32(ov[j]));
            }
        }
    } else if constexpr (MODE == kWide) {
        unsigned long long* u = static_cast<unsigned long long*>(o);
        const uint32_t ov[4] = {o0, o1, o2, o3};
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (!TAIL || lane + 32u * j < limit) __stcs(u + 32 * j, static_cast<unsigned long long>(ov[j]));
    } else if constexpr (MODE == kF64 || MODE == kMC) {
        // Pairs through shared memory: the 128 outputs of the body are staged
        // in order, then lane l reads words (2l, 2l+1) and (64+2l, 65+2l) with
        // one LDS.64 each -- value 32*pair + l in natural order, no shuffles.
        // Two stage buffers alternate between consecutive bodies (PH), so the
        // publishing __syncwarp of body k+1 also retires body k's reads.
        uint32_t* st = ln.stage + 128 * PH;
        st[lane] = o0;
        st[32 + lane] = o1;
        st[64 + lane] = o2;
        st[96 + lane] = o3;
        __syncwarp();
        const uint2 pa = reinterpret_cast<const uint2*>(st)[lane];
        const uint2 pb = reinterpret_cast<const uint2*>(st + 64)[lane];
        if constexpr (MODE == kF64) {
            if (!TAIL || lane < limit) __stcs(static_cast<double*>(o), raw_pair_to_f64(pa.x, pa.y));
            if (!TAIL || lane + 32u < limit) __stcs(static_cast<double*>(o) + 32, raw_pair_to_f64(pb.x, pb.y));
        } else {
            // limit (TAIL) = wanted 64-word blocks of this body (0 or 1): pairs 0..31
            if (!TAIL || limit > 0u) hits += mc_hit(pa.x, pa.y);
            if (!TAIL) hits += mc_hit(pb.x, pb.y);
        }
    }
}

// K2/K3/K4: fill / fused conversion / fused Monte Carlo / skip for streams
// [g_begin, g_begin + g_count) of the ensemble, `words` words per stream,
// continuing from (and saving back) each stream's state.
//   kU32/kF32: out is stream-major with `words` values per stream, out[0] is
//              stream g_begin's first value.
//   kF64:      `words` must be even; words/2 doubles per stream.
//   kMC:       `words` a multiple of 64; words/2 samples per stream; the hit
//              total is added to *hits_out.
template <class P, int MODE>
__global__ void __launch_bounds__(kThreads)
fill_kernel(P p, uint32_t* __restrict__ win, uint32_t* __restrict__ weyl, uint32_t g_begin,
            uint32_t g_count, uint64_t words, void* __restrict__ out,
            unsigned long long* __restrict__ hits_out, uint64_t ld, uint32_t rg) {
    const unsigned lane = threadIdx.x & 31;
    const uint32_t gl = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (gl >= g_count) return;
    const uint32_t g = g_begin + gl;
    constexpr bool kPairs = (MODE == kF64 || MODE == kMC);

    uint32_t* w = win + static_cast<size_t>(g) * kR;
    uint32_t R[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) R[j] = w[32 * j + lane];
    const uint32_t weyl0 = weyl[g];
    uint32_t wl = weyl0 + (lane + 1u) * p.omega;
    const uint32_t w_step = 32u * p.omega;
    Lane ln = make_lane(p.delta);
    __shared__ uint32_t ring[kWarpsPerBlock][256 + 32];
    ln.ring_w = ring[threadIdx.x >> 5] + lane;
    ln.ring_r = ring[threadIdx.x >> 5] + p.delta + lane;
    // the window's blocks 0..3 count as produced at steps -4..-1: slots 4..7
#pragma unroll
    for (int j = 0; j < 4; ++j) ln.ring_w[32 * (4 + j)] = R[j];
    __syncwarp();
    if constexpr (kPairs) {
        __shared__ __align__(16) uint32_t stage[kWarpsPerBlock][256];
        ln.stage = stage[threadIdx.x >> 5];
    }

    // Output cursor: single-word modes index words, pair modes index pairs.
    const uint64_t per_stream_vals = kPairs ? (words >> 1) : words;
    void* o = out;
    if constexpr (MODE == kU32 || MODE == kF32 || MODE == kF64 || MODE == kRaw || MODE == kWide) {
        // row gl: groups of rg contiguous rows, ld elements apart (pair_kernel)
        const uint64_t first = static_cast<uint64_t>(gl / rg) * ld +
                               static_cast<uint64_t>(gl % rg) * per_stream_vals + lane;
        if constexpr (MODE == kF64) o = static_cast<double*>(out) + first;
        else if constexpr (MODE == kWide) o = static_cast<unsigned long long*>(out) + first;
        else o = static_cast<uint32_t*>(out) + first;
    }
    constexpr int kValsPerBody = kPairs ? 64 : 128;
    uint32_t hits = 0;

    uint64_t iters = words >> 7;  // 4 steps = 128 words per body
    while (iters != 0) {
        const uint32_t n = static_cast<uint32_t>(iters < (1ull << 30) ? iters : (1ull << 30));
        iters -= n;
        uint32_t i = 0;
#pragma unroll 1
        for (; i + 2 <= n; i += 2) {
            body4<MODE, false, 0>(R, p, ln, wl, w_step, o, hits, 0);
            body4<MODE, false, 1>(R, p, ln, wl, w_step, advance<MODE>(o, kValsPerBody), hits, 0);
            o = advance<MODE>(o, 2 * kValsPerBody);
        }
        // a chunk of 2^30 bodies is even, so every chunk starts at parity 0
        if (i < n) {
            body4<MODE, false, 0>(R, p, ln, wl, w_step, o, hits, 0);
            o = advance<MODE>(o, kValsPerBody);
        }
    }

    const unsigned tail = static_cast<unsigned>(words & 127u);
    if (tail != 0) {
        // One more (full) 4-step body; only the first `tail` words are
        // emitted.  The state saved below ends exactly at word `words`.
        const uint32_t O[4] = {R[0], R[1], R[2], R[3]};
        const unsigned lim = MODE == kMC ? tail >> 6 : (kPairs ? tail >> 1 : tail);
        if ((words >> 7) & 1)
            body4<MODE, true, 1>(R, p, ln, wl, w_step, o, hits, lim);
        else
            body4<MODE, true, 0>(R, p, ln, wl, w_step, o, hits, lim);
        // New logical window = words [words-128, words): positions tail..tail+127
        // of the 256 words held in O (old window) followed by R (new block).
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const unsigned q = 32u * j + lane;
            if (q >= tail && q < tail + kR) w[q - tail] = (j < 4) ? O[j & 3] : R[j & 3];
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) w[32 * j + lane] = R[j];
    }
    if (MODE != kRaw && lane == 0) weyl[g] = weyl0 + static_cast<uint32_t>(words) * p.omega;

    if constexpr (MODE == kMC) {
        unsigned long long t = hits;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(kFull, t, s);
        if (lane == 0 && t != 0) atomicAdd(hits_out, t);
    }
}

}  // namespace xgk

// xg_generic.cuh -- the general-parameter GPU path: any GeneratorParams the
// reference accepts (w in {8, 16, 32, 64}, any r, s with 0 < s < r,
// gcd(r, s) = 1), including the sets the register-window kernels cannot take
// (lane_bound < 32, w != 32, r != 128: the tiny verification sets and the
// w = 64 set of PAPER.md:448-449).
//
// One warp per stream, the circular buffer of r w-bit words (as uint64) in
// shared memory, L = min(32, lane_bound) lanes per step -- batch_step's
// gather-then-commit (proj/src/parallel.cpp:8-42) with a __syncwarp between the
// gather and the commit, and the Weyl term of lane l = weyl + (l+1)*omega.
// Correctness-first: it exists so that no valid parameter set is rejected;
// the production set runs the register-window kernels of xg_kernels.cuh.
#pragma once

#include <cstdint>

namespace xgk {

struct GenParams {
    unsigned r, s, a, b, c, d, w, gamma, lanes;
    uint64_t omega, mask;
};

enum GenMode : int { kGenU32 = 0, kGenRawU32 = 1, kGenWide = 2, kGenSkip = 3 };

__device__ __forceinline__ uint64_t gen_xs(uint64_t x, unsigned l, unsigned r, uint64_t mask) {
    const uint64_t t = (x ^ (x << l)) & mask;  // xorgens.hpp:13-18
    return t ^ (t >> r);
}

// Advances the stream held in x[0..r) (circular, oldest at idx) by `words`
// words, emitting them through emit(k, value).  Returns nothing; idx and
// weyl are updated.  All lanes of the warp must call it.
template <bool RAW, class Emit>
__device__ __forceinline__ void gen_advance(const GenParams& p, uint64_t* x, unsigned& idx,
                                            uint64_t& weyl, uint64_t words, Emit emit) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned back_s = p.r - p.s;
    for (uint64_t done = 0; done < words;) {
        const unsigned n = static_cast<unsigned>(words - done < p.lanes ? words - done : p.lanes);
        const bool on = lane < n;
        unsigned pos_r = idx + lane;
        if (pos_r >= p.r) pos_r -= p.r;
        unsigned pos_s = pos_r + back_s;
        if (pos_s >= p.r) pos_s -= p.r;
        uint64_t fresh = 0;
        if (on) fresh = gen_xs(x[pos_r], p.a, p.b, p.mask) ^ gen_xs(x[pos_s], p.c, p.d, p.mask);
        __syncwarp();  // every gather reads the pre-batch buffer
        if (on) {
            x[pos_r] = fresh;
            const uint64_t wk = (weyl + (lane + 1) * p.omega) & p.mask;
            emit(done + lane, RAW ? fresh : (((wk ^ (wk >> p.gamma)) + fresh) & p.mask));
        }
        __syncwarp();
        idx += n;
        if (idx >= p.r) idx -= p.r;
        if (!RAW) weyl = (weyl + n * p.omega) & p.mask;
        done += n;
    }
}

// XorgensState(params, seed) (proj/src/xorgens.cpp:19-32) for stream g.
__global__ void gen_seed_kernel(GenParams p, uint64_t* __restrict__ win, uint64_t* __restrict__ weyl,
                                uint32_t nstreams, uint64_t seed0) {
    extern __shared__ uint64_t gsm[];
    const uint32_t g = blockIdx.x;
    if (g >= nstreams) return;
    const unsigned lane = threadIdx.x & 31u;
    const uint64_t seed = seed0 + g;
    uint64_t any = 0;
    for (unsigned j = lane; j < p.r; j += 32) {
        uint64_t z = seed + (j + 1ull) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        gsm[j] = (z ^ (z >> 31)) & p.mask;
        any |= gsm[j];
    }
    uint64_t z = seed + (p.r + 1ull) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    uint64_t wy = (z ^ (z >> 31)) & p.mask;
    const bool nonzero = __any_sync(0xffffffffu, any != 0);
    __syncwarp();
    if (!nonzero && lane == 0) gsm[0] = 0x9e3779b97f4a7c15ull & p.mask;
    __syncwarp();
    unsigned idx = 0;
    gen_advance<false>(p, gsm, idx, wy, 4ull * p.r, [](uint64_t, uint64_t) {});
    for (unsigned i = lane; i < p.r; i += 32) {
        unsigned q = idx + i;
        if (q >= p.r) q -= p.r;
        win[static_cast<size_t>(g) * p.r + i] = gsm[q];
    }
    if (lane == 0) weyl[g] = wy;
}

// Fill / skip for streams [g_begin, g_begin + g_count), continuing each.
template <int MODE>
__global__ void gen_fill_kernel(GenParams p, uint64_t* __restrict__ win, uint64_t* __restrict__ weyl,
                                uint32_t g_begin, uint32_t g_count, uint64_t words,
                                void* __restrict__ out) {
    extern __shared__ uint64_t gsm[];
    const uint32_t gl = blockIdx.x;
    if (gl >= g_count) return;
    const uint32_t g = g_begin + gl;
    const unsigned lane = threadIdx.x & 31u;
    uint64_t* w = win + static_cast<size_t>(g) * p.r;
    for (unsigned i = lane; i < p.r; i += 32) gsm[i] = w[i];
    __syncwarp();
    uint64_t wy = weyl[g];
    unsigned idx = 0;
    const uint64_t base = static_cast<uint64_t>(gl) * words;
    if constexpr (MODE == kGenU32) {
        uint32_t* o = static_cast<uint32_t*>(out) + base;
        gen_advance<false>(p, gsm, idx, wy, words,
                           [o](uint64_t k, uint64_t v) { o[k] = static_cast<uint32_t>(v); });
    } else if constexpr (MODE == kGenRawU32) {
        uint32_t* o = static_cast<uint32_t*>(out) + base;
        gen_advance<true>(p, gsm, idx, wy, words,
                          [o](uint64_t k, uint64_t v) { o[k] = static_cast<uint32_t>(v); });
    } else if constexpr (MODE == kGenWide) {
        uint64_t* o = static_cast<uint64_t*>(out) + base;
        gen_advance<false>(p, gsm, idx, wy, words, [o](uint64_t k, uint64_t v) { o[k] = v; });
    } else {
        gen_advance<false>(p, gsm, idx, wy, words, [](uint64_t, uint64_t) {});
    }
    for (unsigned i = lane; i < p.r; i += 32) {
        unsigned q = idx + i;
        if (q >= p.r) q -= p.r;
        w[i] = gsm[q];
    }
    if (lane == 0) weyl[g] = wy;
}

}  // namespace xgk

// xg_pairs.cuh -- the pair-lane generation kernel (sm_100a), default for
// every w = 32, r = 128 set with r - s < 64 (xorgensgp32 and the J = 1
// runtime sets).
//
// Layout.  The 128-word window is held as 64 word PAIRS: lane l owns pair l
// (words 2l, 2l+1: "A") and pair 32 + l (words 64 + 2l, 65 + 2l: "B").  One
// "double step" makes the next 64 words, lane l producing the pair
//
//   N.x = T(W[2l],   a, b) ^ T(W[2l + q],     c, d)      q = r - s
//   N.y = T(W[2l+1], a, b) ^ T(W[2l + q + 1], c, d)      (xorgens.hpp:39-47)
//
// Every operand predates the step iff 63 + q < 128, i.e. s >= 64 -- one more
// than the reference's lane bound min(s, r-s) = 63 needs, because the window
// is not an in-place circular buffer (proj/src/parallel.cpp:8-42 writes its
// results back into the slots it reads; here the new pair only replaces A
// after both operands are read).  For xorgensgp32 (q = 63):
//   W[2l + 63] = .y of pair l + 31: lane l-1's B.y, or lane 31's A.y for l = 0
//   W[2l + 64] = .x of pair l + 32: the lane's OWN B.x
// so a double step needs ONE shuffle (and the giver's register choice, done
// with IMADs on the FMA pipe) for 64 words, against one shared-memory load +
// store per 32 words in the word-per-lane kernel (xg_kernels.cuh).  N then becomes B and B becomes A by
// register renaming (2-step unroll), so there are no moves.
//
// Outputs.  A lane holds two consecutive words of the stream, so every store
// is one 64-bit (u32/f32 pairs, one f64) or 128-bit (zero-extended u64
// words) coalesced, evict-first store: one STG.64 writes 256 contiguous bytes
// per warp.  f64 = (u64 >> 11) * 2^-53 of the lane's own (lo, hi) pair, and
// the Monte Carlo sample is the lane's own pair -- no data movement between
// lanes for either.
#pragma once

#include <cstdint>
#include <type_traits>

#include "xg_kernels.cuh"

namespace xgk {

__device__ __forceinline__ uint32_t xs(uint32_t x, unsigned l, unsigned r) {
    const uint32_t t = x ^ (x << l);
    return t ^ (t >> r);
}

struct PairLane {
    unsigned m;         // q = 2m + 1
    unsigned src1, src2;  // shuffle sources of pair l+m (.y) and pair l+m+1 (.x)
    bool a1, a2;        // this lane gives A (else B) to shuffle 1 / 2
    uint32_t is31, not31;  // 1 / 0 on lane 31 (the GP32 giver of A.y), 0 / 1 elsewhere
};

__device__ __forceinline__ PairLane make_pair_lane(unsigned delta) {
    PairLane pl;
    const unsigned lane = threadIdx.x & 31u;
    pl.m = 16u + (delta - 1u) / 2u;  // q = 32 + delta (J = 1), delta odd
    pl.src1 = (lane + pl.m) & 31u;
    pl.src2 = (lane + pl.m + 1u) & 31u;
    // Giver lane L serves reader L - m (A) when L >= m, else reader L + 32 - m (B).
    pl.a1 = lane >= pl.m;
    pl.a2 = lane >= pl.m + 1u;
    pl.is31 = lane == 31u ? 1u : 0u;
    pl.not31 = 1u - pl.is31;
    return pl;
}

// One double step: the next 64 words from the window (A, B); returns the
// lane's new pair.
template <int GIVE, class P>
__device__ __forceinline__ uint2 double_step(const uint2 A, const uint2 B, const P& p,
                                             const PairLane& pl) {
    uint32_t ty, tx;
    if constexpr (std::is_same_v<P, GP32>) {
        const unsigned lane = threadIdx.x & 31u;
        // give = lane 31 ? A.y : B.y on the FMA pipe instead of a SEL on the
        // busier ALU pipe.  GIVE 0: B.y * (1 - is31) + A.y * is31 -- A.y * is31
        // does not depend on the previous step, so one IMAD sits on the
        // step-to-step chain (MC +3 %, one stream +16 %); GIVE 1:
        // B.y + is31 * (A.y - B.y) (IADD + IMAD, both on the chain), 2 % faster
        // for f32 (profiles/ab_r1/README_round1.md, r1w/r1z).
        uint32_t give;
        if constexpr (GIVE == 0)
            asm("{\n\t.reg .u32 t;\n\tmul.lo.u32 t, %1, %3;\n\tmad.lo.u32 %0, %2, %4, t;\n\t}"
                : "=r"(give) : "r"(A.y), "r"(B.y), "r"(pl.is31), "r"(pl.not31));
        else
            asm("{\n\t.reg .u32 d;\n\tsub.u32 d, %1, %2;\n\tmad.lo.u32 %0, d, %3, %2;\n\t}"
                : "=r"(give) : "r"(A.y), "r"(B.y), "r"(pl.is31));
        ty = __shfl_sync(kFull, give, (lane + 31u) & 31u);
        tx = B.x;
    } else {
        ty = __shfl_sync(kFull, pl.a1 ? A.y : B.y, pl.src1);
        tx = __shfl_sync(kFull, pl.a2 ? A.x : B.x, pl.src2);
    }
    uint2 n;
    n.x = xs(A.x, p.a, p.b) ^ xs(ty, p.c, p.d);
    n.y = xs(A.y, p.a, p.b) ^ xs(tx, p.c, p.d);
    return n;
}

template <class P>
__device__ __forceinline__ uint32_t weyl_mix(uint32_t w, uint32_t v, const P& p) {
    return (w ^ (w >> p.gamma)) + v;  // xorgens.hpp:58-62
}

// Ranks over GF(2) of the two 32 x 32 matrices of a double step (words
// 0..31 and 32..63; row i = word i).  The 64 words are first transposed so
// lane l holds row l of each matrix (four shuffles), then Gaussian
// elimination runs column by column from the MSB, both matrices at once: a
// ballot finds the rows with the column's bit set, the last of them is the
// pivot and is broadcast, and every row with the bit set -- the pivot too,
// which thereby becomes zero and drops out -- is reduced by it.  The rank is
// the number of columns with a pivot.  Same rank as the row-by-row
// elimination of proj/src/stattests/gf2.cpp:8-33.  (Getting the pivot value
// with redux.sync.max instead of ballot + bfind + shuffle is 6 % slower;
// profiles/ab_r1/README_round1.md, r1zm.)
__device__ __forceinline__ void rank_pair(uint2 v, unsigned& rank_a, unsigned& rank_b) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned half = lane >> 1;
    const bool odd = lane & 1u;
    const uint32_t ax = __shfl_sync(kFull, v.x, half), ay = __shfl_sync(kFull, v.y, half);
    const uint32_t bx = __shfl_sync(kFull, v.x, 16u + half), by = __shfl_sync(kFull, v.y, 16u + half);
    uint32_t ra = odd ? ay : ax;  // word l
    uint32_t rb = odd ? by : bx;  // word 32 + l
    unsigned za = 0, zb = 0;  // columns without a pivot
#pragma unroll 8
    for (int c = 31; c >= 0; --c) {
        // One column of both matrices: the bit tests feed the ballots and
        // predicate the row reductions (no selects); bfind picks the highest
        // lane with the bit set as pivot (~0 if none, counted as no pivot).
        asm("{\n\t"
            ".reg .pred pa, pb;\n\t"
            ".reg .u32 t, ma, mb, qa, qb, va, vb;\n\t"
            "and.b32 t, %0, %4;\n\t"
            "setp.ne.u32 pa, t, 0;\n\t"
            "and.b32 t, %1, %4;\n\t"
            "setp.ne.u32 pb, t, 0;\n\t"
            "vote.sync.ballot.b32 ma, pa, 0xffffffff;\n\t"
            "vote.sync.ballot.b32 mb, pb, 0xffffffff;\n\t"
            "bfind.u32 qa, ma;\n\t"
            "bfind.u32 qb, mb;\n\t"
            "shfl.sync.idx.b32 va, %0, qa, 0x1f, 0xffffffff;\n\t"
            "shfl.sync.idx.b32 vb, %1, qb, 0x1f, 0xffffffff;\n\t"
            "@pa xor.b32 %0, %0, va;\n\t"
            "@pb xor.b32 %1, %1, vb;\n\t"
            "shr.u32 t, qa, 31;\n\t"
            "add.u32 %2, %2, t;\n\t"
            "shr.u32 t, qb, 31;\n\t"
            "add.u32 %3, %3, t;\n\t"
            "}"
            : "+r"(ra), "+r"(rb), "+r"(za), "+r"(zb)
            : "r"(1u << c));
    }
    const unsigned na = 32u - za, nb = 32u - zb;
    rank_a = na;
    rank_b = nb;
}

// matrix_rank_test's counting loop over a word buffer (any source: file
// words, the Weyl-ablated stream, sets the fused kRank mode does not take):
// matrix k = words [32k, 32k + 32), row i = word i.  One warp per pair of
// matrices (grid-stride), rank_pair as in the fused mode; bins (rank 32, 31,
// <= 30) added to counts[0..2].
__global__ void __launch_bounds__(256)
rank_words_kernel(const uint32_t* __restrict__ words, uint64_t matrices,
                  unsigned long long* __restrict__ counts) {
    const unsigned lane = threadIdx.x & 31u;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    uint32_t full = 0, minus1 = 0, rest = 0;
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         2 * j < matrices; j += warps) {
        const bool second = 2 * j + 1 < matrices;
        const uint64_t w = 64 * j + 2 * lane;
        uint2 v;
        v.x = (lane < 16u || second) ? words[w] : 0u;
        v.y = (lane < 16u || second) ? words[w + 1] : 0u;
        unsigned ra, rb;
        rank_pair(v, ra, rb);
        full += ra == 32u;
        minus1 += ra == 31u;
        rest += ra < 31u;
        if (second) {
            full += rb == 32u;
            minus1 += rb == 31u;
            rest += rb < 31u;
        }
    }
    if (lane == 0) {
        if (full) atomicAdd(counts, static_cast<unsigned long long>(full));
        if (minus1) atomicAdd(counts + 1, static_cast<unsigned long long>(minus1));
        if (rest) atomicAdd(counts + 2, static_cast<unsigned long long>(rest));
    }
}

// Per-lane accumulators: MC hits, or the rank-test bins.
struct RankAcc {
    uint32_t full = 0, minus1 = 0, rest = 0;  // rank 32, 31, <= 30
};
template <int MODE>
using AccT = std::conditional_t<MODE == kRank, RankAcc, uint32_t>;

// Emit double step `j` (0 or 1) of a body (128 words).  o is the lane's output
// cursor at the body start; `limit` (TAIL only) = values of this body wanted.
template <int MODE, bool TAIL>
__device__ __forceinline__ void pair_emit(uint2 v, void* o, int j, unsigned limit,
                                          AccT<MODE>& hits) {
    const unsigned lane = threadIdx.x & 31u;
    if constexpr (MODE == kU32 || MODE == kRaw) {
        if (!TAIL || 64u * j + 2u * lane < limit) __stcs(static_cast<uint2*>(o) + 32 * j, v);
    } else if constexpr (MODE == kF32) {
        if (!TAIL || 64u * j + 2u * lane < limit)
            __stcs(static_cast<float2*>(o) + 32 * j, make_float2(u32_to_f32(v.x), u32_to_f32(v.y)));
    } else if constexpr (MODE == kWide) {
        if (!TAIL || 64u * j + 2u * lane < limit)
            __stcs(static_cast<ulonglong2*>(o) + 32 * j, make_ulonglong2(v.x, v.y));
    } else if constexpr (MODE == kF64) {
        if (!TAIL || 32u * j + lane < limit) __stcs(static_cast<double*>(o) + 32 * j, raw_pair_to_f64(v.x, v.y));
    } else if constexpr (MODE == kMC) {
        if (!TAIL || 32u * j + lane < limit) hits += mc_hit(v.x, v.y);
    } else if constexpr (MODE == kRank) {
        // this double step holds matrices 2j and 2j+1 of the body
        unsigned ra, rb;
        rank_pair(v, ra, rb);
        if (lane == 0u) {
            if (!TAIL || 2u * j < limit) {
                hits.full += ra == 32u;
                hits.minus1 += ra == 31u;
                hits.rest += ra < 31u;
            }
            if (!TAIL || 2u * j + 1u < limit) {
                hits.full += rb == 32u;
                hits.minus1 += rb == 31u;
                hits.rest += rb < 31u;
            }
        }
    }
}

template <int MODE>
__device__ __forceinline__ void* pair_advance(void* o) {  // one body
    if constexpr (MODE == kU32 || MODE == kRaw) return static_cast<uint2*>(o) + 64;
    else if constexpr (MODE == kF32) return static_cast<float2*>(o) + 64;
    else if constexpr (MODE == kWide) return static_cast<ulonglong2*>(o) + 64;
    else if constexpr (MODE == kF64) return static_cast<double*>(o) + 64;
    else return o;
}

// One body = two double steps = 128 words; (A, B) := (N0, N1).
template <int MODE, bool TAIL, class P>
__device__ __forceinline__ void pair_body(uint2& A, uint2& B, const P& p, const PairLane& pl,
                                          uint32_t& wl, uint32_t w64, void* o, AccT<MODE>& hits,
                                          unsigned limit) {
    constexpr bool kW = MODE != kRaw;
    constexpr int kGive = MODE == kF32 ? 1 : 0;
    const uint2 n0 = double_step<kGive>(A, B, p, pl);
    const uint2 n1 = double_step<kGive>(B, n0, p, pl);
    if constexpr (MODE != kSkip) {
        uint2 o0 = n0, o1 = n1;
        if constexpr (kW) {
            const uint32_t w1 = wl + w64;
            o0.x = weyl_mix(wl, n0.x, p);
            o0.y = weyl_mix(wl + p.omega, n0.y, p);
            o1.x = weyl_mix(w1, n1.x, p);
            o1.y = weyl_mix(w1 + p.omega, n1.y, p);
        }
        pair_emit<MODE, TAIL>(o0, o, 0, limit, hits);
        pair_emit<MODE, TAIL>(o1, o, 1, limit, hits);
    }
    wl += 2u * w64;
    A = n0;
    B = n1;
}

// Fill / conversion / Monte Carlo / skip for streams [g_begin, g_begin +
// g_count), `words` words per stream, continuing from and saving back each
// stream's state (same contract as fill_kernel in xg_kernels.cuh).
// Requirements checked by the host: u32/f32/raw rows 8-byte aligned (even
// `words`), u64 rows 16-byte aligned, f64 `words` even, MC `words` a
// multiple of 64, rank `words` a multiple of 32.
// CTAs of 1..32 warps (one stream each).  GP32 fits 32 registers (64 warps
// per SM) -- except the Monte Carlo mode, which is bound by its integer pipes
// at any occupancy and schedules better with the 52 registers ptxas takes when
// allowed 64 (32 warps per SM: +1.4 %, profiles/s2m_lib_ab.txt); the
// runtime-parameter sets (CTAs of <= 8 warps) keep their extra shift
// registers rather than spill.
template <class P, int MODE>
__global__ void __launch_bounds__(std::is_same_v<P, GP32> ? 1024 : 256,
                                  std::is_same_v<P, GP32> ? (MODE == kMC ? 1 : 2) : 5)
pair_kernel(P p, uint32_t* __restrict__ win, uint32_t* __restrict__ weyl, uint32_t g_begin,
            uint32_t g_count, uint64_t words, void* __restrict__ out,
            unsigned long long* __restrict__ hits_out, uint64_t ld, uint32_t rg) {
    const unsigned lane = threadIdx.x & 31u;
    // CTAs hold 1..8 streams (the host spreads small ensembles over the SMs)
    const uint32_t gl = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gl >= g_count) return;
    const uint32_t g = g_begin + gl;
    const PairLane pl = make_pair_lane(p.delta);

    uint32_t* w = win + static_cast<size_t>(g) * kR;
    uint2 A = reinterpret_cast<const uint2*>(w)[lane];
    uint2 B = reinterpret_cast<const uint2*>(w)[32 + lane];
    const uint32_t weyl0 = weyl[g];
    uint32_t wl = weyl0 + (2u * lane + 1u) * p.omega;  // Weyl term of word 2l (parallel.cpp:33-39)
    const uint32_t w64 = 64u * p.omega;

    // Row gl of the output: rows come in groups of rg contiguous rows, the
    // groups ld elements apart (rg = 1, ld = the row length: plain block-major
    // rows; jump-ahead segments of several streams: rg > 1).
    const uint64_t seg = MODE == kF64 ? (words >> 1) : words;  // output elements per row
    const uint64_t row0 = static_cast<uint64_t>(gl / rg) * ld + static_cast<uint64_t>(gl % rg) * seg;
    void* o = out;
    if constexpr (MODE == kU32 || MODE == kRaw || MODE == kF32)
        o = static_cast<uint32_t*>(out) + row0 + 2u * lane;
    else if constexpr (MODE == kWide)
        o = static_cast<unsigned long long*>(out) + row0 + 2u * lane;
    else if constexpr (MODE == kF64)
        o = static_cast<double*>(out) + row0 + lane;
    AccT<MODE> hits{};

    uint64_t left = words >> 7;  // bodies of 128 words
    while (left != 0) {
        const uint32_t n = static_cast<uint32_t>(left < (1ull << 30) ? left : (1ull << 30));
        left -= n;
        uint32_t i = 0;
#pragma unroll 1
        for (; i + 4 <= n; i += 4) {
            pair_body<MODE, false>(A, B, p, pl, wl, w64, o, hits, 0);
            pair_body<MODE, false>(A, B, p, pl, wl, w64, pair_advance<MODE>(o), hits, 0);
            o = pair_advance<MODE>(pair_advance<MODE>(o));
            pair_body<MODE, false>(A, B, p, pl, wl, w64, o, hits, 0);
            pair_body<MODE, false>(A, B, p, pl, wl, w64, pair_advance<MODE>(o), hits, 0);
            o = pair_advance<MODE>(pair_advance<MODE>(o));
        }
#pragma unroll 1
        for (; i < n; ++i) {
            pair_body<MODE, false>(A, B, p, pl, wl, w64, o, hits, 0);
            o = pair_advance<MODE>(o);
        }
    }

    const unsigned tail = static_cast<unsigned>(words & 127u);
    if (tail != 0) {
        // One more full body; only the first `tail` words are emitted and the
        // saved window ends exactly at word `words`: positions tail..tail+127
        // of (old window, new 128 words).
        const uint2 OA = A, OB = B;
        const unsigned lim = (MODE == kF64 || MODE == kMC) ? tail >> 1 : (MODE == kRank ? tail >> 5 : tail);
        pair_body<MODE, true>(A, B, p, pl, wl, w64, o, hits, lim);
        const uint32_t v[8] = {OA.x, OA.y, OB.x, OB.y, A.x, A.y, B.x, B.y};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const unsigned q = 64u * (k >> 1) + 2u * lane + (k & 1);
            if (q >= tail && q < tail + kR) w[q - tail] = v[k];
        }
    } else {
        reinterpret_cast<uint2*>(w)[lane] = A;
        reinterpret_cast<uint2*>(w)[32 + lane] = B;
    }
    if (MODE != kRaw && lane == 0) weyl[g] = weyl0 + static_cast<uint32_t>(words) * p.omega;

    if constexpr (MODE == kMC) {
        unsigned long long t = hits;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(kFull, t, s);
        if (lane == 0 && t != 0) atomicAdd(hits_out, t);
    } else if constexpr (MODE == kRank) {
        // lane 0 holds the counts; hits_out[0..2] = rank 32, 31, <= 30
        const uint32_t f = hits.full, m = hits.minus1, r = hits.rest;
        if (lane == 0) {
            if (f) atomicAdd(hits_out, static_cast<unsigned long long>(f));
            if (m) atomicAdd(hits_out + 1, static_cast<unsigned long long>(m));
            if (r) atomicAdd(hits_out + 2, static_cast<unsigned long long>(r));
        }
    }
}

}  // namespace xgk

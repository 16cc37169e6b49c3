// xg_chunks.cuh -- the chunk-lane kernel (sm_100a) for xorgensgp32 on large
// ensembles: u32 / f32 / f64 fills, the fused Monte Carlo mode and the
// generator core alone (skip).
//
// Layout.  LPS lanes share one stream (32 / LPS streams per warp).  With
// C = 64 / LPS, lane `sub` of a stream owns the window words
//
//   A[i] = W[C*sub + i],  B[i] = W[64 + C*sub + i]      i = 0 .. C-1
//
// (W oldest first).  One step makes the next 64 words, lane `sub` producing
// the C consecutive words n = C*sub + i:
//
//   N[i] = T(W[n], a, b) ^ T(W[n + 63], c, d)        (xorgens.hpp:39-47)
//
// W[n] is the lane's own A[i]; W[n + 63] = W[64 + C*sub + i - 1] is the lane's
// own B[i-1] for i >= 1, and for i = 0 the last B word of lane sub-1 (lane 0:
// the last A word of lane LPS-1) -- ONE shuffle per C words, against one per
// 2 words in the pair-lane kernel (xg_pairs.cuh), whose lanes each hold a
// pair.  Every operand predates the step (63 + 63 < 128, the lane-bound
// argument of proj/src/parallel.cpp:8-42), so N overwrites A in place and the
// roles rotate by renaming (2-step unroll).  The Weyl term of word n of step
// j is weyl + (64j + n + 1)*omega (parallel.cpp:33-39), the output
// ((w ^ (w >> 16)) + x) mod 2^32 (xorgens.hpp:58-62).  A Monte Carlo sample
// is the pair (out[2m], out[2m+1]) and an f64 value the pair (lo, hi) -- C is
// even, so neither crosses lanes.
//
// Stores.  A lane's C outputs are contiguous (4C bytes; 8 for LPS = 8 is one
// 32-byte sector), and the LPS lanes of a stream cover 256 contiguous bytes
// per step, so one warp store instruction (STG.E.ENL2.256, evict-first)
// writes 32 / LPS rows x 256 bytes: as coalesced as the pair-lane kernel's
// STG.64 (one row x 256 bytes) with a quarter of the store instructions.
#pragma once

#include <cstdint>

#include "xg_kernels.cuh"

namespace xgk {

template <int C>
__device__ __forceinline__ void chunk_step(uint32_t (&X)[C], const uint32_t (&Y)[C], uint32_t t0) {
    // X := the next C words (X held the oldest half, Y the newer one)
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const uint32_t y = i == 0 ? t0 : Y[i - 1];
        const uint32_t x = X[i];
        const uint32_t t1 = x ^ (x << GP32::a);
        const uint32_t t2 = y ^ (y << GP32::c);
        X[i] = t1 ^ (t1 >> GP32::b) ^ t2 ^ (t2 >> GP32::d);
    }
}

// 32 bytes, evict-first (st.global.cs.v8: STG.E.ENL2.256 on sm_100), only
// if `on` -- a predicated store, no branch around it
__device__ __forceinline__ void st_cs_v8(void* p, uint32_t on, uint32_t a0, uint32_t a1,
                                         uint32_t a2, uint32_t a3, uint32_t a4, uint32_t a5,
                                         uint32_t a6, uint32_t a7) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
                 "@q st.global.cs.v8.b32 [%0], {%2,%3,%4,%5,%6,%7,%8,%9};\n\t}"
                 ::"l"(p), "r"(on), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6),
                 "r"(a7)
                 : "memory");
}

__device__ __forceinline__ void st_cs_v4(void* p, uint32_t on, uint32_t a0, uint32_t a1,
                                         uint32_t a2, uint32_t a3) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
                 "@q st.global.cs.v4.b32 [%0], {%2,%3,%4,%5};\n\t}"
                 ::"l"(p), "r"(on), "r"(a0), "r"(a1), "r"(a2), "r"(a3)
                 : "memory");
}

// Store the lane's C output words (u32 / f32: C values; f64: C/2 values, two
// words each) at o, if `on`.
template <int MODE, int C>
__device__ __forceinline__ void chunk_store(void* o, uint32_t on, const uint32_t (&v)[C]) {
    if constexpr (MODE == kU32 || MODE == kF32) {
        uint32_t u[C];
#pragma unroll
        for (int i = 0; i < C; ++i) u[i] = MODE == kU32 ? v[i] : __float_as_uint(u32_to_f32(v[i]));
        if constexpr (C % 8 == 0) {
#pragma unroll
            for (int i = 0; i < C; i += 8)
                st_cs_v8(static_cast<uint32_t*>(o) + i, on, u[i], u[i + 1], u[i + 2], u[i + 3],
                         u[i + 4], u[i + 5], u[i + 6], u[i + 7]);
        } else {
            st_cs_v4(o, on, u[0], u[1], u[2], u[3]);
        }
    } else if constexpr (MODE == kF64) {
        uint32_t u[C];
#pragma unroll
        for (int i = 0; i < C; i += 2) {
            const double d = raw_pair_to_f64(v[i], v[i + 1]);
            u[i] = __double2loint(d);
            u[i + 1] = __double2hiint(d);
        }
        if constexpr (C % 8 == 0) {
#pragma unroll
            for (int i = 0; i < C; i += 8)
                st_cs_v8(static_cast<uint32_t*>(o) + i, on, u[i], u[i + 1], u[i + 2], u[i + 3],
                         u[i + 4], u[i + 5], u[i + 6], u[i + 7]);
        } else {
            st_cs_v4(o, on, u[0], u[1], u[2], u[3]);
        }
    }
}

// One step: the giver's boundary word by one shuffle inside the stream's
// lane group, the C new words into X, then the consumer (store / MC).
template <int MODE, int LPS, int C>
__device__ __forceinline__ void chunk_body(uint32_t (&X)[C], const uint32_t (&Y)[C], unsigned src,
                                           uint32_t last, uint32_t& wl, uint32_t& hits,
                                           void* o, uint32_t live) {
    // give = last lane of the group ? X[C-1] : Y[C-1] as Y + last * (X - Y)
    // on the FMA pipe (a SEL would take the busier ALU pipe)
    uint32_t give;
    asm("{\n\t.reg .u32 d;\n\tsub.u32 d, %1, %2;\n\tmad.lo.u32 %0, d, %3, %2;\n\t}"
        : "=r"(give) : "r"(X[C - 1]), "r"(Y[C - 1]), "r"(last));
    const uint32_t t0 = __shfl_sync(kFull, give, src, LPS);
    chunk_step<C>(X, Y, t0);
    if constexpr (MODE != kSkip) {
        uint32_t v[C];
#pragma unroll
        for (int i = 0; i < C; ++i) {
            const uint32_t w = wl + static_cast<uint32_t>(i) * GP32::omega;
            v[i] = (w ^ (w >> GP32::gamma)) + X[i];
        }
        if constexpr (MODE == kMC) {
#pragma unroll
            for (int i = 0; i < C; i += 2) hits += mc_hit(v[i], v[i + 1]);
        } else {
            chunk_store<MODE, C>(o, live, v);
        }
    }
    wl += 64u * GP32::omega;
}

// Fill / MC / skip for streams [g_begin, g_begin + g_count), `words` (a
// multiple of 64) words per stream, continuing from and saving back each
// stream's state (the contract of pair_kernel); u32/f32/f64 rows 32-byte
// aligned (checked by the host).  Every shuffle stays inside a lane group;
// groups past g_count run on a copy of the last stream's state and neither
// store, count nor write back (full-warp shuffles: a partial mask costs a
// convergence check per shuffle).
template <int MODE, int LPS>
__global__ void __launch_bounds__(256)
chunk_kernel(uint32_t* __restrict__ win, uint32_t* __restrict__ weyl, uint32_t g_begin,
             uint32_t g_count, uint64_t words, void* __restrict__ out,
             unsigned long long* __restrict__ hits_out) {
    static_assert(MODE == kU32 || MODE == kF32 || MODE == kF64 || MODE == kMC || MODE == kSkip,
                  "chunk-lane modes");
    static_assert(LPS == 4 || LPS == 8 || LPS == 16, "lanes per stream");
    constexpr int C = 64 / LPS;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned sub = lane & (LPS - 1u);
    const uint32_t gid = (blockIdx.x * blockDim.x + threadIdx.x) / LPS;
    if ((blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / LPS >= g_count) return;  // whole warp idle
    const bool live = gid < g_count;
    const uint32_t gl = live ? gid : g_count - 1u;
    const unsigned src = (sub + LPS - 1u) & (LPS - 1u);
    // loop invariants held in registers (opaque, so ptxas keeps them rather
    // than re-deriving them from %tid inside the loop)
    uint32_t last, on;
    asm volatile("mov.u32 %0, %1;" : "=r"(last) : "r"(sub == LPS - 1u ? 1u : 0u));
    asm volatile("mov.u32 %0, %1;" : "=r"(on) : "r"(live ? 1u : 0u));
    const uint32_t g = g_begin + gl;

    uint32_t* w = win + static_cast<size_t>(g) * kR;
    uint32_t A[C], B[C];
#pragma unroll
    for (int i = 0; i < C; i += 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(w + C * sub + i);
        const uint4 b = *reinterpret_cast<const uint4*>(w + 64 + C * sub + i);
        A[i] = a.x; A[i + 1] = a.y; A[i + 2] = a.z; A[i + 3] = a.w;
        B[i] = b.x; B[i + 1] = b.y; B[i + 2] = b.z; B[i + 3] = b.w;
    }
    const uint32_t weyl0 = weyl[g];
    uint32_t wl = weyl0 + (C * sub + 1u) * GP32::omega;  // Weyl term of word C*sub
    uint32_t hits = 0;
    // the lane's output cursor: word C*sub of the row (32-bit elements; an
    // f64 row of words/2 values has the same byte layout)
    uint32_t* o = static_cast<uint32_t*>(out) + static_cast<uint64_t>(gl) * words + C * sub;

    const uint64_t steps = words >> 6;
    for (uint64_t k = steps >> 1; k != 0; --k) {
        chunk_body<MODE, LPS, C>(A, B, src, last, wl, hits, o, on);
        chunk_body<MODE, LPS, C>(B, A, src, last, wl, hits, o + 64, on);
        o += 128;
    }
    const bool odd = steps & 1u;
    if (odd) chunk_body<MODE, LPS, C>(A, B, src, last, wl, hits, o, on);  // window = (B, A)

#pragma unroll
    for (int i = 0; i < C && live; i += 4) {
        const uint4 a = odd ? make_uint4(B[i], B[i + 1], B[i + 2], B[i + 3])
                            : make_uint4(A[i], A[i + 1], A[i + 2], A[i + 3]);
        const uint4 b = odd ? make_uint4(A[i], A[i + 1], A[i + 2], A[i + 3])
                            : make_uint4(B[i], B[i + 1], B[i + 2], B[i + 3]);
        *reinterpret_cast<uint4*>(w + C * sub + i) = a;
        *reinterpret_cast<uint4*>(w + 64 + C * sub + i) = b;
    }
    if (live && sub == 0) weyl[g] = weyl0 + static_cast<uint32_t>(words) * GP32::omega;

    if constexpr (MODE == kMC) {
        unsigned long long t = live ? hits : 0u;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(kFull, t, s);
        if (lane == 0 && t != 0) atomicAdd(hits_out, t);
    }
}

}  // namespace xgk

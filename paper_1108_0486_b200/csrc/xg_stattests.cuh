// xg_stattests.cuh -- GPU Berlekamp-Massey for the reference's linear
// complexity test (proj/src/stattests/tests.cpp:128-178, the per-block
// linear complexity of proj/src/stattests/gf2.cpp:62-110), sm_100a.
//
// One warp per K-bit block (K <= 1023).  The stream words are read as the
// reference's BitSource reads them: bit i of the stream is bit 31 - (i mod 32)
// of word i / 32 (MSB first, proj/include/xg/stream.hpp:99-106), and block b
// is stream bits [b K, b K + K).  The polynomials C (connection) and B
// (previous connection) and the sequence window are 1024-bit vectors spread
// over the warp: coefficient i lives in lane i / 32, bit i mod 32.  Iteration
// n shifts the window by one coefficient (a funnel across lanes), inserts
// s[n] at coefficient 0, and computes the discrepancy
//     d = parity(sum_i c_i s[n - i])
// as one POPC per lane, a ballot of the parities and one POPC.  On d = 1,
// C ^= B x^m (a shift by m bits across lanes: two shuffles and a funnel);
// L, m and the branch are warp-uniform, so the warp never diverges.  The
// result, L, is the block's linear complexity; the kernel histograms it
// (hist[L] += 1), and the host bins the histogram exactly as tests.cpp does.
#pragma once

#include <cstdint>

namespace xgk {

constexpr unsigned kLcMaxK = 1023;  // coefficients 0..L fit 32 lanes x 32 bits

// words: [streams][words_per_stream] uint32 stream words; blocks_per_stream
// blocks of K bits each from the start of every row.
__global__ void __launch_bounds__(256)
lc_kernel(const uint32_t* __restrict__ words, uint32_t streams, uint64_t words_per_stream,
          unsigned K, uint32_t blocks_per_stream, unsigned long long* __restrict__ hist) {
    const unsigned lane = threadIdx.x & 31u;
    const uint64_t wid = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (wid >= static_cast<uint64_t>(streams) * blocks_per_stream) return;
    const uint64_t g = wid / blocks_per_stream, b = wid % blocks_per_stream;

    // Lane k holds block bits [32k, 32k + 32) MSB first (a funnel of two words).
    const uint64_t bit0 = b * K;
    const uint32_t* row = words + g * words_per_stream;
    const uint64_t w0 = (bit0 >> 5) + lane;
    const unsigned sh = static_cast<unsigned>(bit0 & 31u);
    const uint64_t last = (bit0 + K + 31) >> 5;  // one past the block's last word
    const uint32_t hi = w0 < last ? row[w0] : 0u;
    const uint32_t lo = (sh != 0u && w0 + 1 < last) ? row[w0 + 1] : 0u;
    const uint32_t chunk = sh ? __funnelshift_l(lo, hi, sh) : hi;

    uint32_t C = lane == 0u ? 1u : 0u;  // connection polynomial, c_0 = 1
    uint32_t B = C;                      // previous connection polynomial
    uint32_t W = 0u;                     // window: coefficient i <-> s[n - i]
    unsigned L = 0, m = 1;
    const unsigned up = (lane + 31u) & 31u;
#pragma unroll 1
    for (unsigned n = 0; n < K; ++n) {
        // shift the window by one coefficient and insert s[n] at coefficient 0
        const uint32_t carry = __shfl_sync(kFull, W, up) >> 31;
        const uint32_t sw = __shfl_sync(kFull, chunk, n >> 5);
        const uint32_t sn = (sw >> (31u - (n & 31u))) & 1u;
        W = (W << 1) | (lane == 0u ? sn : carry);
        // discrepancy
        const unsigned par = __popc(C & W) & 1u;
        const unsigned d = __popc(__ballot_sync(kFull, par != 0u)) & 1u;
        if (d) {
            // Bs = B x^m: coefficient i of Bs = coefficient i - m of B
            const unsigned ws = m >> 5, bs = m & 31u;
            const uint32_t x1 = __shfl_sync(kFull, B, (lane - ws) & 31u);
            const uint32_t x2 = __shfl_sync(kFull, B, (lane - ws - 1u) & 31u);
            const uint32_t v1 = lane >= ws ? x1 : 0u;
            const uint32_t v2 = lane >= ws + 1u ? x2 : 0u;
            const uint32_t Bs = m >= 1024u ? 0u : __funnelshift_l(v2, v1, bs);
            if (2u * L <= n) {
                B = C;
                C ^= Bs;
                L = n + 1u - L;
                m = 1;
            } else {
                C ^= Bs;
                ++m;
            }
        } else {
            ++m;
        }
    }
    if (lane == 0) atomicAdd(hist + L, 1ull);
}

}  // namespace xgk

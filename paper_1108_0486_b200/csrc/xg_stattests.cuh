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
    // 32 bits of the sequence per outer step: one broadcast of the chunk
    // holding s[32j .. 32j + 31], then one iteration per bit.
#pragma unroll 1
    for (unsigned j = 0; 32u * j < K; ++j) {
        const uint32_t cur = __shfl_sync(kFull, chunk, j);
        const unsigned nend = K - 32u * j < 32u ? K - 32u * j : 32u;
#pragma unroll 4
        for (unsigned t = 0; t < nend; ++t) {
            const unsigned n = 32u * j + t;
            // shift the window by one coefficient and insert s[n] at coefficient 0
            const uint32_t carry = __shfl_sync(kFull, W, up) >> 31;
            const uint32_t sn = (cur >> (31u - t)) & 1u;
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
    }
    if (lane == 0) atomicAdd(hist + L, 1ull);
}

}  // namespace xgk

// ---- monobit / runs / birthday spacings (tests.cpp:33-79, 175-212) --------
#include <cub/block/block_radix_sort.cuh>

namespace xgk {

// Ones and adjacent-bit transitions among the first `nbits` bits of `words`
// read MSB first: out[0] += ones, out[1] += transitions (runs = 1 +
// transitions) -- the counting loops of monobit and runs_test
// (proj/src/stattests/tests.cpp:33-79).  Grid-stride over words.
__global__ void __launch_bounds__(256)
ones_runs_kernel(const uint32_t* __restrict__ words, uint64_t nbits,
                 unsigned long long* __restrict__ out) {
    const uint64_t nwords = (nbits + 31) >> 5;
    unsigned long long ones = 0, trans = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nwords;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t w = words[i];
        const uint64_t rem = nbits - 32 * i;
        const unsigned valid = rem >= 32 ? 32u : static_cast<unsigned>(rem);  // 1..32
        const unsigned low = 32u - valid;                                      // 0..31
        ones += __popc(w & (~0u << low));
        // pair (bit k+1, bit k), k = low..30: both bits among the valid ones
        trans += __popc((w ^ (w >> 1)) & 0x7fffffffu & (~0u << low));
        if (valid == 32u && i + 1 < nwords) trans += (w ^ (words[i + 1] >> 31)) & 1u;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        ones += __shfl_xor_sync(kFull, ones, s);
        trans += __shfl_xor_sync(kFull, trans, s);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (ones) atomicAdd(out, ones);
        if (trans) atomicAdd(out + 1, trans);
    }
}

constexpr int kBdThreads = 256, kBdItems = 32;  // up to 8192 draws per round

// Birthday spacings, one CTA per round (tests.cpp:193-204): the round's
// n_draws words >> drop are sorted, their n - 1 spacings sorted, and equal
// neighbours counted; *dup += the count.  Sorting: cub::BlockRadixSort.
__global__ void __launch_bounds__(kBdThreads)
birthday_kernel(const uint32_t* __restrict__ words, uint32_t n, unsigned drop,
                unsigned long long* __restrict__ dup) {
    using Sort = cub::BlockRadixSort<uint32_t, kBdThreads, kBdItems>;
    // The sort's scratch and the sorted values are never live at once.
    __shared__ union {
        typename Sort::TempStorage tmp;
        uint32_t vals[kBdThreads * kBdItems];
    } sm;
    auto& tmp = sm.tmp;
    uint32_t* vals = sm.vals;
    const uint32_t* base = words + static_cast<uint64_t>(blockIdx.x) * n;
    uint32_t k[kBdItems];
#pragma unroll
    for (int j = 0; j < kBdItems; ++j) {
        const uint32_t idx = threadIdx.x * kBdItems + j;  // blocked arrangement
        k[j] = idx < n ? (base[idx] >> drop) : 0xffffffffu;
    }
    Sort(tmp).Sort(k);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kBdItems; ++j) vals[threadIdx.x * kBdItems + j] = k[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kBdItems; ++j) {
        const uint32_t idx = threadIdx.x * kBdItems + j;
        k[j] = idx + 1 < n ? vals[idx + 1] - vals[idx] : 0xffffffffu;
    }
    __syncthreads();
    Sort(tmp).Sort(k);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kBdItems; ++j) vals[threadIdx.x * kBdItems + j] = k[j];
    __syncthreads();
    unsigned c = 0;
#pragma unroll
    for (int j = 0; j < kBdItems; ++j) {
        const uint32_t idx = threadIdx.x * kBdItems + j;
        if (idx >= 1 && idx + 1 < n) c += vals[idx] == vals[idx - 1];
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(kFull, c, s);
    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(dup, static_cast<unsigned long long>(c));
}

}  // namespace xgk

// ---- w-bit words -> the 32-bit MSB-first bit stream -------------------------
namespace xgk {

// The statistical tests read a WordSource through BitSource: w bits per word,
// MSB first (proj/include/xg/stream.hpp:95-110).  For w < 32 the counting
// kernels take the same bit stream packed into 32-bit words: output word j =
// input words [j * 32/w, (j+1) * 32/w) concatenated, the first in the top
// bits (zero past the end).  left_align: each word shifted to the top of its
// 32 bits instead (birthday spacings reads the top t bits of every w-bit
// word).  Grid-stride.
__global__ void __launch_bounds__(256)
pack_words_kernel(const uint32_t* __restrict__ in, uint64_t n, unsigned w, int left_align,
                  uint32_t* __restrict__ out, uint64_t nout) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint32_t mask = w >= 32 ? ~0u : ((1u << w) - 1u);
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < nout; j += stride) {
        if (left_align) {
            out[j] = w >= 32 ? in[j] : (in[j] & mask) << (32u - w);
            continue;
        }
        const unsigned per = 32u / w;
        uint32_t v = 0;
        for (unsigned k = 0; k < per; ++k) {
            const uint64_t idx = j * per + k;
            const uint32_t x = idx < n ? (in[idx] & mask) : 0u;
            v = w >= 32 ? x : ((v << w) | x);
        }
        out[j] = v;
    }
}

}  // namespace xgk

// ---- Berlekamp-Massey for long sequences (up to 2^18 bits) ----------------
namespace xgk {

constexpr uint64_t kBmMaxBits = 1ull << 18;

// Words needed per polynomial / reversed-sequence buffer for n bits.
__host__ __device__ constexpr uint32_t bm_words(uint64_t nbits) {
    return static_cast<uint32_t>((nbits + 31) / 32 + 2);
}

// One warp per sequence, the reference's formulation (gf2.cpp:62-110) in
// shared memory: the sequence reversed into `rev` (bit j of the buffer =
// s[n_bits - 1 - j]) so the taps of step n are the contiguous slice starting
// at n_bits - 1 - n; C, B and a scratch polynomial rotate between three
// buffers that always hold exact polynomials.  Lane l works on words l,
// l + 32, ...; the discrepancy is one ballot of the lanes' partial parities.
// Bits are read MSB first (bit i of the data = bit 31 - i % 32 of word
// i / 32, as BitSource reads words).  Sequence q = data bits
// [bit0(q), bit0(q) + nbits) with bit0(q) = (q / per_row) * row_bits +
// (q % per_row) * stride_bits.  Its linear complexity goes to L_out[q]
// and/or hist[L].
__global__ void __launch_bounds__(32)
bm_long_kernel(const uint32_t* __restrict__ data, uint64_t data_words, uint64_t nbits,
               uint64_t stride_bits, uint32_t per_row, uint64_t row_bits,
               unsigned long long* __restrict__ hist, uint32_t* __restrict__ L_out) {
    extern __shared__ uint32_t bm_smem[];
    const unsigned lane = threadIdx.x;
    const uint32_t nw = bm_words(nbits);
    uint32_t* rev = bm_smem;
    uint32_t* P0 = rev + nw;
    uint32_t* P1 = P0 + nw;
    uint32_t* P2 = P1 + nw;
    const uint64_t q = blockIdx.x;
    const uint64_t bit0 = (q / per_row) * row_bits + (q % per_row) * stride_bits;
    // 32 data bits from sequence bit 32t on (MSB first); 0 outside the sequence
    auto sword = [&](int64_t t) -> uint32_t {
        if (t < 0 || 32 * t >= static_cast<int64_t>(nbits)) return 0u;
        const uint64_t g = bit0 + 32 * static_cast<uint64_t>(t);
        const uint64_t w = g >> 5;
        const unsigned sh = static_cast<unsigned>(g & 31u);
        const uint32_t hi = w < data_words ? data[w] : 0u;
        const uint32_t lo = (sh && w + 1 < data_words) ? data[w + 1] : 0u;
        uint32_t v = sh ? __funnelshift_l(lo, hi, sh) : hi;
        const int64_t valid = static_cast<int64_t>(nbits) - 32 * t;
        if (valid < 32) v &= ~0u << (32 - valid);
        return v;
    };
    // rev word k = the 32 sequence bits ending at e = nbits - 1 - 32k, bit b = s[e - b]
    for (uint32_t k = lane; k < nw; k += 32) {
        const int64_t e = static_cast<int64_t>(nbits) - 1 - 32 * static_cast<int64_t>(k);
        uint32_t v = 0;
        if (e >= 0) {
            const int64_t st = e - 31;  // first bit of the window (may be negative)
            const int64_t t0 = st >= 0 ? st / 32 : -((31 - st) / 32);
            const unsigned sh = static_cast<unsigned>(st - 32 * t0);
            const uint32_t a = sword(t0), b2 = sword(t0 + 1);
            v = sh ? __funnelshift_l(b2, a, sh) : a;
        }
        rev[k] = v;
        P0[k] = k == 0 ? 1u : 0u;  // C = 1
        P1[k] = k == 0 ? 1u : 0u;  // B = 1
        P2[k] = 0u;
    }
    __syncwarp();
    uint32_t* C = P0;
    uint32_t* B = P1;
    uint32_t* T = P2;
    uint64_t L = 0, m = 1;
    for (uint64_t n = 0; n < nbits; ++n) {
        const uint64_t off = nbits - 1 - n;
        const uint32_t ow = static_cast<uint32_t>(off >> 5), ob = static_cast<uint32_t>(off & 31u);
        const uint64_t taps = L + 1;
        const uint32_t tw = static_cast<uint32_t>((taps + 31) / 32);
        unsigned par = 0;
        for (uint32_t k = lane; k < tw; k += 32) {
            uint32_t chunk = rev[ow + k] >> ob;
            if (ob) chunk |= rev[ow + k + 1] << (32u - ob);
            const uint64_t rem = taps - 32ull * k;
            if (rem < 32) chunk &= (1u << rem) - 1u;
            par ^= __popc(C[k] & chunk);
        }
        const unsigned d = __popc(__ballot_sync(kFull, (par & 1u) != 0u)) & 1u;
        if (d) {
            // T = C ^ B x^m, every word (the buffers always hold exact
            // polynomials, zero above their degree: deg <= n + 1 < 32 nw)
            const uint32_t ws = static_cast<uint32_t>(m >> 5), bs = static_cast<uint32_t>(m & 31u);
            const uint32_t top = static_cast<uint32_t>(
                (n + 2) / 32 + 2 < nw ? (n + 2) / 32 + 2 : nw);  // words above are zero in C and B x^m
            for (uint32_t k = lane; k < nw; k += 32) {
                if (k >= top) {
                    T[k] = 0u;
                    continue;
                }
                uint32_t sh = 0;
                if (k >= ws) {
                    sh = B[k - ws] << bs;
                    if (bs && k >= ws + 1) sh |= B[k - ws - 1] >> (32u - bs);
                }
                T[k] = C[k] ^ sh;
            }
            __syncwarp();
            if (2 * L <= n) {
                uint32_t* oldB = B;
                B = C;
                C = T;
                T = oldB;
                L = n + 1 - L;
                m = 1;
            } else {
                uint32_t* oldC = C;
                C = T;
                T = oldC;
                ++m;
            }
            __syncwarp();
        } else {
            ++m;
        }
    }
    if (lane == 0) {
        if (L_out) L_out[blockIdx.x] = static_cast<uint32_t>(L);
        if (hist) atomicAdd(hist + L, 1ull);
    }
}

}  // namespace xgk

// xg_digest.cuh -- row digests of a device buffer of 32-bit elements (sm_100a).
//
// For each row r of a (rows x per_row) row-major buffer of u32 elements e_k:
//   xor = e_0 ^ e_1 ^ ...,  sum = sum_k e_k,  wsum = sum_k e_k * (k + 1)
// (sums mod 2^64).  The three numbers are the per-stream digests the
// full-size parity checks compare against goldens computed from the
// reference's own words (tests/golden/make_golden.py, xgref_stream_digests in
// oracle/ref_shim.cpp); rows compose into block-major slice digests on the
// host (paper_1108_0486_b200/digest.py).  A float row is digested through its
// bit patterns (f64 as its little-endian u32 halves).
//
// One CTA per row, HBM-read bound: 16-byte loads when the row allows them.
#pragma once

#include <cstdint>

namespace xgk {

constexpr int kDigestThreads = 256;

struct Dig {
    uint32_t x;
    unsigned long long s, ws;
};

__device__ __forceinline__ void dig_add(Dig& d, uint32_t v, uint64_t k1) {
    d.x ^= v;
    d.s += v;
    d.ws += static_cast<unsigned long long>(v) * k1;
}

__global__ void __launch_bounds__(kDigestThreads)
digest_kernel(const uint32_t* __restrict__ data, uint64_t per_row, uint32_t* __restrict__ out_x,
              unsigned long long* __restrict__ out_s, unsigned long long* __restrict__ out_ws) {
    const uint64_t row = blockIdx.x;
    const uint32_t* r = data + row * per_row;
    Dig d{0u, 0ull, 0ull};
    const unsigned t = threadIdx.x;
    if ((reinterpret_cast<uintptr_t>(r) & 15u) == 0 && (per_row & 3u) == 0) {
        const uint4* q = reinterpret_cast<const uint4*>(r);
        const uint64_t nq = per_row >> 2;
#pragma unroll 4
        for (uint64_t i = t; i < nq; i += kDigestThreads) {
            const uint4 v = __ldcs(q + i);
            const uint64_t k1 = 4 * i + 1;
            dig_add(d, v.x, k1);
            dig_add(d, v.y, k1 + 1);
            dig_add(d, v.z, k1 + 2);
            dig_add(d, v.w, k1 + 3);
        }
    } else {
        for (uint64_t i = t; i < per_row; i += kDigestThreads) dig_add(d, __ldcs(r + i), i + 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        d.x ^= __shfl_xor_sync(0xffffffffu, d.x, o);
        d.s += __shfl_xor_sync(0xffffffffu, d.s, o);
        d.ws += __shfl_xor_sync(0xffffffffu, d.ws, o);
    }
    __shared__ Dig part[kDigestThreads / 32];
    if ((t & 31u) == 0) part[t >> 5] = d;
    __syncthreads();
    if (t == 0) {
        Dig a = part[0];
#pragma unroll
        for (int w = 1; w < kDigestThreads / 32; ++w) {
            a.x ^= part[w].x;
            a.s += part[w].s;
            a.ws += part[w].ws;
        }
        out_x[row] = a.x;
        out_s[row] = a.s;
        out_ws[row] = a.ws;
    }
}

}  // namespace xgk

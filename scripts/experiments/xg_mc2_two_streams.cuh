// Experiment: fused MC with TWO streams per warp (interleaved double steps:
// ILP 2 inside every lane).  Streams 2w and 2w+1 of the launch; words a
// multiple of 128 (whole bodies), g_count even (host checks).
namespace xgk {
template <class P>
__global__ void __launch_bounds__(1024, 1)
pair_kernel_mc2(P p, uint32_t* __restrict__ win, uint32_t* __restrict__ weyl, uint32_t g_begin,
                uint32_t g_count, uint64_t words, unsigned long long* __restrict__ hits_out) {
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (2 * wg >= g_count) return;
    const uint32_t g0 = g_begin + 2 * wg, g1 = g0 + 1;
    const PairLane pl = make_pair_lane(p.delta);
    uint32_t* w0 = win + static_cast<size_t>(g0) * kR;
    uint32_t* w1 = win + static_cast<size_t>(g1) * kR;
    uint2 A0 = reinterpret_cast<const uint2*>(w0)[lane], B0 = reinterpret_cast<const uint2*>(w0)[32 + lane];
    uint2 A1 = reinterpret_cast<const uint2*>(w1)[lane], B1 = reinterpret_cast<const uint2*>(w1)[32 + lane];
    const uint32_t y0 = weyl[g0], y1 = weyl[g1];
    uint32_t wl0 = y0 + (2u * lane + 1u) * p.omega, wl1 = y1 + (2u * lane + 1u) * p.omega;
    const uint32_t w64 = 64u * p.omega;
    uint32_t hits = 0;
    uint64_t left = words >> 7;
    while (left != 0) {
        const uint32_t n = static_cast<uint32_t>(left < (1ull << 30) ? left : (1ull << 30));
        left -= n;
        uint32_t i = 0;
#pragma unroll 1
        for (; i + XG_MC2_U <= n; i += XG_MC2_U) {
#pragma unroll
            for (int u = 0; u < XG_MC2_U; ++u) {
                pair_body<kMC, false>(A0, B0, p, pl, wl0, w64, nullptr, hits, 0);
                pair_body<kMC, false>(A1, B1, p, pl, wl1, w64, nullptr, hits, 0);
            }
        }
#pragma unroll 1
        for (; i < n; ++i) {
            pair_body<kMC, false>(A0, B0, p, pl, wl0, w64, nullptr, hits, 0);
            pair_body<kMC, false>(A1, B1, p, pl, wl1, w64, nullptr, hits, 0);
        }
    }
    reinterpret_cast<uint2*>(w0)[lane] = A0; reinterpret_cast<uint2*>(w0)[32 + lane] = B0;
    reinterpret_cast<uint2*>(w1)[lane] = A1; reinterpret_cast<uint2*>(w1)[32 + lane] = B1;
    if (lane == 0) { weyl[g0] = y0 + static_cast<uint32_t>(words) * p.omega; weyl[g1] = y1 + static_cast<uint32_t>(words) * p.omega; }
    unsigned long long t = hits;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) t += __shfl_xor_sync(kFull, t, s);
    if (lane == 0 && t != 0) atomicAdd(hits_out, t);
}
}  // namespace xgk

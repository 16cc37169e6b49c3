// xg_probe.cu -- bench-only helper (libxg_probe.so, not part of the generator
// ABI): write-only HBM ceilings measured by bench.py on the fill's own output
// buffer in the same run, the denominator of "% of HBM write BW" (SURVEY.md
// section 8d).
//
//   xg_probe_memset       cudaMemsetAsync over the buffer (the driver's fill)
//   xg_probe_rows         the fill kernel's store shape without the generator:
//                         one warp per row of `row_bytes`, `vec` = 8 (STG.64,
//                         as pair_kernel stores u32 pairs), 16 (STG.128) or 32
//                         (STG.256)
//                         byte evict-first stores, `warps` rows per CTA and at
//                         most `cap` resident CTAs per SM (0 = no cap) -- the
//                         same occupancy trick as launch_pair (xg_gpu.cu).
//   xg_probe_gridstride   a grid-stride 16-byte store stream over SMs x 8 CTAs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace {

template <int VEC>
__global__ void __launch_bounds__(1024) row_store(char* __restrict__ dst, uint64_t row_bytes,
                                                  uint32_t rows, uint32_t v) {
    const uint32_t row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const unsigned lane = threadIdx.x & 31u;
    char* r = dst + static_cast<uint64_t>(row) * row_bytes;
    const uint64_t n = row_bytes / (32 * VEC);
    if constexpr (VEC == 8) {
        uint2* p = reinterpret_cast<uint2*>(r) + lane;
        const uint2 val = make_uint2(v, v ^ lane);
#pragma unroll 4
        for (uint64_t i = 0; i < n; ++i) __stcs(p + 32 * i, val);
    } else if constexpr (VEC == 16) {
        uint4* p = reinterpret_cast<uint4*>(r) + lane;
        const uint4 val = make_uint4(v, v ^ lane, v, v);
#pragma unroll 4
        for (uint64_t i = 0; i < n; ++i) __stcs(p + 32 * i, val);
    } else {  // 32-byte stores (STG.E.ENL2.256, sm_100)
        char* p = r + 32 * lane;
        const uint32_t a = v, b = v ^ lane;
#pragma unroll 4
        for (uint64_t i = 0; i < n; ++i)
            asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};"
                         :: "l"(p + 1024 * i), "r"(a), "r"(b) : "memory");
    }
}

__global__ void __launch_bounds__(256) grid_stride(uint4* __restrict__ dst, size_t n16, uint32_t v) {
    const uint4 val = make_uint4(v, v, v, v);
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
#pragma unroll 4
    for (; i < n16; i += stride) __stcs(dst + i, val);
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

}  // namespace

extern "C" {

int xg_probe_memset(void* dst, size_t bytes, void* stream) {
    return cudaMemsetAsync(dst, 0x5a, bytes, static_cast<cudaStream_t>(stream)) == cudaSuccess ? 0 : 1;
}

int xg_probe_rows(void* dst, size_t bytes, uint64_t row_bytes, int vec, int warps, int cap,
                  void* stream) {
    if (row_bytes == 0 || row_bytes % (32 * 32) != 0 || warps < 1 || warps > 32) return 2;
    const uint32_t rows = static_cast<uint32_t>(bytes / row_bytes);
    const unsigned grid = (rows + warps - 1) / warps;
    size_t smem = 0;
    if (cap > 0) {
        int dev = 0, per_sm = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        smem = std::min<size_t>(static_cast<size_t>(per_sm) / cap - 2048, static_cast<size_t>(optin));
    }
    auto launch = [&](auto kernel) {
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)) != cudaSuccess)
            return 1;
        kernel<<<grid, 32 * warps, smem, static_cast<cudaStream_t>(stream)>>>(
            static_cast<char*>(dst), row_bytes, rows, 0x9e3779b9u);
        return cudaGetLastError() == cudaSuccess ? 0 : 1;
    };
    return vec == 8 ? launch(row_store<8>) : vec == 16 ? launch(row_store<16>) : launch(row_store<32>);
}

int xg_probe_gridstride(void* dst, size_t bytes, void* stream) {
    grid_stride<<<sm_count() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint4*>(dst), bytes / 16, 0u);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // extern "C"

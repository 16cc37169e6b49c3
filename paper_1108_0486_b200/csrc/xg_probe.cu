// xg_probe.cu -- bench-only helper (libxg_probe.so): a pure HBM write stream
// (128-bit evict-first stores, grid-stride, 148 SMs x 8 CTAs) used by bench.py
// to measure the write-only ceiling beside the fill kernels in the same run.
// Not part of the generator ABI.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__global__ void __launch_bounds__(256) write_stream(uint4* __restrict__ dst, size_t n16, uint32_t v) {
    const uint4 val = make_uint4(v, v, v, v);
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
#pragma unroll 4
    for (; i < n16; i += stride) __stcs(dst + i, val);
}

}  // namespace

extern "C" int xg_probe_write(void* dst, size_t bytes, void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    write_stream<<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint4*>(dst), bytes / 16, 0u);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

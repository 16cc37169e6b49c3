// store_probe.cu -- microbenchmark: which SM-issued write pattern gets closest
// to the copy engine's memset over a 4 GiB buffer on sm_100a?  The fill
// kernel (pair_kernel) writes one 256 KiB row per warp with STG.64 evict-first
// stores at <= 4 CTAs per SM; the memset (copy engine) is ~3 % faster than
// any SM pattern tried so far.  Variants here: cache-policy flavours of the
// row store, contiguous chunks per CTA, and TMA bulk stores
// (cp.async.bulk.global.shared::cta) from a shared-memory tile.  Not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_probe store_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

// FLAVOR: 0 st.global.cs, 1 st.global (wb), 2 st.global.L1::no_allocate,
// 3 st.global.L2::cache_hint evict_first policy, 4 evict_unchanged policy, 5 .wt
template <int FLAVOR>
__device__ __forceinline__ void st64(uint2* p, uint2 v, uint64_t pol) {
    if constexpr (FLAVOR == 0) asm volatile("st.global.cs.v2.b32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
    else if constexpr (FLAVOR == 1) asm volatile("st.global.v2.b32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
    else if constexpr (FLAVOR == 2) asm volatile("st.global.L1::no_allocate.v2.b32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
    else if constexpr (FLAVOR == 3 || FLAVOR == 4)
        asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1,%2}, %3;" :: "l"(p), "r"(v.x), "r"(v.y), "l"(pol) : "memory");
    else asm volatile("st.global.wt.v2.b32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
}

// one warp per row of row_bytes (the fill's shape), 64-bit stores
template <int FLAVOR>
__global__ void __launch_bounds__(1024) rows(char* dst, uint64_t row_bytes, uint32_t nrows) {
    const uint32_t row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= nrows) return;
    uint64_t pol = 0;
    if constexpr (FLAVOR == 3) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if constexpr (FLAVOR == 4) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
    const unsigned lane = threadIdx.x & 31u;
    uint2* p = reinterpret_cast<uint2*>(dst + static_cast<uint64_t>(row) * row_bytes) + lane;
    const uint2 v = make_uint2(row, lane);
    const uint64_t n = row_bytes / 256;
#pragma unroll 8
    for (uint64_t i = 0; i < n; ++i) st64<FLAVOR>(p + 32 * i, v, pol);
}

// each CTA writes one contiguous chunk, all its threads side by side (STG.128)
__global__ void __launch_bounds__(512) chunks(uint4* dst, uint64_t chunk16, uint32_t nchunks) {
    if (blockIdx.x >= nchunks) return;
    uint4* p = dst + static_cast<uint64_t>(blockIdx.x) * chunk16 + threadIdx.x;
    const uint4 v = make_uint4(blockIdx.x, threadIdx.x, 1, 2);
    const uint64_t n = chunk16 / blockDim.x;
#pragma unroll 8
    for (uint64_t i = 0; i < n; ++i) __stcs(p + static_cast<uint64_t>(blockDim.x) * i, v);
}

// TMA bulk stores: each warp owns a row; its lane 0 streams a smem tile of
// `tile` bytes to consecutive row addresses with cp.async.bulk, keeping at
// most `depth` bulk groups in flight.  Smem contents are whatever was written
// once at start (the point is the engine's write rate).
__global__ void __launch_bounds__(1024) bulk_rows(char* dst, uint64_t row_bytes, uint32_t nrows,
                                                  uint32_t tile, int depth) {
    extern __shared__ __align__(128) char sm[];
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    char* t = sm + warp * tile;
    for (uint32_t i = lane * 16; i < tile; i += 512) *reinterpret_cast<uint4*>(t + i) = make_uint4(warp, i, 7, 9);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint32_t row = blockIdx.x * (blockDim.x >> 5) + warp;
    if (row >= nrows || lane != 0) return;
    char* r = dst + static_cast<uint64_t>(row) * row_bytes;
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(t));
    const uint64_t n = row_bytes / tile;
    for (uint64_t i = 0; i < n; ++i) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(r + i * tile), "r"(sa), "r"(tile) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (depth == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        else if (depth == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else if (depth == 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t bytes = size_t(4) << 30;
    char* d;
    CK(cudaMalloc(&d, bytes));
    int sms = 0, smem_sm = 0, optin = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        cudaDeviceSynchronize();
        std::vector<float> ms;
        for (int i = 0; i < 20; ++i) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            ms.push_back(t);
        }
        float best = 1e9, sum = 0;
        for (float t : ms) { best = t < best ? t : best; sum += t; }
        cudaError_t err = cudaGetLastError();
        printf("%-44s mean %.4f ms  %.1f GB/s  (best %.1f)%s%s\n", name, sum / ms.size(),
               bytes / (sum / ms.size()) / 1e6, bytes / best / 1e6, err ? "  ERROR " : "",
               err ? cudaGetErrorString(err) : "");
    };
    timeit("memset (copy engine)", [&] { cudaMemsetAsync(d, 0x5a, bytes); });
    const uint64_t rb = 256 << 10;
    const uint32_t nr = static_cast<uint32_t>(bytes / rb);
    auto rows_cap = [&](auto k, int warps, int cap) {
        size_t smem = cap ? std::min<size_t>(smem_sm / cap - 2048, optin) : 0;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<(nr + warps - 1) / warps, 32 * warps, smem>>>(d, rb, nr);
    };
    char name[128];
    for (int cap : {4, 2}) {
        for (int warps : {4, 8}) {
            snprintf(name, sizeof name, "rows st.cs        %dw cap%d", warps, cap);
            timeit(name, [&] { rows_cap(rows<0>, warps, cap); });
            snprintf(name, sizeof name, "rows st.wb        %dw cap%d", warps, cap);
            timeit(name, [&] { rows_cap(rows<1>, warps, cap); });
            snprintf(name, sizeof name, "rows st.L1noalloc %dw cap%d", warps, cap);
            timeit(name, [&] { rows_cap(rows<2>, warps, cap); });
            snprintf(name, sizeof name, "rows L2 evict_first pol %dw cap%d", warps, cap);
            timeit(name, [&] { rows_cap(rows<3>, warps, cap); });
            snprintf(name, sizeof name, "rows L2 evict_unchanged pol %dw cap%d", warps, cap);
            timeit(name, [&] { rows_cap(rows<4>, warps, cap); });
            snprintf(name, sizeof name, "rows st.wt        %dw cap%d", warps, cap);
            timeit(name, [&] { rows_cap(rows<5>, warps, cap); });
        }
    }
    for (uint64_t chunk : {uint64_t(1) << 20, uint64_t(4) << 20, uint64_t(16) << 20}) {
        for (int th : {256, 512}) {
            const uint32_t nc = static_cast<uint32_t>(bytes / chunk);
            snprintf(name, sizeof name, "chunks %4llu KiB/CTA %d thr", (unsigned long long)(chunk >> 10), th);
            timeit(name, [&] { chunks<<<nc, th>>>(reinterpret_cast<uint4*>(d), chunk / 16, nc); });
        }
    }
    for (uint32_t tile : {4096u, 8192u, 16384u}) {
        for (int warps : {4, 8}) {
            for (int depth : {2, 8}) {
                const size_t smem = size_t(tile) * warps;
                if (smem > static_cast<size_t>(optin)) continue;
                cudaFuncSetAttribute(bulk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                snprintf(name, sizeof name, "bulk rows tile %5u %dw depth %d", tile, warps, depth);
                timeit(name, [&] { bulk_rows<<<(nr + warps - 1) / warps, 32 * warps, smem>>>(d, rb, nr, tile, depth); });
            }
        }
    }
    cudaFree(d);
    return 0;
}

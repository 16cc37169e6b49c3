// gf2_tc_probe.cu -- experiment: GF(2) products C = A B (4096-bit rows, the
// jump-ahead's operation, csrc/xg_jump.cuh) on the 5th-generation tensor
// cores: bits expanded to 0/1 bytes while staging into shared memory,
// tcgen05.mma.kind::i8 (u8 x u8 -> s32 in TMEM), parity of the int32 sums
// packed back to bits in the epilogue; k split over CTAs, the parities
// XOR-reduced (parity is additive mod 2).  Standalone: checks against a
// host GF(2) product and times it.  Not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gf2_tc_probe gf2_tc_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

constexpr int kW = 128;        // u32 words per 4096-bit row
constexpr int TM = 128;        // rows of A per CTA (UMMA M)
constexpr int TN = 256;        // columns per CTA (UMMA N)
constexpr int SK = 128;        // K bytes per stage (4 MMAs of K = 32)
constexpr int kSmemA = TM * SK;  // 16 KB
constexpr int kSmemB = TN * SK;  // 32 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8 bits -> 8 bytes of 0/1 (bit i -> byte i)
__device__ __forceinline__ uint64_t spread8(uint32_t b) {
    uint64_t x = (b & 0xffu) * 0x0101010101010101ull;
    x &= 0x8040201008040201ull;
    // byte i holds bit i at position 8i + i; move it to the byte's bit 0
    x = (x + 0x7f7f7f7f7f7f7f7full) >> 7 & 0x0101010101010101ull;  // nonzero byte -> 1
    return x;
}

// smem descriptor, SWIZZLE_NONE (interleave), version 1 (sm_100)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3fff) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3fff) << 32;
    d |= 1ull << 46;  // version
    return d;         // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
}

// instruction descriptor: u8 x u8 -> s32, A K-major, B MN-major, M = 128, N = 256
__host__ __device__ constexpr uint32_t make_idesc() {
    return (2u << 4)            // c_format S32
         | (0u << 7)            // a_format u8
         | (0u << 10)           // b_format u8
         | (0u << 15)           // a_major K
         | (1u << 16)           // b_major MN
         | ((TN >> 3) << 17)    // n_dim
         | ((TM >> 4) << 24);   // m_dim
}

// part[z][r][col word] = parity bits of A[r] B over k in [z kspan, (z+1) kspan)
// grid (4096 / TN, ceil(rows / TM), ksplit), 128 threads, dynamic smem
// 2 x (A stage + B stage): the 128 threads expand stage s + 1 (bits -> 0/1
// bytes in the canonical layouts) while the tensor core runs stage s.
// B item i -> (K row, N word): i % 8 = K row within an 8-row block, then the
// N word, then the block -- a warp's stores hit 8 distinct 16-byte bank groups
__device__ __forceinline__ void bitem(unsigned i, unsigned& k, unsigned& nw) {
    const unsigned q = i >> 3;
    nw = q % (TN / 32);
    k = (q / (TN / 32)) * 8 + (i & 7u);
}
constexpr int kStages = 2;
constexpr int kStageBytes = kSmemA + kSmemB;
constexpr int kThr = 256;
constexpr int kAW = TM * (SK / 32) / kThr;  // A words per thread per stage (2)
constexpr int kBW = SK * (TN / 32) / kThr;  // B words per thread per stage (4)
__global__ void __launch_bounds__(kThr)
gf2_tc_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B, uint32_t* __restrict__ part,
              uint32_t rows, uint32_t kspan, uint32_t ldb) {
    extern __shared__ __align__(1024) uint8_t dyn[];
    __shared__ uint64_t mbar[kStages];
    __shared__ uint2 lut[256];  // byte b -> its 8 bits as 8 bytes of 0/1
    {
        const uint64_t x = spread8(threadIdx.x);
        lut[threadIdx.x] = make_uint2(static_cast<uint32_t>(x), static_cast<uint32_t>(x >> 32));
    }
    __shared__ uint32_t tmem_base;
    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint32_t n0 = blockIdx.x * TN, r0 = blockIdx.y * TM, k0 = blockIdx.z * kspan;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(TN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    uint32_t phase[kStages] = {0, 0};
    const uint32_t nst = kspan / SK;
    auto wait_buf = [&](int b) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(&mbar[b])), "r"(phase[b]));
        phase[b] ^= 1u;
    };
    // the words a thread expands: A item i = tid + kThr t (row i / 4, word i % 4),
    // B item i = tid + kThr t (K row i / 8, word i % 8)
    uint32_t ra[kAW], rb[kBW];
    auto load = [&](uint32_t ks) {
        #pragma unroll
        for (int t = 0; t < kAW; ++t) {
            const unsigned i = tid + kThr * t, r = i / (SK / 32), kw = i % (SK / 32);
            ra[t] = r0 + r < rows ? A[static_cast<size_t>(r0 + r) * kW + (ks >> 5) + kw] : 0u;
        }
        #pragma unroll
        for (int t = 0; t < kBW; ++t) {
            unsigned k, nw;
            bitem(tid + kThr * t, k, nw);
            rb[t] = B[static_cast<size_t>(ks + k) * ldb + (n0 >> 5) + nw];
        }
    };
    load(k0);
    for (uint32_t st = 0; st < nst; ++st) {
        const int b = st & 1;
        uint8_t* sA = dyn + b * kStageBytes;
        uint8_t* sB = sA + kSmemA;
        uint32_t ca[kAW], cb[kBW];
        #pragma unroll
        for (int t = 0; t < kAW; ++t) ca[t] = ra[t];
        #pragma unroll
        for (int t = 0; t < kBW; ++t) cb[t] = rb[t];
        if (st + 1 < nst) load(k0 + (st + 1) * SK);  // next stage's words in flight meanwhile
        if (st >= kStages) wait_buf(b);  // the MMAs that last read this buffer are done
#ifdef PROBE_MMA_ONLY
        if (st < kStages)
#endif
        #pragma unroll
        for (int t = 0; t < kAW; ++t) {  // A: K-major canonical
            const unsigned i = tid + kThr * t, r = i / (SK / 32), kw = i % (SK / 32);
            #pragma unroll
            for (int h = 0; h < 2; ++h) {
                const unsigned kc = kw * 2 + h;
                const uint2 lo = lut[(ca[t] >> (16 * h)) & 0xffu], hi = lut[(ca[t] >> (16 * h + 8)) & 0xffu];
                uint8_t* dst = sA + kc * (TM / 8) * 128 + (r / 8) * 128 + (r % 8) * 16;
                *reinterpret_cast<uint4*>(dst) = make_uint4(lo.x, lo.y, hi.x, hi.y);
            }
        }
#ifdef PROBE_MMA_ONLY
        if (st < kStages)
#endif
        #pragma unroll
        for (int t = 0; t < kBW; ++t) {  // B: MN-major canonical
            unsigned k, nw;
            bitem(tid + kThr * t, k, nw);
            #pragma unroll
            for (int h = 0; h < 2; ++h) {
                const unsigned nb = nw * 2 + h;
                const uint2 lo = lut[(cb[t] >> (16 * h)) & 0xffu], hi = lut[(cb[t] >> (16 * h + 8)) & 0xffu];
                uint8_t* dst = sB + (k / 8) * (TN / 16) * 128 + nb * 128 + (k % 8) * 16;
                *reinterpret_cast<uint4*>(dst) = make_uint4(lo.x, lo.y, hi.x, hi.y);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            #pragma unroll
            for (int m = 0; m < SK / 32; ++m) {
                const uint64_t da = make_desc(smem_u32(sA) + 2 * m * (TM / 8) * 128, (TM / 8) * 128, 128);
                const uint64_t db = make_desc(smem_u32(sB) + 4 * m * (TN / 16) * 128, (TN / 16) * 128, 128);
                const uint32_t acc = (st > 0 || m > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                    ::"r"(tmem), "l"(da), "l"(db), "r"(make_idesc()), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar[b])));
        }
    }
    for (uint32_t st = (nst > kStages ? nst - kStages : 0); st < nst; ++st) wait_buf(st & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {  // warps 0..3 own TMEM lanes 0..127
        const uint32_t r = r0 + warp * 32 + lane;
        #pragma unroll 1
        for (int c = 0; c < TN / 32; ++c) {
            uint32_t v[32];
            const uint32_t taddr = tmem + ((warp * 32u) << 16) + c * 32u;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            uint32_t word = 0;
            #pragma unroll
            for (int j = 0; j < 32; ++j) word |= (v[j] & 1u) << j;
            if (r < rows) part[(static_cast<size_t>(blockIdx.z) * rows + r) * kW + (n0 >> 5) + c] = word;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TN));
}

__global__ void xor_reduce(const uint32_t* part, uint32_t* C, uint32_t rows, uint32_t ksplit) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x, n = static_cast<size_t>(rows) * kW;
    if (i >= n) return;
    uint32_t v = 0;
    for (uint32_t z = 0; z < ksplit; ++z) v ^= part[z * n + i];
    C[i] = v;
}

int main() {
    std::mt19937_64 rng(7);
    for (uint32_t rows : {128u, 763u, 4096u}) {
        std::vector<uint32_t> A(static_cast<size_t>(rows) * kW), B(static_cast<size_t>(4096) * kW), C(A.size()), R(A.size(), 0);
        for (auto& x : A) x = static_cast<uint32_t>(rng());
        for (auto& x : B) x = static_cast<uint32_t>(rng());
        for (uint32_t r = 0; r < rows; ++r)  // host reference
            for (int k = 0; k < 4096; ++k)
                if ((A[static_cast<size_t>(r) * kW + k / 32] >> (k % 32)) & 1u)
                    for (int w = 0; w < kW; ++w) R[static_cast<size_t>(r) * kW + w] ^= B[static_cast<size_t>(k) * kW + w];
        uint32_t *dA, *dB, *dC, *dP;
        const uint32_t ksplit = rows >= 1024 ? 1 : (rows >= 512 ? 2 : 4), kspan = 4096 / ksplit;
        CK(cudaFuncSetAttribute(gf2_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStageBytes));
        CK(cudaMalloc(&dA, A.size() * 4));
        CK(cudaMalloc(&dB, B.size() * 4));
        CK(cudaMalloc(&dC, C.size() * 4));
        CK(cudaMalloc(&dP, C.size() * 4 * 8));
        CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
        dim3 grid(4096 / TN, (rows + TM - 1) / TM, ksplit);
        auto run = [&] {
            gf2_tc_kernel<<<grid, kThr, kStages * kStageBytes>>>(dA, dB, dP, rows, kspan, kW);
            xor_reduce<<<(rows * kW + 255) / 256, 256>>>(dP, dC, rows, ksplit);
        };
        run();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
        size_t bad = 0;
        for (size_t i = 0; i < C.size(); ++i) bad += C[i] != R[i];
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int t = 0; t < 20; ++t) run();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("rows %u: %zu / %zu words differ from the host product; %.1f us per product (incl. reduce)\n", rows,
               bad, C.size(), ms / 20 * 1e3);
        if (bad) {
            for (size_t i = 0; i < 8; ++i) printf("  C[%zu] = %08x  R = %08x\n", i, C[i], R[i]);
        }
        cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dP);
    }
    return 0;
}

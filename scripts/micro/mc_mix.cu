// mc_mix.cu -- the instruction mix of the fused Monte Carlo loop
// (pair_kernel<GP32, kMC>, xg_pairs.cuh) with every dependency removed: per
// 64 words 10 LOP3, 6 SHF, 1 LEA.HI (ALU pipe); 4 IMAD.SHL, 2 IMAD, 2 IMAD.IADD,
// 1 IMAD.WIDE, 1 IMAD.HI, 2 VIADD (FMA pipe); 1 SHFL -- the per-512-word
// counts of scripts/sass_loops.py / 8.  Independent chains, full occupancy:
// the rate this mix can issue at on sm_100a, i.e. the ceiling of any kernel
// with this instruction mix (the MC kernel's "mix roofline").  Reports words
// per SM per clock and the implied RN/s at 1965 MHz x 148 SMs; not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_mix mc_mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

__global__ void __launch_bounds__(256) mc_mix(uint32_t* out, uint32_t k1, uint32_t k2) {
    uint32_t l[10], s[6], acc = 0, m[4], g[2], ad[2], va[2], w, h, sh;
    uint64_t wd;
#pragma unroll
    for (int i = 0; i < 10; ++i) l[i] = threadIdx.x * 7919u + i;
#pragma unroll
    for (int i = 0; i < 6; ++i) s[i] = threadIdx.x * 31u + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = threadIdx.x + i;
    g[0] = g[1] = ad[0] = ad[1] = va[0] = va[1] = threadIdx.x;
    w = h = sh = threadIdx.x;
    wd = threadIdx.x;
    const uint32_t rot = (threadIdx.x + 1) & 31;  // lane rotation: shuffles do not fold
    const uint32_t one = k2 - 4u;                   // 1 at run time (k2 = 5), unknown to ptxas
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // 8 x 64 words = one 512-word loop trip
            // every op reads a value that changes each time (a LOP3 chain) and
            // accumulates into its own chain, so ptxas can neither fold nor drop it
#pragma unroll
            for (int i = 0; i < 10; ++i)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(l[i]) : "r"(k1), "r"(k2));
#pragma unroll
            for (int i = 0; i < 6; ++i) asm volatile("shf.r.wrap.b32 %0, %1, %0, 14;" : "+r"(s[i]) : "r"(l[i]));
            asm volatile("{\n\t.reg .u32 t;\n\tshr.u32 t, %1, 31;\n\tadd.u32 %0, %0, t;\n\t}" : "+r"(acc) : "r"(l[u & 7]));
#pragma unroll
            for (int i = 0; i < 4; ++i) asm volatile("mad.lo.u32 %0, %1, 32768, %0;" : "+r"(m[i]) : "r"(l[i + 2]));
#pragma unroll
            for (int i = 0; i < 2; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(g[i]) : "r"(k1), "r"(l[i + 6]));
#pragma unroll
            for (int i = 0; i < 2; ++i)  // the "+ v" adds (IMAD.IADD in the kernel)
                asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(ad[i]) : "r"(l[i + 8]), "r"(one));
            asm volatile("mad.wide.s32 %0, %1, %1, %0;" : "+l"(wd) : "r"(l[u & 3]));
            asm volatile("mad.hi.u32 %0, %1, %1, %0;" : "+r"(h) : "r"(l[(u + 4) & 7]));
#pragma unroll
            for (int i = 0; i < 2; ++i)  // the Weyl VIADDs
                asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(va[i]) : "r"(s[i + 2]), "r"(one));
            asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(sh) : "r"(rot));
        }
    }
    uint32_t x = acc ^ w ^ h ^ sh ^ (uint32_t)wd;
#pragma unroll
    for (int i = 0; i < 10; ++i) x ^= l[i];
#pragma unroll
    for (int i = 0; i < 6; ++i) x ^= s[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) x ^= m[i];
    x ^= g[0] ^ g[1] ^ ad[0] ^ ad[1] ^ va[0] ^ va[1];
    if (x == 0x12345678u) out[0] = x;
}

int main() {
    uint32_t* out;
    cudaMalloc(&out, 4);
    int sms = 148, dev = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 2;  // 16 warps per SM, ~30 independent chains each
    mc_mix<<<blocks, 256>>>(out, 3u, 5u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        mc_mix<<<blocks, 256>>>(out, 3u, 5u);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double words = (double)blocks * 256 / 32 * ITERS * 512;  // warps x trips x 512
    printf("mc_mix: %.3f ms, %.4e words/s (mix ceiling at the clock of this run), "
           "%.4f words/SM/clk at 1965 MHz\n", best, words / (best * 1e-3),
           words / (best * 1e-3) / sms / 1.965e9);
    return 0;
}

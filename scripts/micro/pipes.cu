// pipes.cu -- microbenchmark: issue throughput of the integer instructions the
// xorgensGP kernels are made of (SHF, LOP3, IMAD.SHL, IMAD.HI, IMAD.WIDE,
// VIADD/IADD3, LEA.HI, SEL, PRMT, SHFL) on sm_100a.  Reports warp-instructions
// per SM-cycle (4.0 = one per SMSP per cycle).  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_ACC 8
#define ITERS 2048

template <int OP>
__global__ void __launch_bounds__(256) bench(uint32_t* out, uint32_t k1, uint32_t k2,
                                            unsigned long long* cycles) {
    uint32_t a[N_ACC];
#pragma unroll
    for (int i = 0; i < N_ACC; ++i) a[i] = threadIdx.x * 7919u + i * 104729u + k2;
    const bool p = (threadIdx.x & 31) == 31;
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < N_ACC; ++i) {
            uint32_t x = a[i];
            if (OP == 0) asm volatile("shf.r.clamp.b32 %0, %1, %1, 14;" : "=r"(x) : "r"(x));
            if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(k1), "r"(k2));
            if (OP == 2) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x) : "r"(k1));
            if (OP == 3) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(k1));
            if (OP == 4) { uint64_t w; asm volatile("mul.wide.u32 %0, %1, %1;" : "=l"(w) : "r"(x)); x = (uint32_t)w ^ (uint32_t)(w >> 32); }
            if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(k1));
            if (OP == 6) asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; selp.b32 %0, %0, %1, q;}" : "+r"(x) : "r"(k1), "r"((int)p));
            if (OP == 7) asm volatile("prmt.b32 %0, %0, 0, 0x1032;" : "+r"(x));
            if (OP == 8) asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(x) : "r"(k1));
            if (OP == 9) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(k1), "r"(k2));
            if (OP == 10) asm volatile("xor.b32 %0, %0, %1;" : "+r"(x) : "r"(k1));
            if (OP == 11) asm volatile("shl.b32 %0, %0, 15;" : "+r"(x));
            if (OP == 12) asm volatile("{.reg .u32 t; shr.u32 t, %0, 16; add.u32 %0, t, %1;}" : "+r"(x) : "r"(k1));
            a[i] = x;
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < N_ACC; ++i) s ^= a[i];
    if (s == 0x12345678u) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
}

template <int OP>
void run(const char* name, uint32_t* out, unsigned long long* cyc) {
    const int blocks = 148 * 8;
    bench<OP><<<blocks, 256>>>(out, 3u, 5u, cyc);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<OP><<<blocks, 256>>>(out, 1u << 18, 5u, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double warp_instr = (double)blocks * 8 * ITERS * N_ACC;
    // cycles of one block ~ whole kernel at full occupancy (one wave)
    double per_sm_clk = warp_instr / 148.0 / (double)c;
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("%-10s %6.3f warp-instr/SM/clk  (block cycles %llu, %.3f ms, eff clk %.0f MHz)\n", name,
           per_sm_clk, c, ms, c / (ms * 1e3));
}

int main() {
    uint32_t* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 8);
    run<0>("SHF.R", out, cyc);
    run<1>("LOP3", out, cyc);
    run<2>("IMUL.LO", out, cyc);
    run<3>("IMAD.HI", out, cyc);
    run<4>("IMAD.WIDE", out, cyc);
    run<5>("IADD", out, cyc);
    run<6>("SEL", out, cyc);
    run<7>("PRMT", out, cyc);
    run<8>("SHFL", out, cyc);
    run<9>("IMAD", out, cyc);
    run<10>("XOR", out, cyc);
    run<11>("SHL", out, cyc);
    run<12>("LEA.HI", out, cyc);
    return 0;
}

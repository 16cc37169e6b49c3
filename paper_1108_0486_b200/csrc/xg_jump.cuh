// xg_jump.cuh -- jump-ahead for the register-window sets (w = 32, r = 128).
//
// The Weyl-free part of xorgens is linear over GF(2): the 128-word window
// (oldest first, proj/include/xg/xorgens.hpp:39-47) is a 4096-bit row vector
// s, and one word step is s' = s G for a fixed 4096 x 4096 bit matrix G
// (rows: the images of the unit windows; built on the host in xg_gpu.cu).
// The state n words ahead is s G^n, and the Weyl accumulator is
// weyl + n omega (proj/include/xg/xorgens.hpp:50-53), so ONE stream can be
// cut into K segments whose start states are computed directly and generated
// by K warps at once -- a single generator's fill-buffer then runs at the
// ensemble rate instead of one warp's.  The reference has no jump-ahead (its
// streams come from consecutive seeds, proj/src/parallel.cpp:84-95); the
// output is the reference's stream word for word, which the parity tests
// check against the reference's own words (config 1: 10^8 words of seed 1).
//
// Layout: a row is the window itself, 128 u32 words, element k = bit k % 32
// of word k / 32.  C = A B (row-vector convention) is
//   C[r] = XOR over k with bit k of A[r] set of B[k]
// computed in two kernels: k is split into `ksplit` ranges, each CTA stages
// 64 rows of B in shared memory (32 KB) and XORs them, masked by the bits of
// A, into 8 RW output rows (a warp per RW rows, a lane per 4 words), writing
// partial rows; a second kernel XORs the partials.
#pragma once

#include <cstdint>

namespace xgk {

constexpr int kJWords = 128;  // u32 words per 4096-bit row
constexpr int kJStage = 64;   // rows of B per shared-memory stage


// part[c][r][:] = XOR over k in [c * kspan, (c + 1) * kspan) of A[r]_k B[k].
// grid (ceil(rows / (8 RW)), ksplit), 256 threads: warp w owns the RW rows
// blockIdx.x * 8 RW + w RW .. + RW.  Per staged row k of B one LDS.128 per
// lane serves all RW rows (predicated XORs, k unrolled: no data-dependent
// branches, the loads of a stage pipeline freely).
template <int RW>
__global__ void __launch_bounds__(256)
gf2_mul_partial_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                       uint32_t* __restrict__ part, uint32_t rows, uint32_t kspan) {
    __shared__ uint4 Bs[kJStage][kJWords / 4];
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t r0 = blockIdx.x * (8u * RW) + warp * RW;
    const uint32_t k0 = blockIdx.y * kspan;
    uint4 acc[RW];
#pragma unroll
    for (int m = 0; m < RW; ++m) acc[m] = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t kc = k0; kc < k0 + kspan; kc += kJStage) {
        __syncthreads();
        const uint4* src = reinterpret_cast<const uint4*>(B + static_cast<size_t>(kc) * kJWords);
#pragma unroll
        for (unsigned i = threadIdx.x; i < kJStage * (kJWords / 4); i += 256)
            Bs[i >> 5][i & 31u] = src[i];
        uint32_t lo[RW], hi[RW];  // bits kc .. kc + 63 of each row (0 past `rows`)
#pragma unroll
        for (int m = 0; m < RW; ++m) {
            const uint32_t r = r0 + m;
            const uint32_t* a = A + static_cast<size_t>(r < rows ? r : 0) * kJWords + (kc >> 5);
            lo[m] = r < rows ? a[0] : 0u;
            hi[m] = r < rows ? a[1] : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kJStage; ++k) {
            const uint4 b = Bs[k][lane];
#pragma unroll
            for (int m = 0; m < RW; ++m) {
                const uint32_t word = k < 32 ? lo[m] : hi[m];
                const uint32_t msk = static_cast<uint32_t>(static_cast<int32_t>(word << (31 - (k & 31))) >> 31);
                acc[m].x ^= b.x & msk;
                acc[m].y ^= b.y & msk;
                acc[m].z ^= b.z & msk;
                acc[m].w ^= b.w & msk;
            }
        }
    }
#pragma unroll
    for (int m = 0; m < RW; ++m) {
        const uint32_t r = r0 + m;
        if (r < rows)
            reinterpret_cast<uint4*>(part + (static_cast<size_t>(blockIdx.y) * rows + r) * kJWords)[lane] =
                acc[m];
    }
}

// The same product by the method of the four Russians, for many rows: per
// group of 8 rows of B (bits 8g .. 8g + 7 of every A row) a table of all 256
// XOR combinations of those rows is built in shared memory (Gray-code order,
// one XOR per entry), and every A row then takes ONE table lookup per group
// instead of 8 masked XORs.  CTA = (column slab of 32 words, 8 RW rows,
// k-split range of kspan <= 256 rows of B); its slab of B and its rows' bits
// of A are staged in shared memory first, so the group loop touches no
// global memory; lane = word of the slab, so a lookup is one conflict-free
// LDS.32 per warp.  Row k of B starts at B + k ldb (ldb = 128 for a matrix,
// 1 for the overlapping windows of a raw run, which then need no expansion).
// grid (4, ceil(rows / (8 RW)), ksplit).
constexpr int kM4Span = 256;  // max kspan of the four-Russians kernel
constexpr size_t kM4Smem = (256 + kM4Span) * 32 * sizeof(uint32_t);  // table + staged B
template <int RW>
__global__ void __launch_bounds__(256)
gf2_mul_m4rm_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                    uint32_t* __restrict__ part, uint32_t rows, uint32_t kspan, uint32_t ldb) {
    extern __shared__ uint32_t m4_dyn[];           // kM4Smem bytes (dynamic, > 48 KB)
    uint32_t(*T)[32] = reinterpret_cast<uint32_t(*)[32]>(m4_dyn);                 // [256][32]
    uint32_t(*Bsl)[32] = reinterpret_cast<uint32_t(*)[32]>(m4_dyn + 256 * 32);    // B rows k0.., this slab
    __shared__ uint32_t As[8 * RW][kM4Span / 32];  // A words of the CTA's rows in range
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const unsigned col = blockIdx.x * 32u + lane;  // word of the row this lane owns
    const uint32_t rt = blockIdx.y * (8u * RW);
    const uint32_t k0 = blockIdx.z * kspan;
    const unsigned kw_n = kspan >> 5;
    // staging: every load of a thread issued before its first store (latency once)
    if (kspan == kM4Span) {
        uint32_t v[kM4Span / 8];
#pragma unroll
        for (int i = 0; i < kM4Span / 8; ++i) v[i] = B[static_cast<size_t>(k0 + warp + 8 * i) * ldb + col];
#pragma unroll
        for (int i = 0; i < kM4Span / 8; ++i) Bsl[warp + 8 * i][lane] = v[i];
    } else {
        for (unsigned i = warp; i < kspan; i += 8) Bsl[i][lane] = B[static_cast<size_t>(k0 + i) * ldb + col];
    }
    {
        constexpr int kAn = (8 * RW * (kM4Span / 32) + 255) / 256;
        uint32_t v[kAn];
#pragma unroll
        for (int t = 0; t < kAn; ++t) {
            const unsigned i = threadIdx.x + 256u * t, r = i / kw_n, w = i % kw_n;
            v[t] = (i < 8u * RW * kw_n && rt + r < rows) ? A[static_cast<size_t>(rt + r) * kJWords + (k0 >> 5) + w] : 0u;
        }
#pragma unroll
        for (int t = 0; t < kAn; ++t) {
            const unsigned i = threadIdx.x + 256u * t;
            if (i < 8u * RW * kw_n) As[i / kw_n][i % kw_n] = v[t];
        }
    }
    uint32_t acc[RW];
#pragma unroll
    for (int m = 0; m < RW; ++m) acc[m] = 0u;
    for (unsigned g = 0; g < (kspan >> 3); ++g) {
        __syncthreads();  // staging done / the previous group's lookups are done
        // warp w writes entries 32w .. 32w + 31: base = rows 5..7 picked by w,
        // then the 32 combinations of rows 0..4 in Gray-code order
        uint32_t b[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) b[i] = Bsl[8 * g + i][lane];
        uint32_t cur = ((warp & 1u) ? Bsl[8 * g + 5][lane] : 0u) ^ ((warp & 2u) ? Bsl[8 * g + 6][lane] : 0u) ^
                       ((warp & 4u) ? Bsl[8 * g + 7][lane] : 0u);
        T[32u * warp][lane] = cur;
#pragma unroll
        for (int t = 1; t < 32; ++t) {  // row ctz(t) flips between Gray codes t-1 and t
            cur ^= (t & 1) ? b[0] : (t & 2) ? b[1] : (t & 4) ? b[2] : (t & 8) ? b[3] : b[4];
            T[32u * warp + (t ^ (t >> 1))][lane] = cur;
        }
        __syncthreads();
        const unsigned sh = 8u * (g & 3u);
#pragma unroll
        for (int m = 0; m < RW; ++m) acc[m] ^= T[(As[warp * RW + m][g >> 2] >> sh) & 0xffu][lane];
    }
#pragma unroll
    for (int m = 0; m < RW; ++m) {
        const uint32_t r = rt + warp * RW + m;
        if (r < rows) part[(static_cast<size_t>(blockIdx.z) * rows + r) * kJWords + col] = acc[m];
    }
}

// C[r] = XOR over c < ksplit of part[c][r]   (one thread per 16 bytes; the
// ksplit loads are independent, eight in flight)
__global__ void __launch_bounds__(256)
gf2_reduce_kernel(const uint32_t* __restrict__ part, uint32_t* __restrict__ C, uint32_t rows,
                  uint32_t ksplit) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t n = static_cast<uint64_t>(rows) * (kJWords / 4);
    if (i >= n) return;
    const uint4* p = reinterpret_cast<const uint4*>(part);
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t c = 0; c < ksplit; c += 8) {  // ksplit is a multiple of 8
        uint4 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = p[(c + u) * n + i];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v.x ^= q[u].x;
            v.y ^= q[u].y;
            v.z ^= q[u].z;
            v.w ^= q[u].w;
        }
    }
    reinterpret_cast<uint4*>(C)[i] = v;
}

// W[i][w] = seq[i + w]: the 4096 windows of a raw run (seq = s_0 ++ 4096
// raw words) as the rows of a GF(2) matrix.
__global__ void __launch_bounds__(256)
jump_windows_kernel(const uint32_t* __restrict__ seq, uint32_t* __restrict__ W) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // < 4096 * 128
    W[t] = seq[(t >> 7) + (t & 127u)];
}

// Start of a jump fill, one launch: the source window (128 words) copied to
// dst_a and, if given, dst_b; the segment Weyl words wout[k] = w0[0] + k step
// (mod 2^32), k < n.
__global__ void __launch_bounds__(256)
jump_begin_kernel(const uint32_t* __restrict__ win, const uint32_t* __restrict__ w0, uint32_t* __restrict__ dst_a,
                  uint32_t* __restrict__ dst_b, uint32_t* __restrict__ wout, uint32_t n, uint32_t step) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < kJWords) {
        const uint32_t v = win[t];
        dst_a[t] = v;
        if (dst_b) dst_b[t] = v;
    }
    if (t < n) wout[t] = w0[0] + t * step;
}

// End of a jump fill: the stream continues from the last segment's state.
__global__ void jump_end_kernel(const uint32_t* __restrict__ win, const uint32_t* __restrict__ w,
                                uint32_t* __restrict__ dst_win, uint32_t* __restrict__ dst_w) {
    const uint32_t t = threadIdx.x;  // 128 threads
    dst_win[t] = win[t];
    if (t == 0) dst_w[0] = w[0];
}

// Many streams, Q full segments (+ one remainder if cq = Q + 1) each
// (jump_fill_many): the jumped windows come q-major (row q P + g, so each
// doubling level is one contiguous product); the fill wants the full
// segments g-major (row g Q + q: segment q of stream g, output at g ld + q J)
// followed by the P remainders (row P Q + g, already contiguous).
// dst[g Q + q] = src[q P + g], dst[P Q + g] = src[Q P + g];
// Weyl words w[g] + q step alike.  One warp per row, 16 bytes per lane.
__global__ void __launch_bounds__(256)
jump_permute_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, const uint32_t* __restrict__ w,
                    uint32_t* __restrict__ wout, uint32_t P, uint32_t Q, uint32_t cq, uint32_t step) {
    const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (row >= P * cq) return;
    uint32_t g, q;
    if (row < P * Q) {
        g = row / Q;
        q = row % Q;
    } else {
        g = row - P * Q;
        q = Q;
    }
    reinterpret_cast<uint4*>(dst + static_cast<size_t>(row) * kJWords)[lane] =
        reinterpret_cast<const uint4*>(src + (static_cast<size_t>(q) * P + g) * kJWords)[lane];
    if (lane == 0) wout[row] = w[g] + q * step;
}

// ... and after the fill every stream continues from its last segment:
// the remainder (row P Q + g) if there is one, else row g Q + Q - 1.
__global__ void __launch_bounds__(256)
jump_finish_many_kernel(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ wrows,
                        uint32_t* __restrict__ win, uint32_t* __restrict__ weyl, uint32_t P, uint32_t Q,
                        bool has_rem) {
    const uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (g >= P) return;
    const size_t last = has_rem ? static_cast<size_t>(P) * Q + g : static_cast<size_t>(g) * Q + Q - 1;
    reinterpret_cast<uint4*>(win + static_cast<size_t>(g) * kJWords)[lane] =
        reinterpret_cast<const uint4*>(rows + last * kJWords)[lane];
    if (lane == 0) weyl[g] = wrows[last];
}

// w[k] += step (mod 2^32), k < n: the Weyl words of skipped streams.
__global__ void jump_weyl_add_kernel(uint32_t* __restrict__ w, uint32_t n, uint32_t step) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) w[k] += step;
}

}  // namespace xgk

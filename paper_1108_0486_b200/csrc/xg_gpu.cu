// xg_gpu.cu -- host side of libxg_gpu.so: the C ABI declared in
// include/xg_gpu.h over the sm_100a kernels (xg_pairs.cuh, xg_kernels.cuh,
// xg_generic.cuh, xg_jump.cuh, xg_stattests.cuh, xg_digest.cuh).
//
// Host validation mirrors the reference exactly (check order and error
// classes of proj/src/params.cpp:22-37 and proj/src/parallel.cpp:84-95); all
// generator arithmetic runs on the device.  There is no CPU fallback: a call
// without a usable CUDA device returns XG_ECUDA.  (The host computes only the
// jump-ahead tables' polynomial algebra -- Berlekamp-Massey over 8192 bits the
// device generated, squarings mod m(x) -- once per parameter set; every word
// is generated on the device.)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <numeric>
#include <thread>
#include <type_traits>
#include <vector>

#include "xg_gpu.h"
#include "xg_digest.cuh"
#include "xg_generic.cuh"
#include "xg_jump.cuh"
#include "xg_kernels.cuh"
#include "xg_pairs.cuh"
#include "xg_stattests.cuh"

using namespace xgk;

namespace {

std::atomic<uint64_t> g_launches{0};

constexpr uint32_t kMask32 = 0xffffffffu;
constexpr uint64_t kNextBuf = 1u << 16;  // words per next_word refill slot
constexpr unsigned kGenMaxR = 16384;   // generic path: r words of state in shared memory

// kGP32 / kRtJ*: register-window kernels (w = 32, r = 128, lane_bound >= 32);
// kGeneric: any other valid set (xg_generic.cuh).
enum Kind { kGP32 = 0, kRtJ1 = 1, kRtJ2 = 2, kGeneric = 3 };

struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// The device that owns a device pointer (entry points without a handle run on
// it, whatever device is current for the calling thread).  Host or
// unregistered pointers are XG_EINVAL.
int ptr_device(const void* p, int* dev) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return XG_EINVAL;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return XG_EINVAL;
    *dev = a.device;
    return XG_OK;
}

}  // namespace

struct xg_ensemble {
    xg_params_t params{};
    Kind kind = kGP32;
    int device = 0;
    uint32_t num_streams = 0;
    uint64_t base_seed = 0, first_stream = 0;
    unsigned lanes = 0;
    int sms = 148;          // multiprocessors of `device` (CTA sizing)
    int smem_per_sm = 0;    // shared memory per SM (occupancy cap of the fills)
    int smem_optin = 0;     // largest dynamic shared memory a CTA may request
    bool pair_smem_ok = false;  // pair kernels accept that much (prepare_pair_kernels)
    uint32_t* d_win = nullptr;   // [num_streams][128] logical window, oldest first
    uint32_t* d_weyl = nullptr;  // [num_streams] Weyl accumulator
    uint64_t* d_win64 = nullptr;   // generic path: [num_streams][r] words, oldest first
    uint64_t* d_weyl64 = nullptr;  // generic path: [num_streams]
    // next_word service (one-stream handles): two refill slots of kNextBuf
    // words in pinned host memory, one being served while the other is
    // generated and copied on a private stream (NextRing in xg_gpu.cu).
    struct NextRing {
        bool active = false;     // slots hold words not yet given back to the device state
        int cur = 0;             // slot being served
        uint64_t pos = 0;        // words of slot `cur` served
        void* host[2] = {};      // pinned
        void* dev[2] = {};       // device staging
        void* snap[2] = {};      // generator state before slot i's words
        cudaStream_t st = nullptr;
        cudaEvent_t ev[2] = {};
    } nr;
    // xg_generate_host staging
    void* d_stage = nullptr;
    size_t stage_words = 0;  // bytes
    // xg_generate_host_rows pinned staging
    void* h_stage = nullptr;
    size_t h_stage_bytes = 0;
    // xg_linear_complexity_test word buffer
    uint32_t* d_lc = nullptr;
    size_t lc_bytes = 0;
    // jump-ahead scratch (one-stream fills, xg_jump.cuh): segment start
    // windows + Weyl words, GF(2) partial products, a side stream for the
    // last (short) segment
    uint32_t* d_jrows = nullptr;
    uint32_t* d_jweyl = nullptr;
    uint32_t* d_jpart = nullptr;
    uint32_t* d_jW = nullptr;    // the 4096 windows W[i] of a raw run (Krylov form)
    uint32_t* d_jseq = nullptr;  // that run: 128 + 4096 words
    uint32_t jrows_cap = 0;
    cudaStream_t jside = nullptr;
    cudaEvent_t jev[2] = {};
};

namespace {

int check_params_impl(const xg_params_t* p) {
    if (!p) return XG_EINVAL;
    if (p->w != 8 && p->w != 16 && p->w != 32 && p->w != 64) return XG_EPARAM_BAD_WORD_SIZE;
    if (p->s == 0 || p->s >= p->r) return XG_EPARAM_S_OUT_OF_RANGE;
    if (std::gcd(p->r, p->s) != 1u) return XG_EPARAM_GCD_NOT_ONE;
    for (unsigned sh : {p->a, p->b, p->c, p->d})
        if (sh == 0 || sh >= p->w) return XG_EPARAM_SHIFT_OUT_OF_RANGE;
    if (p->gamma == 0 || p->gamma >= p->w) return XG_EPARAM_GAMMA_OUT_OF_RANGE;
    if ((p->omega & 1u) == 0) return XG_EPARAM_EVEN_WEYL_INCREMENT;
    return XG_OK;
}

unsigned lane_bound_impl(const xg_params_t* p) {
    return p->s < p->r - p->s ? p->s : p->r - p->s;
}

bool is_gp32(const xg_params_t* p) {
    return p->r == 128 && p->s == 65 && p->a == 15 && p->b == 14 && p->c == 12 &&
           p->d == 17 && p->w == 32 && p->omega == 2654435769ull && p->gamma == 16;
}

int classify(const xg_params_t* p, Kind* kind) {
    int e = check_params_impl(p);
    if (e) return e;
    if (p->w != 32 || p->r != kR || lane_bound_impl(p) < 32) {
        if (p->r > kGenMaxR) return XG_EUNSUPPORTED;
        *kind = kGeneric;
        return XG_OK;
    }
    if (is_gp32(p)) {
        *kind = kGP32;
    } else {
        const unsigned q = p->r - p->s;  // odd, 33..95
        *kind = (q / 32 == 1) ? kRtJ1 : kRtJ2;
    }
    return XG_OK;
}

template <int J>
RtParams<J> rt_params(const xg_params_t& p) {
    RtParams<J> r;
    r.delta = (p.r - p.s) % 32;
    r.a = p.a;
    r.b = p.b;
    r.c = p.c;
    r.d = p.d;
    r.gamma = p.gamma;
    r.omega = static_cast<uint32_t>(p.omega & kMask32);
    return r;
}

int cuda_rc(cudaError_t e) {
    if (e == cudaSuccess) return XG_OK;
    if (e == cudaErrorMemoryAllocation) return XG_ENOMEM;
    return XG_ECUDA;
}

unsigned grid_for(uint32_t n) {
    return static_cast<unsigned>((static_cast<uint64_t>(n) + kWarpsPerBlock - 1) / kWarpsPerBlock);
}

// Kernel choice for the register-window sets: the pair-lane kernel
// (xg_pairs.cuh) wherever it applies (r - s < 64 and aligned output rows),
// else the word-per-lane kernel with the shared-memory s-tap (xg_kernels.cuh).
constexpr int kFillWarpsPerCta = 4;  // u32/raw fills of large ensembles: streams per CTA
constexpr int kFillCtasPerSm = 4;    // ... and resident CTAs per SM (launch_pair)

// The pair-lane kernel stores 8-byte word pairs (16 for the zero-extended
// u64 words): every output row must start on that boundary.
template <int MODE>
bool pair_aligned(const void* out, uint64_t words) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(out);
    if constexpr (MODE == kU32 || MODE == kF32 || MODE == kRaw) return (a & 7u) == 0 && (words & 1u) == 0;
    else if constexpr (MODE == kWide) return (a & 15u) == 0 && (words & 1u) == 0;
    else return true;  // f64 (8-byte values, words even), MC, skip
}

// Output row geometry of a fill: rows come in groups of rg contiguous rows
// (each row `words` words long), the groups ld output elements apart;
// ld = 0 means plain block-major rows (ld = the row length, rg = 1).
template <int MODE>
uint64_t row_ld(uint64_t words, uint64_t ld) {
    return ld ? ld : (MODE == kF64 ? words >> 1 : words);
}

template <int MODE, class P>
int launch_pair(const P& p, xg_ensemble* h, uint32_t g_begin, uint32_t g_count, uint64_t words,
                void* out, unsigned long long* hits, cudaStream_t s, uint64_t ld = 0, uint32_t rg = 1) {
    // Streams (warps) per CTA.  Every stream is the same amount of work, so
    // what matters is how evenly the warps land on the SMs.  Up to 32 streams
    // per SM, launch one CTA per SM holding ceil(P / SMs) streams: the
    // busiest SM carries at most one stream more than the average, and small
    // ensembles use every SM (8-stream CTAs put 64 streams on 8 SMs: 1.32e11
    // against 0.95e11 RN/s; 4096 streams: 1.57e12 against 1.44e12;
    // profiles/ab_r1/README_round1.md, r1p).  Larger ensembles: below.
    const uint64_t sms = static_cast<uint64_t>(std::max(1, h->sms));
    // u32 / raw fills of large ensembles: 4-stream CTAs, at most
    // kFillCtasPerSm = 4 of them resident per SM (16 write streams per SM
    // instead of 64), enforced by reserving shared memory the kernel does not
    // use.  The fill is HBM-bound far below full occupancy (~7 streams
    // saturate an SM's ALU pipe), and fewer concurrent write streams, started
    // in small staggered CTA waves, write faster: 1.596e12 against 1.53e12
    // RN/s under the power cap, 1.737e12 against 1.72e12 in bursts (r1u,
    // r1zg in profiles/ab_r1/README_round1.md).  The conversions gain nothing from the cap
    // and run full (8-stream CTAs, 64 streams per SM).
    constexpr bool kCapped = MODE == kU32 || MODE == kRaw;
    const bool large = g_count > 32 * sms;
    uint32_t wpb = kWarpsPerBlock;
    int cap = 0;
    if (large) {
        if (kCapped) {
            wpb = kFillWarpsPerCta;
            cap = kFillCtasPerSm;
        }
    } else {
        // one CTA per SM holding ceil(P / SMs) streams (see above)
        wpb = static_cast<uint32_t>((g_count + sms - 1) / sms);  // 1..32
        if (!std::is_same_v<P, GP32>) wpb = std::min<uint32_t>(wpb, kWarpsPerBlock);
    }
    size_t smem = 0;
    if (cap > 0 && h->smem_per_sm > 0 && h->pair_smem_ok) {
        // cap CTAs fit, cap + 1 do not (each CTA also reserves 1 KB).  The
        // kernels' dynamic shared memory limit was raised at ensemble
        // creation (prepare_pair_kernels), so nothing here is a
        // non-stream call -- fills capture into CUDA graphs.
        smem = std::min<size_t>(static_cast<size_t>(h->smem_per_sm) / cap - 2048,
                                static_cast<size_t>(h->smem_optin));
    }
    const unsigned grid = static_cast<unsigned>((static_cast<uint64_t>(g_count) + wpb - 1) / wpb);
    pair_kernel<P, MODE><<<grid, 32 * wpb, smem, s>>>(p, h->d_win, h->d_weyl, g_begin, g_count,
                                                      words, out, hits, row_ld<MODE>(words, ld), rg);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

template <int MODE, class P>
int launch_word_lane(const P& p, xg_ensemble* h, uint32_t g_begin, uint32_t g_count,
                     uint64_t words, void* out, unsigned long long* hits, cudaStream_t s,
                     uint64_t ld = 0, uint32_t rg = 1) {
    fill_kernel<P, MODE><<<grid_for(g_count), kThreads, 0, s>>>(p, h->d_win, h->d_weyl, g_begin,
                                                                g_count, words, out, hits,
                                                                row_ld<MODE>(words, ld), rg);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

GenParams gen_params(const xg_params_t& p) {
    GenParams g;
    g.r = p.r; g.s = p.s; g.a = p.a; g.b = p.b; g.c = p.c; g.d = p.d; g.w = p.w;
    g.gamma = p.gamma;
    g.lanes = std::min(32u, lane_bound_impl(&p));
    g.omega = p.omega;
    g.mask = p.w >= 64 ? ~0ull : ((1ull << p.w) - 1);
    return g;
}

size_t gen_smem(const xg_params_t& p) { return static_cast<size_t>(p.r) * sizeof(uint64_t); }

// Dynamic shared-memory limit of `kernel` raised once per device, always to
// the same value (the device's opt-in maximum, or a kernel's fixed maximum), so
// launches make no non-stream driver call and concurrent host threads can
// never lower the limit under one another's launch.
template <class K>
int raise_smem_once(K kernel, size_t bytes, std::atomic<uint64_t>& done) {
    if (bytes <= 48 * 1024) return XG_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return XG_ECUDA;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return XG_OK;
    int rc = cuda_rc(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(bytes)));
    if (!rc) done.fetch_or(bit, std::memory_order_acq_rel);
    return rc;
}

int smem_optin_current() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

// The generic kernels take r words of shared memory; beyond 48 KB (r > 6144)
// their limit is raised once per device to the opt-in maximum.
template <auto Kernel>
int gen_smem_attr(size_t smem) {
    static std::atomic<uint64_t> done{0};  // one flag set per kernel
    if (smem <= 48 * 1024) return XG_OK;
    if (smem > static_cast<size_t>(smem_optin_current())) return XG_EUNSUPPORTED;
    return raise_smem_once(Kernel, static_cast<size_t>(smem_optin_current()), done);
}

template <int GM>
int launch_gen(xg_ensemble* h, uint32_t g_begin, uint32_t g_count, uint64_t words, void* out,
               cudaStream_t s) {
    const size_t smem = gen_smem(h->params);
    int rc = gen_smem_attr<&gen_fill_kernel<GM>>(smem);
    if (rc) return rc;
    gen_fill_kernel<GM><<<g_count, 32, smem, s>>>(gen_params(h->params), h->d_win64, h->d_weyl64,
                                                   g_begin, g_count, words, out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

template <int MODE>
int launch_fill_direct(xg_ensemble* h, uint32_t g_begin, uint32_t g_count, uint64_t words, void* out,
                       unsigned long long* hits, cudaStream_t s, uint64_t ld = 0, uint32_t rg = 1) {
    if (words == 0 || g_count == 0) return XG_OK;
    if (h->kind == kGeneric) {
        // The conversions (f32/f64/u64 pairs) and the MC predicate are defined
        // on 32-bit words; the generic path offers the words themselves.
        const bool narrow = h->params.w <= 32;
        if constexpr (MODE == kU32) {
            if (narrow) return launch_gen<kGenU32>(h, g_begin, g_count, words, out, s);
        } else if constexpr (MODE == kRaw) {
            if (narrow) return launch_gen<kGenRawU32>(h, g_begin, g_count, words, out, s);
        } else if constexpr (MODE == kWide) {
            return launch_gen<kGenWide>(h, g_begin, g_count, words, out, s);
        } else if constexpr (MODE == kSkip) {
            return launch_gen<kGenSkip>(h, g_begin, g_count, words, out, s);
        }
        return XG_EUNSUPPORTED;
    }
    if constexpr (MODE == kRank) {  // pair-lane kernel only (needs r - s < 64)
        if (h->kind == kGP32) return launch_pair<MODE>(GP32{}, h, g_begin, g_count, words, out, hits, s, ld, rg);
        if (h->kind == kRtJ1)
            return launch_pair<MODE>(rt_params<1>(h->params), h, g_begin, g_count, words, out, hits, s, ld, rg);
        return XG_EUNSUPPORTED;
    } else {
        // pair stores need every row start aligned: an odd group stride ld
        // (rows of u32 / u64 words) sends the call to the word-lane kernel
        const bool ld_ok = ld == 0 || MODE == kF64 || (ld & 1u) == 0;
        if (h->kind != kRtJ2 && pair_aligned<MODE>(out, words) && ld_ok) {
            if (h->kind == kGP32) return launch_pair<MODE>(GP32{}, h, g_begin, g_count, words, out, hits, s, ld, rg);
            return launch_pair<MODE>(rt_params<1>(h->params), h, g_begin, g_count, words, out, hits, s, ld, rg);
        }
        switch (h->kind) {
        case kGP32: return launch_word_lane<MODE>(GP32{}, h, g_begin, g_count, words, out, hits, s, ld, rg);
        case kRtJ1: return launch_word_lane<MODE>(rt_params<1>(h->params), h, g_begin, g_count, words, out, hits, s, ld, rg);
        default: return launch_word_lane<MODE>(rt_params<2>(h->params), h, g_begin, g_count, words, out, hits, s, ld, rg);
        }
    }
}

// ---- jump-ahead (xg_jump.cuh) --------------------------------------------
//
// One stream of a register-window set cut into segments: the start window
// of segment k is s0 G^(kJ) (J = 2^j words, G the one-word transition matrix
// over GF(2)), its Weyl word weyl + kJ omega; K segments are then generated
// by one launch of the ordinary kernels as a K-stream ensemble whose rows
// are consecutive pieces of the output.  Powers G^(2^i) are computed once
// per (device, parameter set) by repeated squaring and kept for the process.

constexpr uint64_t kJumpMin = 1ull << 20;  // words: below this one warp is faster
constexpr uint64_t kJumpSkipMany = 1ull << 22;  // skips of more streams than 64: jump from here
constexpr uint64_t kJumpManyMin = 1ull << 18;   // 2 .. 700 streams: segments of >= 2^16 words, >= 2 each
constexpr uint32_t kJumpManyMax = 700;          // from ~760 streams one warp each saturates HBM
constexpr unsigned kJumpMinLog = 16;       // segments of at least 2^16 words
#ifndef XG_JUMP_MAX_SEG
#define XG_JUMP_MAX_SEG 1024
#endif
constexpr uint32_t kJumpMaxSeg = XG_JUMP_MAX_SEG;  // ... and at most 1024 of them (A/B: 512 / 1024 / 2048)
constexpr uint32_t kJCoeffRows = kJumpMaxSeg + 1;  // K full segments + a short last one
constexpr size_t kJRowBytes = kJWords * sizeof(uint32_t);
constexpr uint32_t kJPartRows = 16 * 4096;  // partial rows of the largest product (see gf2_mul)

struct JumpPowers {
    xg_params_t p{};
    int device = 0;
    std::vector<uint32_t*> pow;  // pow[i] = G^(2^i): 4096 rows of 128 words on `device`
    std::vector<cudaEvent_t> ready;
    uint32_t* part = nullptr;    // partials scratch of the squarings
    // Krylov form: m(x) = the minimal polynomial of G (degree 4096, found by
    // Berlekamp-Massey), and per segment length 2^j the rows
    // C[k] = x^(k 2^j) mod m(x), k < kJCoeffRows, so that the window kJ
    // words ahead of s_0 is C[k] W with W[i] = the window i raw words ahead.
    int poly = 0;                // 0 not tried, 1 m(x) known, -1 unavailable
    std::vector<uint64_t> mlow;  // m(x) - x^4096: 64 words, bit k = coefficient of x^k
    struct Coeffs {
        unsigned j = 0;
        uint32_t* rows = nullptr;
        cudaEvent_t ready = nullptr;
        bool done = false;  // `ready` seen complete: later calls need no wait
    };
    std::vector<Coeffs> coeffs;
    std::mutex mu;
};

std::mutex g_jump_mu;
std::vector<std::unique_ptr<JumpPowers>> g_jump;  // process lifetime

bool same_params(const xg_params_t& a, const xg_params_t& b) {
    return a.r == b.r && a.s == b.s && a.a == b.a && a.b == b.b && a.c == b.c && a.d == b.d &&
           a.w == b.w && a.omega == b.omega && a.gamma == b.gamma;
}

JumpPowers* jump_powers(const xg_ensemble* h) {
    std::lock_guard<std::mutex> lk(g_jump_mu);
    for (auto& j : g_jump)
        if (j->device == h->device && same_params(j->p, h->params)) return j.get();
    g_jump.push_back(std::make_unique<JumpPowers>());
    g_jump.back()->p = h->params;
    g_jump.back()->device = h->device;
    // pow[i] is read without the lock once jump_ensure has returned: never
    // reallocate (i < 64 always)
    g_jump.back()->pow.reserve(64);
    g_jump.back()->ready.reserve(64);
    return g_jump.back().get();
}

// G on the host: row i = the window after one raw step from the unit window
// e_i (bit i % 32 of word i / 32): v = T1(W[0]) ^ T2(W[r - s]), W' = W[1..]
// ++ v (proj/include/xg/xorgens.hpp:13-18,39-47).
std::vector<uint32_t> transition_matrix(const xg_params_t& p) {
    auto xs = [](uint32_t x, unsigned l, unsigned r) {
        const uint32_t t = x ^ (x << l);
        return t ^ (t >> r);
    };
    const unsigned q = p.r - p.s;
    std::vector<uint32_t> g(static_cast<size_t>(4096) * kJWords, 0u);
    for (unsigned i = 0; i < 4096; ++i) {
        const unsigned j = i / 32;
        const uint32_t e = 1u << (i % 32);
        uint32_t* row = g.data() + static_cast<size_t>(i) * kJWords;
        if (j > 0) row[j - 1] ^= e;
        if (j == 0) row[kJWords - 1] ^= xs(e, p.a, p.b);
        if (j == q) row[kJWords - 1] ^= xs(e, p.c, p.d);
    }
    return g;
}

// C = A B over GF(2) (A: rows x 4096, B: 4096 x 4096, row-vector convention);
// `part` holds ksplit * rows partial rows (<= kJPartRows).
int gf2_mul(const uint32_t* A, uint32_t rows, const uint32_t* B, uint32_t* C, uint32_t* part,
            cudaStream_t s, uint32_t ldb = kJWords) {
    if (rows == 0) return XG_OK;
    if (ldb != kJWords && rows < 256) return XG_EINVAL;  // strided B: four-Russians kernel only
    // k-split: as many ranges as the partials buffer holds (64 up to 512
    // rows, 8 at 4096); rows per warp: 8 for large products, fewer for the
    // small ones so that their rows spread over more warps.
    uint32_t ksplit = 64;
    while (ksplit > 8 && static_cast<uint64_t>(ksplit) * rows > kJPartRows) ksplit >>= 1;
    const uint32_t kspan = 4096u / ksplit;
    auto launch = [&](auto kernel, uint32_t rw) {
        const dim3 grid((rows + 8 * rw - 1) / (8 * rw), ksplit);
        kernel<<<grid, 256, 0, s>>>(A, B, part, rows, kspan);
    };
    if (rows >= 256) {  // many rows: tables pay for themselves
        ksplit = 4096u / kM4Span;  // the staged span of B; 16 x 4096 partial rows at most
#ifndef XG_M4RM_RW
#define XG_M4RM_RW 16
#endif
        constexpr int RW = XG_M4RM_RW;  // rows per warp: 8 RW rows share each CTA's tables
        const dim3 grid(4, (rows + 8 * RW - 1) / (8 * RW), ksplit);
        static std::atomic<uint64_t> done{0};
        const int rc = raise_smem_once(gf2_mul_m4rm_kernel<RW>, kM4Smem, done);
        if (rc) return rc;
        gf2_mul_m4rm_kernel<RW><<<grid, 256, kM4Smem, s>>>(A, B, part, rows, 4096u / ksplit, ldb);
    } else if (rows >= 64) {
        launch(gf2_mul_partial_kernel<2>, 2);
    } else {
        launch(gf2_mul_partial_kernel<1>, 1);
    }
    const uint64_t n16 = static_cast<uint64_t>(rows) * (kJWords / 4);
    gf2_reduce_kernel<<<static_cast<unsigned>((n16 + 255) / 256), 256, 0, s>>>(part, C, rows, ksplit);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

// Make G^(2^i) available for i <= upto (squarings on `s`, once per process)
// and order `s` after their computation.
int jump_ensure(JumpPowers* jp, unsigned upto, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(jp->mu);
    int rc = XG_OK;
    if (jp->pow.empty()) {
        const std::vector<uint32_t> g = transition_matrix(jp->p);
        uint32_t* d = nullptr;
        rc = cuda_rc(cudaMalloc(&d, g.size() * sizeof(uint32_t)));
        if (!rc) rc = cuda_rc(cudaMemcpy(d, g.data(), g.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
        if (!rc && !jp->part) rc = cuda_rc(cudaMalloc(&jp->part, static_cast<size_t>(kJPartRows) * kJRowBytes));
        cudaEvent_t ev = nullptr;
        if (!rc) rc = cuda_rc(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        if (!rc) rc = cuda_rc(cudaEventRecord(ev, s));
        if (rc) {
            cudaFree(d);
            return rc;
        }
        jp->pow.push_back(d);
        jp->ready.push_back(ev);
    }
    while (jp->pow.size() <= upto) {
        uint32_t* d = nullptr;
        rc = cuda_rc(cudaMalloc(&d, static_cast<size_t>(4096) * kJRowBytes));
        if (rc) return rc;
        cudaStreamWaitEvent(s, jp->ready.back(), 0);
        rc = gf2_mul(jp->pow.back(), 4096, jp->pow.back(), d, jp->part, s);
        cudaEvent_t ev = nullptr;
        if (!rc) rc = cuda_rc(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        if (!rc) rc = cuda_rc(cudaEventRecord(ev, s));
        if (rc) {
            cudaFree(d);
            return rc;
        }
        jp->pow.push_back(d);
        jp->ready.push_back(ev);
    }
    // squarings share jp->part: order this stream after the newest one
    return cuda_rc(cudaStreamWaitEvent(s, jp->ready.back(), 0));
}

int jump_scratch(xg_ensemble* h, uint32_t rows) {
    int rc = XG_OK;
    if (h->jrows_cap < rows) {
        cudaFree(h->d_jrows);
        cudaFree(h->d_jweyl);
        h->d_jrows = nullptr;
        h->d_jweyl = nullptr;
        h->jrows_cap = 0;
        rc = cuda_rc(cudaMalloc(&h->d_jrows, static_cast<size_t>(rows) * kJRowBytes));
        if (!rc) rc = cuda_rc(cudaMalloc(&h->d_jweyl, static_cast<size_t>(rows) * sizeof(uint32_t)));
        if (rc) return rc;
        h->jrows_cap = rows;
    }
    // partial rows of a product of at most kJCoeffRows rows (16 k-ranges)
    if (!h->d_jpart) rc = cuda_rc(cudaMalloc(&h->d_jpart, static_cast<size_t>(16) * kJCoeffRows * kJRowBytes));
    if (!rc && !h->d_jW) rc = cuda_rc(cudaMalloc(&h->d_jW, static_cast<size_t>(4096) * kJRowBytes));
    if (!rc && !h->d_jseq) rc = cuda_rc(cudaMalloc(&h->d_jseq, (2 * kJWords + 4096) * sizeof(uint32_t)));
    if (!rc && !h->jside) rc = cuda_rc(cudaStreamCreateWithFlags(&h->jside, cudaStreamNonBlocking));
    for (int i = 0; i < 2 && !rc; ++i)
        if (!h->jev[i]) rc = cuda_rc(cudaEventCreateWithFlags(&h->jev[i], cudaEventDisableTiming));
    return rc;
}

unsigned ceil_log2(uint64_t x) {
    unsigned l = 0;
    while ((1ull << l) < x) ++l;
    return l;
}

// Streams [g, g + count) advanced by `words` (skip: no output) in
// O(log words) products: the windows (rows) times the cached G^(2^i) over the
// set bits of `words`, in chunks of kJumpMaxSeg rows; Weyl + words omega.
int jump_skip(xg_ensemble* h, uint32_t g, uint32_t count, uint64_t words, cudaStream_t s) {
    JumpPowers* jp = jump_powers(h);
    int rc = jump_ensure(jp, 63 - static_cast<unsigned>(__builtin_clzll(words)), s);
    if (!rc) rc = jump_scratch(h, std::min<uint32_t>(count, kJumpMaxSeg));
    for (uint32_t c0 = 0; c0 < count && !rc; c0 += kJumpMaxSeg) {
        const uint32_t n = std::min<uint32_t>(kJumpMaxSeg, count - c0);
        uint32_t* win = h->d_win + static_cast<size_t>(g + c0) * kJWords;
        uint32_t* a = win;  // ping-pong between the state rows and the scratch
        uint32_t* b = h->d_jrows;
        for (unsigned i = 0; i < 64 && !rc; ++i) {
            if (!((words >> i) & 1u)) continue;
            rc = gf2_mul(a, n, jp->pow[i], b, h->d_jpart, s);
            std::swap(a, b);
        }
        if (!rc && a != win)
            rc = cuda_rc(cudaMemcpyAsync(win, a, static_cast<size_t>(n) * kJRowBytes, cudaMemcpyDeviceToDevice, s));
    }
    if (rc) return rc;
    // weyl += words * omega (mod 2^32) for every stream, on the device
    const uint32_t step = static_cast<uint32_t>(words * (h->params.omega & kMask32));
    jump_weyl_add_kernel<<<(count + 255) / 256, 256, 0, s>>>(h->d_weyl + g, count, step);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

// ---- Krylov form of the jump (one product per call) ----------------------

constexpr unsigned kPolyWords = 64;                // 4096-bit polynomials as uint64

// The raw (Weyl-free) words of a register-window set from `window`, on the
// host: x_k = T1(W[0]) ^ T2(W[r - s]), W shifts by one (xorgens.hpp:39-47).
// Only the host-only analysis call xg_jump_minpoly uses it; the jump path
// takes the same words from the device (find_minpoly).
void host_raw_words(const xg_params_t& p, std::vector<uint32_t> window, size_t n, uint32_t* out) {
    auto xs = [](uint32_t x, unsigned l, unsigned r) {
        const uint32_t t = x ^ (x << l);
        return t ^ (t >> r);
    };
    const unsigned q = p.r - p.s;
    std::vector<uint32_t> w(window.begin(), window.end());
    w.reserve(window.size() + n);
    for (size_t k = 0; k < n; ++k) {
        const uint32_t v = xs(w[k], p.a, p.b) ^ xs(w[k + q], p.c, p.d);
        w.push_back(v);
        out[k] = v;
    }
}

// Berlekamp-Massey over GF(2): the shortest connection polynomial c
// (c[0] = 1, b_n = XOR_{i=1..L} c_i b_{n-i}) of the bit sequence; returns L.
// Bit-packed: the discrepancy at step i is the parity of C AND (the sequence
// reversed, shifted so bit k lines up with b_{i-k}) -- one multiword shift
// and AND per step (8192 bits: ~1 ms).
unsigned berlekamp_massey_bits(const std::vector<uint8_t>& b, std::vector<uint8_t>& c) {
    const size_t n = b.size(), nw = (n + 1 + 63) / 64 + 1;
    std::vector<uint64_t> rev(nw, 0), C(nw, 0), B(nw, 0), T(nw, 0), t(nw, 0);
    for (size_t j = 0; j < n; ++j)  // rev bit j = b_{n-1-j}
        if (b[n - 1 - j]) rev[j / 64] |= 1ull << (j % 64);
    auto shr = [&](const std::vector<uint64_t>& x, size_t sh, std::vector<uint64_t>& out) {
        const size_t ws = sh / 64, bs = sh % 64;
        for (size_t w = 0; w < nw; ++w) {
            const size_t src = w + ws;
            uint64_t v = src < nw ? x[src] >> bs : 0;
            if (bs && src + 1 < nw) v |= x[src + 1] << (64 - bs);
            out[w] = v;
        }
    };
    auto xor_shl = [&](std::vector<uint64_t>& x, const std::vector<uint64_t>& y, size_t sh) {  // x ^= y << sh
        const size_t ws = sh / 64, bs = sh % 64;
        for (size_t w = nw; w-- > ws;) {
            const size_t src = w - ws;
            uint64_t v = y[src] << bs;
            if (bs && src > 0) v |= y[src - 1] >> (64 - bs);
            x[w] ^= v;
        }
    };
    C[0] = B[0] = 1;
    unsigned L = 0;
    size_t m = 1;
    for (size_t i = 0; i < n; ++i) {
        shr(rev, n - 1 - i, t);  // t bit k = b_{i-k} (k <= i), 0 beyond
        uint64_t acc = 0;
        for (size_t w = 0; w <= L / 64 && w < nw; ++w) acc ^= C[w] & t[w];
        const unsigned d = __builtin_popcountll(acc) & 1u;
        if (!d) {
            ++m;
        } else if (2 * L <= i) {
            T = C;
            xor_shl(C, B, m);
            L = static_cast<unsigned>(i + 1 - L);
            B = T;
            m = 1;
        } else {
            xor_shl(C, B, m);
            ++m;
        }
    }
    c.assign(n + 1, 0);
    for (size_t k = 0; k <= n; ++k) c[k] = static_cast<uint8_t>((C[k / 64] >> (k % 64)) & 1u);
    return L;
}

// a <- a x mod m (a: 64 words, degree < 4096)
void poly_mulx(std::vector<uint64_t>& a, const std::vector<uint64_t>& mlow) {
    const uint64_t top = a[kPolyWords - 1] >> 63;
    for (unsigned i = kPolyWords - 1; i > 0; --i) a[i] = (a[i] << 1) | (a[i - 1] >> 63);
    a[0] <<= 1;
    if (top)
        for (unsigned i = 0; i < kPolyWords; ++i) a[i] ^= mlow[i];
}

// a <- a^2 mod m: spread the bits (no cross terms over GF(2)), then fold every
// x^i, i >= 4096, as x^(i-4096) (m(x) - x^4096), highest first.
void poly_sqr(std::vector<uint64_t>& a, const std::vector<uint64_t>& mlow) {
    std::vector<uint64_t> t(2 * kPolyWords, 0);
    for (unsigned i = 0; i < kPolyWords; ++i)
        for (unsigned b = 0; b < 64; ++b)
            if ((a[i] >> b) & 1u) t[(2 * (64 * i + b)) / 64] |= 1ull << ((2 * b) % 64);
    for (unsigned i = 2 * 4096 - 1; i >= 4096; --i) {
        if (!((t[i / 64] >> (i % 64)) & 1u)) continue;
        t[i / 64] ^= 1ull << (i % 64);
        const unsigned sh = i - 4096, w = sh / 64, o = sh % 64;
        for (unsigned k = 0; k < kPolyWords; ++k) {
            t[w + k] ^= mlow[k] << o;
            if (o) t[w + k + 1] ^= mlow[k] >> (64 - o);
        }
    }
    a.assign(t.begin(), t.begin() + kPolyWords);
}

// Find m(x) once per parameter set: Berlekamp-Massey on bit 0 of 8192 raw
// words, degree 4096 required (then m is G's minimal AND characteristic
// polynomial, so it annihilates every state), checked on two windows.
// `raw(window, n, out)` produces the n raw (Weyl-free) words that follow a
// 128-word window: on the device for the jump path (find_minpoly), on the
// host only for the xg_jump_minpoly analysis call.
template <class Raw>
int minpoly_of(Raw raw, std::vector<uint64_t>& mlow, bool* ok) {
    *ok = false;
    std::vector<uint32_t> w0(kJWords);
    for (unsigned i = 0; i < kJWords; ++i) w0[i] = 0x9e3779b9u * (i + 1) ^ (i << 7);
    std::vector<uint32_t> x(2 * 4096);
    int rc = raw(w0, x.size(), x.data());
    if (rc) return rc;
    std::vector<uint8_t> bits(x.size()), c;
    for (size_t i = 0; i < x.size(); ++i) bits[i] = x[i] & 1u;
    const unsigned L = berlekamp_massey_bits(bits, c);
    if (L != 4096) return XG_OK;
    mlow.assign(kPolyWords, 0);
    for (unsigned k = 0; k < 4096; ++k)  // m_k = c_(L-k)
        if (c[L - k]) mlow[k / 64] |= 1ull << (k % 64);
    // check s_4096 = XOR_(k < 4096, m_k = 1) s_k on two windows
    for (int trial = 0; trial < 2; ++trial) {
        std::vector<uint32_t> win(kJWords);
        for (unsigned i = 0; i < kJWords; ++i) win[i] = trial ? (i * 2654435761u + 12345u) : w0[i];
        std::vector<uint32_t> seq(win), more(4096);
        rc = raw(win, more.size(), more.data());
        if (rc) return rc;
        seq.insert(seq.end(), more.begin(), more.end());  // seq[i .. i + 128) = s_i
        std::vector<uint32_t> acc(kJWords, 0);
        for (unsigned k = 0; k < 4096; ++k)
            if ((mlow[k / 64] >> (k % 64)) & 1u)
                for (unsigned j = 0; j < kJWords; ++j) acc[j] ^= seq[k + j];
        for (unsigned j = 0; j < kJWords; ++j)
            if (acc[j] != seq[4096 + j]) return XG_OK;
    }
    *ok = true;
    return XG_OK;
}

// m(x) of the handle's parameter set from raw words generated on the device
// (a one-stream view over scratch: 128-word state slot + output), on `s`.
int find_minpoly(JumpPowers* jp, xg_ensemble* h, cudaStream_t s, bool* ok) {
    uint32_t* d = nullptr;  // [128 state][8192 output][1 weyl]
    int rc = cuda_rc(cudaMalloc(&d, (kJWords + 2 * 4096 + 1) * sizeof(uint32_t)));
    if (rc) return rc;
    auto raw = [&](const std::vector<uint32_t>& window, size_t n, uint32_t* out) {
        xg_ensemble gen = *h;
        gen.d_win = d;
        gen.d_weyl = d + kJWords + 2 * 4096;  // read, not advanced, by a raw fill
        gen.num_streams = 1;
        int e = cuda_rc(cudaMemcpyAsync(d, window.data(), kJRowBytes, cudaMemcpyHostToDevice, s));
        if (!e) e = launch_fill_direct<kRaw>(&gen, 0, 1, n, d + kJWords, nullptr, s);
        if (!e) e = cuda_rc(cudaMemcpyAsync(out, d + kJWords, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        if (!e) e = cuda_rc(cudaStreamSynchronize(s));
        return e;
    };
    rc = minpoly_of(raw, jp->mlow, ok);
    cudaFree(d);
    return rc;
}

// The matrix of "multiply by p(x) mod m": row i = x^i p mod m, as 4096
// GF(2) rows of 128 u32 words (bit k = coefficient of x^k).
void mul_matrix(const std::vector<uint64_t>& p, const std::vector<uint64_t>& mlow, std::vector<uint32_t>& rows) {
    rows.resize(static_cast<size_t>(4096) * kJWords);
    std::vector<uint64_t> a(p);
    for (unsigned i = 0; i < 4096; ++i) {
        std::memcpy(rows.data() + static_cast<size_t>(i) * kJWords, a.data(), kJRowBytes);
        poly_mulx(a, mlow);
    }
}

// C rows for segment length 2^j (once per parameter set and j): C[0] = 1,
// C[2^l .. 2^(l+1)) = C[0 .. 2^l) (x^(2^(j+l)) mod m) by products with the
// multiplication matrices, on `s`.  Called with jp->mu held.
int build_coeffs(JumpPowers* jp, unsigned j, cudaStream_t s, uint32_t** out) {
    for (auto& c : jp->coeffs)
        if (c.j == j) {
            *out = c.rows;
            if (!c.done) {
                c.done = cudaEventQuery(c.ready) == cudaSuccess;
                if (!c.done) cudaGetLastError();  // cudaErrorNotReady is not a failure
            }
            return c.done ? XG_OK : cuda_rc(cudaStreamWaitEvent(s, c.ready, 0));
        }
    JumpPowers::Coeffs c;
    c.j = j;
    int rc = cuda_rc(cudaMalloc(&c.rows, static_cast<size_t>(kJCoeffRows) * kJRowBytes));
    uint32_t* dmat = nullptr;
    if (!rc) rc = cuda_rc(cudaMalloc(&dmat, static_cast<size_t>(4096) * kJRowBytes));
    uint32_t* part = nullptr;  // own partials: squarings may be running on another stream
    if (!rc) rc = cuda_rc(cudaMalloc(&part, static_cast<size_t>(kJPartRows) * kJRowBytes));
    std::vector<uint32_t> one(kJWords, 0);
    one[0] = 1u;
    if (!rc) rc = cuda_rc(cudaMemcpyAsync(c.rows, one.data(), kJRowBytes, cudaMemcpyHostToDevice, s));
    std::vector<uint64_t> p(kPolyWords, 0);
    p[0] = 2u;  // x
    for (unsigned i = 0; i < j; ++i) poly_sqr(p, jp->mlow);  // x^(2^j)
    std::vector<uint32_t> rows;
    for (unsigned l = 0; !rc && (1u << l) < kJCoeffRows; ++l) {
        mul_matrix(p, jp->mlow, rows);
        // synchronous upload: the previous level's product must be done with dmat
        rc = cuda_rc(cudaStreamSynchronize(s));
        if (!rc) rc = cuda_rc(cudaMemcpy(dmat, rows.data(), rows.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
        const uint32_t have = 1u << l, n = std::min(have, kJCoeffRows - have);
        if (!rc) rc = gf2_mul(c.rows, n, dmat, c.rows + static_cast<size_t>(have) * kJWords, part, s);
        poly_sqr(p, jp->mlow);
    }
    if (!rc) rc = cuda_rc(cudaStreamSynchronize(s));
    cudaFree(dmat);
    cudaFree(part);
    if (!rc) rc = cuda_rc(cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming));
    if (!rc) rc = cuda_rc(cudaEventRecord(c.ready, s));
    if (rc) {
        cudaFree(c.rows);
        return rc;
    }
    jp->coeffs.push_back(c);
    *out = c.rows;
    return XG_OK;
}

// The C rows for 2^j-word segments of this parameter set, or nullptr when
// the set has no degree-4096 minimal polynomial (the doubling path then).
int jump_coeffs(JumpPowers* jp, xg_ensemble* h, unsigned j, cudaStream_t s, uint32_t** out) {
    std::lock_guard<std::mutex> lk(jp->mu);
    *out = nullptr;
    if (jp->poly == 0) {
        bool ok = false;
        const int rc = find_minpoly(jp, h, s, &ok);
        if (rc) return rc;
        jp->poly = ok ? 1 : -1;
    }
    if (jp->poly < 0) return XG_OK;
    return build_coeffs(jp, j, s, out);
}

// Element offset of word `k` of a stream's output for MODE.
template <int MODE>
void* out_at(void* out, uint64_t k) {
    if constexpr (MODE == kU32 || MODE == kRaw || MODE == kF32) return static_cast<uint32_t*>(out) + k;
    else if constexpr (MODE == kWide) return static_cast<uint64_t*>(out) + k;
    else if constexpr (MODE == kF64) return static_cast<double*>(out) + k / 2;
    else return out;
}

// Stream g, `words` words, generated as K segments of J = 2^j words (plus a
// shorter last one on a side stream), continuing stream g exactly.
template <int MODE>
int jump_fill(xg_ensemble* h, uint32_t g, uint64_t words, void* out, unsigned long long* hits,
              cudaStream_t s) {
    if constexpr (MODE == kSkip) {
        return jump_skip(h, g, 1, words, s);
    } else {
        const unsigned j = std::max(kJumpMinLog, ceil_log2((words + kJumpMaxSeg - 1) / kJumpMaxSeg));
        const uint64_t J = 1ull << j;
        const uint32_t K = static_cast<uint32_t>(words >> j);
        const uint64_t rem = words - static_cast<uint64_t>(K) * J;
        const uint32_t cnt = K + (rem ? 1u : 0u);
        const unsigned levels = ceil_log2(cnt);
        JumpPowers* jp = jump_powers(h);
        uint32_t* coeffs = nullptr;
        int rc = jump_coeffs(jp, h, j, s, &coeffs);
        if (!rc) rc = jump_scratch(h, cnt);
        if (rc) return rc;
        uint32_t* win = h->d_win + static_cast<size_t>(g) * kJWords;
        // Raw (Weyl-ablated) fills leave the accumulator alone.
        const uint32_t step = MODE == kRaw ? 0u : static_cast<uint32_t>(J * (h->params.omega & kMask32));
        const uint32_t nb = (std::max<uint32_t>(cnt, kJWords) + 255) / 256;
        if (coeffs) {
            // Krylov form, one product: S[k] = C[k] W, W[i] = the window i raw
            // words ahead of s_0 = seq[i .. i + 128) of a 4096-word raw run
            // (s_0 also seeds the raw run's own state slot, seq + 128 + 4096).
            jump_begin_kernel<<<nb, 256, 0, s>>>(win, h->d_weyl + g, h->d_jseq, h->d_jseq + kJWords + 4096,
                                                 h->d_jweyl, cnt, step);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            rc = cuda_rc(cudaGetLastError());
            xg_ensemble gen = *h;  // a one-stream view over the copy of s_0
            gen.d_win = h->d_jseq + kJWords + 4096;
            gen.d_weyl = h->d_jweyl;  // read, not advanced, by a raw fill
            gen.num_streams = 1;
            if (!rc) rc = launch_fill_direct<kRaw>(&gen, 0, 1, 4096, h->d_jseq + kJWords, nullptr, s);
            if (!rc && cnt >= 256) {  // the four-Russians kernel reads the windows in place
                rc = gf2_mul(coeffs, cnt, h->d_jseq, h->d_jrows, h->d_jpart, s, 1);
            } else if (!rc) {
                jump_windows_kernel<<<4096 * kJWords / 256, 256, 0, s>>>(h->d_jseq, h->d_jW);
                g_launches.fetch_add(1, std::memory_order_relaxed);
                rc = cuda_rc(cudaGetLastError());
                if (!rc) rc = gf2_mul(coeffs, cnt, h->d_jW, h->d_jrows, h->d_jpart, s);
            }
        } else {
            // doubling: rows [2^l, 2^(l+1)) = rows [0, 2^l) G^(J 2^l)
            rc = jump_ensure(jp, j + (levels ? levels - 1 : 0), s);
            if (!rc) {
                jump_begin_kernel<<<nb, 256, 0, s>>>(win, h->d_weyl + g, h->d_jrows, nullptr, h->d_jweyl, cnt,
                                                     step);
                g_launches.fetch_add(1, std::memory_order_relaxed);
                rc = cuda_rc(cudaGetLastError());
            }
            for (unsigned l = 0; l < levels && !rc; ++l) {
                const uint32_t have = 1u << l;
                const uint32_t n = std::min(have, cnt - have);
                rc = gf2_mul(h->d_jrows, n, jp->pow[j + l], h->d_jrows + static_cast<size_t>(have) * kJWords,
                             h->d_jpart, s);
            }
        }
        if (rc) return rc;
        // the segments as an ensemble of cnt streams over the scratch state
        xg_ensemble view = *h;
        view.d_win = h->d_jrows;
        view.d_weyl = h->d_jweyl;
        view.num_streams = cnt;
        if (rem) {  // the short last segment concurrently on the side stream
            rc = cuda_rc(cudaEventRecord(h->jev[0], s));
            if (!rc) rc = cuda_rc(cudaStreamWaitEvent(h->jside, h->jev[0], 0));
            if (!rc)
                rc = launch_fill_direct<MODE>(&view, K, 1, rem, out_at<MODE>(out, static_cast<uint64_t>(K) * J),
                                              hits, h->jside);
            if (!rc) rc = cuda_rc(cudaEventRecord(h->jev[1], h->jside));
        }
        if (!rc && K) rc = launch_fill_direct<MODE>(&view, 0, K, J, out, hits, s);
        if (!rc && rem) rc = cuda_rc(cudaStreamWaitEvent(s, h->jev[1], 0));
        if (rc) return rc;
        // stream g continues from the end of the last segment
        jump_end_kernel<<<1, kJWords, 0, s>>>(h->d_jrows + static_cast<size_t>(cnt - 1) * kJWords,
                                              h->d_jweyl + cnt - 1, win, h->d_weyl + g);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cuda_rc(cudaGetLastError());
    }
}

// 2 .. 700 streams, any length >= 2^18: every stream cut into Q segments of
// J = 2^j words (P Q <= max(kJumpMaxSeg, 2 P); Q = words / J, so the remainder
// rem = words - Q J < J), the start windows of all P (Q + 1) segments by
// doubling over q with the cached powers -- every stream of a level in one
// product, rows q-major -- then ONE fill of the P Q full segments (rows
// g-major; output row (g, q) at g ld + q J: groups of Q rows, ld apart) and,
// concurrently on the side stream, one of the P remainders.
template <int MODE>
int jump_fill_many(xg_ensemble* h, uint32_t g0, uint32_t P, uint64_t words, void* out,
                   unsigned long long* hits, cudaStream_t s) {
    // P Q <= kJumpMaxSeg segments; 513 .. 700 streams still get Q = 2 (up to
    // ~1400 segments: fewer than ~760 warps leave the fill below the HBM rate)
    const uint64_t qmax = std::max<uint64_t>(2, kJumpMaxSeg / P);
    unsigned j = kJumpMinLog;
    while ((words >> j) > qmax) ++j;
    const uint64_t J = 1ull << j;
    const uint32_t Q = static_cast<uint32_t>(words >> j);
    const uint64_t rem = words - static_cast<uint64_t>(Q) * J;
    if (Q < 2) return launch_fill_direct<MODE>(h, g0, P, words, out, hits, s);
    const uint32_t cq = Q + (rem ? 1u : 0u);  // segment starts per stream
    const unsigned lq = ceil_log2(cq);
    JumpPowers* jp = jump_powers(h);
    int rc = jump_ensure(jp, j + lq - 1, s);
    if (!rc) rc = jump_scratch(h, P * cq);
    if (rc) return rc;
    rc = cuda_rc(cudaMemcpyAsync(h->d_jrows, h->d_win + static_cast<size_t>(g0) * kJWords,
                                 static_cast<size_t>(P) * kJRowBytes, cudaMemcpyDeviceToDevice, s));
    for (unsigned l = 0; l < lq && !rc; ++l) {  // rows [P 2^l, ..) = rows [0, ..) G^(J 2^l), q-major
        const uint32_t have = P << l;
        const uint32_t n = std::min(have, P * cq - have);
        rc = gf2_mul(h->d_jrows, n, jp->pow[j + l], h->d_jrows + static_cast<size_t>(have) * kJWords,
                     h->d_jpart, s);
    }
    if (rc) return rc;
    const uint32_t step = MODE == kRaw ? 0u : static_cast<uint32_t>(J * (h->params.omega & kMask32));
    jump_permute_kernel<<<(P * cq * 32 + 255) / 256, 256, 0, s>>>(h->d_jrows, h->d_jW, h->d_weyl + g0,
                                                                h->d_jweyl, P, Q, cq, step);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    rc = cuda_rc(cudaGetLastError());
    xg_ensemble view = *h;
    view.d_win = h->d_jW;
    view.d_weyl = h->d_jweyl;
    view.num_streams = P * cq;
    const uint64_t ld = row_ld<MODE>(words, 0);  // output elements per stream row
    if (!rc && rem) {  // the P remainders (rows P Q + g) concurrently on the side stream
        rc = cuda_rc(cudaEventRecord(h->jev[0], s));
        if (!rc) rc = cuda_rc(cudaStreamWaitEvent(h->jside, h->jev[0], 0));
        if (!rc)
            rc = launch_fill_direct<MODE>(&view, P * Q, P, rem, out_at<MODE>(out, static_cast<uint64_t>(Q) * J),
                                          hits, h->jside, ld, 1);
        if (!rc) rc = cuda_rc(cudaEventRecord(h->jev[1], h->jside));
    }
    if (!rc) rc = launch_fill_direct<MODE>(&view, 0, P * Q, J, out, hits, s, ld, Q);
    if (!rc && rem) rc = cuda_rc(cudaStreamWaitEvent(s, h->jev[1], 0));
    if (rc) return rc;
    jump_finish_many_kernel<<<(P * 32 + 255) / 256, 256, 0, s>>>(h->d_jW, h->d_jweyl,
                                                                 h->d_win + static_cast<size_t>(g0) * kJWords,
                                                                 h->d_weyl + g0, P, Q, rem != 0);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

// Every generation call goes through here; the jump-ahead paths where one
// warp per stream would leave the GPU idle (xg_jump.cuh), else the kernels
// directly:
//   skip of >= 2^20 words (more than 64 streams: >= 2^22)     -> jump_skip, O(log n)
//   one stream, >= 2^20 words                                  -> jump_fill (Krylov)
//   2 .. 700 streams, >= 2^18 words                            -> jump_fill_many
template <int MODE>
int launch_fill(xg_ensemble* h, uint32_t g_begin, uint32_t g_count, uint64_t words, void* out,
                unsigned long long* hits, cudaStream_t s) {
    if (h->kind == kGeneric || words < kJumpManyMin || g_count == 0)
        return launch_fill_direct<MODE>(h, g_begin, g_count, words, out, hits, s);
    if constexpr (MODE == kSkip) {
        if (words >= kJumpMin && (g_count <= 64 || words >= kJumpSkipMany))
            return jump_skip(h, g_begin, g_count, words, s);
    } else {
        if (g_count == 1) {
            if (words >= kJumpMin) return jump_fill<MODE>(h, g_begin, words, out, hits, s);
        } else if (g_count <= kJumpManyMax) {
            return jump_fill_many<MODE>(h, g_begin, g_count, words, out, hits, s);
        }
    }
    return launch_fill_direct<MODE>(h, g_begin, g_count, words, out, hits, s);
}

// Raise the dynamic shared-memory limit of the pair kernels once, at
// ensemble creation (a function attribute, not a stream operation), so the
// occupancy cap of launch_pair needs no driver call at launch time.
template <class P>
bool prepare_pair_kernels_for(int bytes) {
    auto set = [bytes](auto kernel) {
        return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) ==
               cudaSuccess;
    };
    bool ok = set(pair_kernel<P, kU32>) && set(pair_kernel<P, kRaw>) && set(pair_kernel<P, kF32>) &&
              set(pair_kernel<P, kF64>) && set(pair_kernel<P, kWide>);
    return ok;
}

void prepare_pair_kernels(xg_ensemble* h) {
    cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->device);
    cudaDeviceGetAttribute(&h->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device);
    cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
    if (h->smem_optin <= 0) return;
    if (h->kind == kGP32) h->pair_smem_ok = prepare_pair_kernels_for<GP32>(h->smem_optin);
    else if (h->kind == kRtJ1) h->pair_smem_ok = prepare_pair_kernels_for<RtParams<1>>(h->smem_optin);
    cudaGetLastError();  // a refused attribute only disables the cap
}

int launch_seed(xg_ensemble* h, uint64_t seed0, cudaStream_t s) {
    const unsigned grid = grid_for(h->num_streams);
    switch (h->kind) {
    case kGeneric: {
        const size_t smem = gen_smem(h->params);
        int rc = gen_smem_attr<&gen_seed_kernel>(smem);
        if (rc) return rc;
        gen_seed_kernel<<<h->num_streams, 32, smem, s>>>(gen_params(h->params), h->d_win64,
                                                        h->d_weyl64, h->num_streams, seed0);
        break;
    }
    case kGP32:
        seed_kernel<<<grid, kThreads, 0, s>>>(GP32{}, h->d_win, h->d_weyl, h->num_streams, seed0);
        break;
    case kRtJ1:
        seed_kernel<<<grid, kThreads, 0, s>>>(rt_params<1>(h->params), h->d_win, h->d_weyl,
                                             h->num_streams, seed0);
        break;
    default:
        seed_kernel<<<grid, kThreads, 0, s>>>(rt_params<2>(h->params), h->d_win, h->d_weyl,
                                             h->num_streams, seed0);
        break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

int alloc_state(xg_ensemble* h) {
    const size_t n = static_cast<size_t>(h->num_streams);
    if (h->kind == kGeneric) {
        int rc = cuda_rc(cudaMalloc(&h->d_win64, n * h->params.r * sizeof(uint64_t)));
        if (rc) return rc;
        return cuda_rc(cudaMalloc(&h->d_weyl64, n * sizeof(uint64_t)));
    }
    int rc = cuda_rc(cudaMalloc(&h->d_win, n * kR * sizeof(uint32_t)));
    if (rc) return rc;
    return cuda_rc(cudaMalloc(&h->d_weyl, n * sizeof(uint32_t)));
}

void free_handle(xg_ensemble* h) {
    if (!h) return;
    {
        DeviceGuard dg(h->device);
        cudaFree(h->d_win);
        cudaFree(h->d_weyl);
        cudaFree(h->d_win64);
        cudaFree(h->d_weyl64);
        if (h->nr.st) cudaStreamSynchronize(h->nr.st);
        for (int i = 0; i < 2; ++i) {
            cudaFreeHost(h->nr.host[i]);
            cudaFree(h->nr.dev[i]);
            cudaFree(h->nr.snap[i]);
            if (h->nr.ev[i]) cudaEventDestroy(h->nr.ev[i]);
        }
        if (h->nr.st) cudaStreamDestroy(h->nr.st);
        cudaFree(h->d_stage);
        cudaFreeHost(h->h_stage);
        cudaFree(h->d_lc);
        cudaFree(h->d_jrows);
        cudaFree(h->d_jweyl);
        cudaFree(h->d_jpart);
        cudaFree(h->d_jW);
        cudaFree(h->d_jseq);
        if (h->jside) cudaStreamDestroy(h->jside);
        for (int i = 0; i < 2; ++i)
            if (h->jev[i]) cudaEventDestroy(h->jev[i]);
    }
    delete h;
}

// Device-side copy of stream 0's whole state to / from a snapshot buffer.
size_t state_bytes(const xg_ensemble* h, size_t* win_bytes) {
    *win_bytes = h->kind == kGeneric ? h->params.r * sizeof(uint64_t) : kR * sizeof(uint32_t);
    return *win_bytes + sizeof(uint64_t);
}

int copy_state(xg_ensemble* h, void* snap, bool to_snapshot, cudaStream_t s) {
    size_t wb;
    state_bytes(h, &wb);
    char* sn = static_cast<char*>(snap);
    void* win = h->kind == kGeneric ? static_cast<void*>(h->d_win64) : static_cast<void*>(h->d_win);
    void* wy = h->kind == kGeneric ? static_cast<void*>(h->d_weyl64) : static_cast<void*>(h->d_weyl);
    const size_t wyb = h->kind == kGeneric ? sizeof(uint64_t) : sizeof(uint32_t);
    const cudaMemcpyKind k = cudaMemcpyDeviceToDevice;
    int rc = cuda_rc(to_snapshot ? cudaMemcpyAsync(sn, win, wb, k, s) : cudaMemcpyAsync(win, sn, wb, k, s));
    if (rc) return rc;
    return cuda_rc(to_snapshot ? cudaMemcpyAsync(sn + wb, wy, wyb, k, s)
                               : cudaMemcpyAsync(wy, sn + wb, wyb, k, s));
}

// next_word words generated but not served are given back before any other
// use of the handle: wait for the ring's stream, restore the state saved
// before the slot being served and re-advance it by the words served, so the
// device state is exactly "after the last word the caller saw".
int settle_next(xg_ensemble* h, cudaStream_t s) {
    auto& r = h->nr;
    if (!r.active) return XG_OK;
    r.active = false;
    int rc = cuda_rc(cudaStreamSynchronize(r.st));
    if (!rc) rc = copy_state(h, r.snap[r.cur], /*to_snapshot=*/false, s);
    if (!rc && r.pos) rc = launch_fill<kSkip>(h, 0, 1, r.pos, nullptr, nullptr, s);
    r.pos = 0;
    return rc;
}

bool mul_overflows(uint64_t a, uint64_t b, uint64_t* out) {
    return __builtin_mul_overflow(a, b, out);
}

int fill_common(xg_ensemble_t h, uint64_t per_stream, void* dev_out, size_t align, int mode,
                xg_stream_t stream) {
    if (!h) return XG_EINVAL;
    uint64_t total;
    if (mul_overflows(per_stream, h->num_streams, &total)) return XG_EINVAL;
    if (per_stream == 0) return XG_OK;
    if (!dev_out || (reinterpret_cast<uintptr_t>(dev_out) % align) != 0) return XG_EINVAL;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    switch (mode) {
    case kU32: return launch_fill<kU32>(h, 0, h->num_streams, per_stream, dev_out, nullptr, s);
    case kF32: return launch_fill<kF32>(h, 0, h->num_streams, per_stream, dev_out, nullptr, s);
    case kRaw: return launch_fill<kRaw>(h, 0, h->num_streams, per_stream, dev_out, nullptr, s);
    case kWide: return launch_fill<kWide>(h, 0, h->num_streams, per_stream, dev_out, nullptr, s);
    case kF64: {
        uint64_t words;
        if (mul_overflows(per_stream, 2, &words)) return XG_EINVAL;
        return launch_fill<kF64>(h, 0, h->num_streams, words, dev_out, nullptr, s);
    }
    default: return XG_EINVAL;
    }
}

int launch_bm_long(const uint32_t* data, uint64_t data_words, uint64_t nbits, uint64_t stride_bits,
                   uint32_t per_row, uint64_t row_bits, uint64_t count, unsigned long long* hist,
                   uint32_t* L_out, cudaStream_t s) {
    const size_t smem = 4ull * bm_words(nbits) * sizeof(uint32_t);
    static std::atomic<uint64_t> done{0};
    int rc = raise_smem_once(bm_long_kernel, 4ull * bm_words(kBmMaxBits) * sizeof(uint32_t), done);
    if (rc) return rc;
    bm_long_kernel<<<static_cast<unsigned>(count), 32, smem, s>>>(data, data_words, nbits, stride_bits,
                                                                 per_row, row_bits, hist, L_out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

}  // namespace

extern "C" {

int xg_params_check(const xg_params_t* p) { return check_params_impl(p); }

const char* xg_strerror(int code) {
    switch (code) {
    case XG_OK: return "ok";
    // proj/src/params.cpp:7-18
    case XG_EPARAM_BAD_WORD_SIZE: return "word size must be 8, 16, 32 or 64";
    case XG_EPARAM_S_OUT_OF_RANGE: return "tap offset s must satisfy 0 < s < r";
    case XG_EPARAM_GCD_NOT_ONE: return "r and s must be coprime";
    case XG_EPARAM_SHIFT_OUT_OF_RANGE: return "shifts a, b, c, d must lie in (0, w)";
    case XG_EPARAM_GAMMA_OUT_OF_RANGE: return "output shift gamma must lie in (0, w)";
    case XG_EPARAM_EVEN_WEYL_INCREMENT: return "Weyl increment omega must be odd";
    case XG_ERANGE: return "argument out of range";
    case XG_EINVAL: return "invalid argument";
    case XG_EUNSUPPORTED: return "not available for these parameters (the f32/f64/u64/MC conventions need w=32, r=128, lane_bound>=32; r <= 16384)";
    case XG_ECUDA: return "CUDA runtime error";
    case XG_ENOMEM: return "device memory allocation failed";
    default: return "unknown error";
    }
}

unsigned xg_lane_bound(const xg_params_t* p) { return p ? lane_bound_impl(p) : 0u; }

uint64_t xg_recommended_weyl_increment(unsigned w) {
    switch (w) {
    case 8: return 159u;
    case 16: return 40503u;
    case 32: return 2654435769ull;
    case 64: return 11400714819323198485ull;
    default: return 0;
    }
}

unsigned xg_default_output_shift(unsigned w) { return w / 2; }

static xg_params_t make_set(unsigned r, unsigned s, unsigned a, unsigned b, unsigned c, unsigned d,
                            unsigned w) {
    xg_params_t p;
    p.r = r; p.s = s; p.a = a; p.b = b; p.c = c; p.d = d; p.w = w;
    p.omega = xg_recommended_weyl_increment(w);
    p.gamma = xg_default_output_shift(w);
    return p;
}

xg_params_t xg_params_xorgensgp32(void) { return make_set(128, 65, 15, 14, 12, 17, 32); }
xg_params_t xg_params_tiny_r2w8(void) { return make_set(2, 1, 1, 1, 5, 7, 8); }
xg_params_t xg_params_tiny_r2w16(void) { return make_set(2, 1, 1, 1, 6, 11, 16); }
xg_params_t xg_params_tiny_r4w16(void) { return make_set(4, 3, 1, 2, 5, 8, 16); }

int xg_gpu_supported(const xg_params_t* p) {
    Kind k;
    return classify(p, &k);
}

int xg_fast_path(const xg_params_t* p) {
    Kind k;
    return classify(p, &k) == XG_OK && k != kGeneric ? 1 : 0;
}

int xg_ensemble_create(const xg_params_t* p, uint64_t base_seed, uint64_t first_stream,
                       uint32_t num_streams, unsigned lanes, int device, xg_stream_t stream,
                       xg_ensemble_t* out) {
    if (!out) return XG_EINVAL;
    *out = nullptr;
    // proj/src/parallel.cpp:86-91: validate_params, then blocks, then lanes.
    int e = check_params_impl(p);
    if (e) return e;
    if (num_streams == 0) return XG_ERANGE;
    if (lanes == 0 || lanes > lane_bound_impl(p)) return XG_ERANGE;
    Kind kind;
    e = classify(p, &kind);
    if (e) return e;
    DeviceGuard dg(device);
    if (!dg.ok) return XG_ECUDA;
    auto* h = new (std::nothrow) xg_ensemble;
    if (!h) return XG_ENOMEM;
    h->params = *p;
    h->kind = kind;
    h->device = device;
    h->num_streams = num_streams;
    h->base_seed = base_seed;
    h->first_stream = first_stream;
    h->lanes = lanes;
    prepare_pair_kernels(h);
    int rc = alloc_state(h);
    if (!rc) rc = launch_seed(h, base_seed + first_stream, reinterpret_cast<cudaStream_t>(stream));
    if (rc) {
        free_handle(h);
        return rc;
    }
    *out = h;
    return XG_OK;
}

int xg_ensemble_create_from_raw(const xg_params_t* p, uint32_t num_streams,
                                const uint64_t* buffers, const uint64_t* weyls, int device,
                                xg_stream_t stream, xg_ensemble_t* out) {
    if (!out) return XG_EINVAL;
    *out = nullptr;
    int e = check_params_impl(p);
    if (e) return e;
    if (num_streams == 0) return XG_ERANGE;
    if (!buffers || !weyls) return XG_EINVAL;
    Kind kind;
    e = classify(p, &kind);
    if (e) return e;
    DeviceGuard dg(device);
    if (!dg.ok) return XG_ECUDA;
    auto* h = new (std::nothrow) xg_ensemble;
    if (!h) return XG_ENOMEM;
    h->params = *p;
    h->kind = kind;
    h->device = device;
    h->num_streams = num_streams;
    h->lanes = lane_bound_impl(p);
    prepare_pair_kernels(h);
    int rc = alloc_state(h);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!rc && kind == kGeneric) {
        const uint64_t mask = p->w >= 64 ? ~0ull : ((1ull << p->w) - 1);
        std::vector<uint64_t> win(static_cast<size_t>(num_streams) * p->r), wy(num_streams);
        for (size_t i = 0; i < win.size(); ++i) win[i] = buffers[i] & mask;
        for (size_t i = 0; i < wy.size(); ++i) wy[i] = weyls[i] & mask;
        rc = cuda_rc(cudaMemcpyAsync(h->d_win64, win.data(), win.size() * 8, cudaMemcpyHostToDevice, s));
        if (!rc) rc = cuda_rc(cudaMemcpyAsync(h->d_weyl64, wy.data(), wy.size() * 8, cudaMemcpyHostToDevice, s));
        if (!rc) rc = cuda_rc(cudaStreamSynchronize(s));
    } else if (!rc) {
        std::vector<uint32_t> win(static_cast<size_t>(num_streams) * kR), wy(num_streams);
        for (size_t i = 0; i < win.size(); ++i) win[i] = static_cast<uint32_t>(buffers[i] & kMask32);
        for (size_t i = 0; i < wy.size(); ++i) wy[i] = static_cast<uint32_t>(weyls[i] & kMask32);
        rc = cuda_rc(cudaMemcpyAsync(h->d_win, win.data(), win.size() * 4, cudaMemcpyHostToDevice, s));
        if (!rc) rc = cuda_rc(cudaMemcpyAsync(h->d_weyl, wy.data(), wy.size() * 4, cudaMemcpyHostToDevice, s));
        if (!rc) rc = cuda_rc(cudaStreamSynchronize(s));
    }
    if (rc) {
        free_handle(h);
        return rc;
    }
    *out = h;
    return XG_OK;
}

int xg_ensemble_destroy(xg_ensemble_t h) {
    if (!h) return XG_EINVAL;
    free_handle(h);
    return XG_OK;
}

int xg_ensemble_info(xg_ensemble_t h, uint32_t* num_streams, uint64_t* base_seed,
                     uint64_t* first_stream, unsigned* lanes, int* device) {
    if (!h) return XG_EINVAL;
    if (num_streams) *num_streams = h->num_streams;
    if (base_seed) *base_seed = h->base_seed;
    if (first_stream) *first_stream = h->first_stream;
    if (lanes) *lanes = h->lanes;
    if (device) *device = h->device;
    return XG_OK;
}

int xg_fill_u32(xg_ensemble_t h, uint64_t per_stream, uint32_t* dev_out, xg_stream_t stream) {
    return fill_common(h, per_stream, dev_out, 4, kU32, stream);
}

int xg_fill_words(xg_ensemble_t h, uint64_t per_stream, uint64_t* dev_out, xg_stream_t stream) {
    return fill_common(h, per_stream, dev_out, 8, kWide, stream);
}

int xg_fill_u64(xg_ensemble_t h, uint64_t per_stream, uint64_t* dev_out, xg_stream_t stream) {
    if (h && h->kind == kGeneric) return XG_EUNSUPPORTED;
    uint64_t words;
    if (mul_overflows(per_stream, 2, &words)) return XG_EINVAL;
    if (reinterpret_cast<uintptr_t>(dev_out) % 8 != 0) return XG_EINVAL;
    // Little-endian: (lo, hi) word pairs are exactly the uint64 values.
    return fill_common(h, words, dev_out, 8, kU32, stream);
}

int xg_fill_raw_u32(xg_ensemble_t h, uint64_t per_stream, uint32_t* dev_out, xg_stream_t stream) {
    return fill_common(h, per_stream, dev_out, 4, kRaw, stream);
}

int xg_fill_f32(xg_ensemble_t h, uint64_t per_stream, float* dev_out, xg_stream_t stream) {
    return fill_common(h, per_stream, dev_out, 4, kF32, stream);
}

int xg_fill_f64(xg_ensemble_t h, uint64_t per_stream, double* dev_out, xg_stream_t stream) {
    return fill_common(h, per_stream, dev_out, 8, kF64, stream);
}

int xg_mc_pi(xg_ensemble_t h, uint64_t samples_per_stream, uint64_t* dev_hits,
             xg_stream_t stream) {
    if (!h || !dev_hits || (reinterpret_cast<uintptr_t>(dev_hits) % 8) != 0) return XG_EINVAL;
    // Samples come in blocks of 32 per stream (64 words, one lane-pair of warp steps).
    if (samples_per_stream % 32 != 0) return XG_EINVAL;
    if (samples_per_stream == 0) return XG_OK;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    // Per-lane hit counters are 32-bit: bound samples per launch to 2^36.
    constexpr uint64_t kChunk = 1ull << 36;
    uint64_t left = samples_per_stream;
    while (left) {
        const uint64_t n = std::min(left, kChunk);
        rc = launch_fill<kMC>(h, 0, h->num_streams, 2 * n, nullptr,
                              reinterpret_cast<unsigned long long*>(dev_hits), s);
        if (rc) return rc;
        left -= n;
    }
    return XG_OK;
}

int xg_rank_test(xg_ensemble_t h, uint64_t matrices_per_stream, uint64_t* dev_counts,
                 xg_stream_t stream) {
    if (!h || !dev_counts || (reinterpret_cast<uintptr_t>(dev_counts) % 8) != 0) return XG_EINVAL;
    if (h->kind == kGeneric || h->kind == kRtJ2) return XG_EUNSUPPORTED;
    if (matrices_per_stream == 0) return XG_OK;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    // Per-lane bin counters are 32-bit: bound matrices per stream and launch.
    constexpr uint64_t kChunk = 1ull << 31;
    uint64_t left = matrices_per_stream;
    while (left) {
        const uint64_t n = std::min(left, kChunk);
        rc = launch_fill<kRank>(h, 0, h->num_streams, 32 * n, nullptr,
                                reinterpret_cast<unsigned long long*>(dev_counts), s);
        if (rc) return rc;
        left -= n;
    }
    return XG_OK;
}

int xg_linear_complexity_test(xg_ensemble_t h, unsigned block_length, uint64_t blocks_per_stream,
                              uint64_t* dev_hist, xg_stream_t stream) {
    if (!h || !dev_hist || (reinterpret_cast<uintptr_t>(dev_hist) % 8) != 0) return XG_EINVAL;
    if (block_length == 0 || block_length > kBmMaxBits) return XG_EINVAL;
    if (h->params.w != 32) return XG_EUNSUPPORTED;  // BitSource reads w bits per word
    if (blocks_per_stream == 0) return XG_OK;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    const uint64_t P = h->num_streams, K = block_length;
    // Chunks of whole words: 32 blocks are exactly K words.  Aim at <= 2^26
    // buffered words; only the last chunk may end inside a word, whose
    // remaining bits are dropped as a fresh BitSource drops them.
    const uint64_t per32 = std::max<uint64_t>(1, (1ull << 26) / std::max<uint64_t>(1, P * K));
    const uint64_t bc = std::min<uint64_t>(32 * per32, 1ull << 31);
    uint64_t left = blocks_per_stream;
    while (left) {
        const uint64_t nb = std::min(left, bc);
        const uint64_t wc = (nb * K + 31) / 32;
        const size_t need = static_cast<size_t>(P * wc) * sizeof(uint32_t);
        if (h->lc_bytes < need) {
            // Stream-ordered (re)allocation: no device synchronisation, and
            // capturable into a CUDA graph like the fills.  The buffer is
            // per-handle state, ordered like the generator state itself:
            // calls on one handle must be ordered on the host or by stream.
            if (h->d_lc) cudaFreeAsync(h->d_lc, s);
            h->d_lc = nullptr;
            h->lc_bytes = 0;
            rc = cuda_rc(cudaMallocAsync(reinterpret_cast<void**>(&h->d_lc), need, s));
            if (rc) return rc;
            h->lc_bytes = need;
        }
        rc = launch_fill<kU32>(h, 0, h->num_streams, wc, h->d_lc, nullptr, s);
        if (rc) return rc;
        const uint64_t warps = P * nb;
        if (K <= kLcMaxK) {  // register-resident polynomials (1024 bits per warp)
            lc_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(
                h->d_lc, h->num_streams, wc, block_length, static_cast<uint32_t>(nb),
                reinterpret_cast<unsigned long long*>(dev_hist));
            g_launches.fetch_add(1, std::memory_order_relaxed);
            rc = cuda_rc(cudaGetLastError());
        } else {  // longer blocks: polynomials in shared memory
            rc = launch_bm_long(h->d_lc, P * wc, K, K, static_cast<uint32_t>(nb), wc * 32, warps,
                                reinterpret_cast<unsigned long long*>(dev_hist), nullptr, s);
        }
        if (rc) return rc;
        left -= nb;
    }
    return XG_OK;
}

int xg_berlekamp_massey(const uint32_t* dev_seqs, uint64_t nbits, uint32_t count,
                        uint64_t stride_words, uint32_t* dev_L, xg_stream_t stream) {
    if (!dev_seqs || !dev_L || nbits == 0 || nbits > kBmMaxBits) return XG_EINVAL;
    if (count == 0) return XG_OK;
    uint64_t stride_bits = 0, span = 0;  // one sequence: the stride is never used
    if (count > 1 && (mul_overflows(stride_words, 32, &stride_bits) ||
                      mul_overflows(static_cast<uint64_t>(count - 1), stride_words, &span) ||
                      stride_bits < nbits))
        return XG_EINVAL;
    int dev;
    int rc = ptr_device(dev_seqs, &dev);
    if (rc) return rc;
    DeviceGuard dg(dev);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t data_words = span + (nbits + 31) / 32;
    return launch_bm_long(dev_seqs, data_words, nbits, stride_bits, count, 0, count, nullptr,
                          dev_L, s);
}

int xg_rank_words(const uint32_t* dev_words, uint64_t matrices, uint64_t* dev_counts,
                  xg_stream_t stream) {
    if (!dev_words || !dev_counts || (reinterpret_cast<uintptr_t>(dev_counts) % 8) != 0) return XG_EINVAL;
    if (matrices == 0) return XG_OK;
    if (matrices > (1ull << 58)) return XG_EINVAL;
    int dev;
    int rc = ptr_device(dev_words, &dev);
    if (rc) return rc;
    DeviceGuard dg(dev);
    if (!dg.ok) return XG_ECUDA;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t pairs = (matrices + 1) / 2;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((pairs + 7) / 8, 8ull * sms));
    rank_words_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        dev_words, matrices, reinterpret_cast<unsigned long long*>(dev_counts));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

int xg_lc_words(const uint32_t* dev_words, uint64_t nwords, unsigned block_length, uint64_t blocks,
                uint64_t* dev_hist, xg_stream_t stream) {
    if (!dev_words || !dev_hist || (reinterpret_cast<uintptr_t>(dev_hist) % 8) != 0) return XG_EINVAL;
    if (block_length == 0 || block_length > kBmMaxBits || blocks > 0xffffffffull) return XG_EINVAL;
    if (blocks == 0) return XG_OK;
    uint64_t nbits_in;
    if (mul_overflows(nwords, 32, &nbits_in)) nbits_in = ~0ull;  // more bits than any request
    if (nbits_in < static_cast<uint64_t>(block_length) * blocks) return XG_EINVAL;
    int dev;
    int rc = ptr_device(dev_words, &dev);
    if (rc) return rc;
    DeviceGuard dg(dev);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto* hist = reinterpret_cast<unsigned long long*>(dev_hist);
    if (block_length <= kLcMaxK) {
        lc_kernel<<<static_cast<unsigned>((blocks + 7) / 8), 256, 0, s>>>(
            dev_words, 1, nwords, block_length, static_cast<uint32_t>(blocks), hist);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cuda_rc(cudaGetLastError());
    }
    return launch_bm_long(dev_words, nwords, block_length, block_length, static_cast<uint32_t>(blocks),
                          static_cast<uint64_t>(block_length) * blocks, blocks, hist, nullptr, s);
}

int xg_pack_words(const uint32_t* dev_in, uint64_t n, unsigned w, int left_align, uint32_t* dev_out,
                  xg_stream_t stream) {
    if (!dev_in || !dev_out || (w != 8 && w != 16 && w != 32)) return XG_EINVAL;
    if (n == 0) return XG_OK;
    uint64_t nbits;
    if (mul_overflows(n, w, &nbits) || nbits > ~0ull - 31) return XG_EINVAL;
    int dev;
    int rc = ptr_device(dev_in, &dev);
    if (rc) return rc;
    DeviceGuard dg(dev);
    if (!dg.ok) return XG_ECUDA;
    const uint64_t nout = left_align ? n : (nbits + 31) / 32;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((nout + 255) / 256, 8ull * sms));
    pack_words_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(dev_in, n, w, left_align,
                                                                              dev_out, nout);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

int xg_bits_ones_runs(const uint32_t* dev_words, uint64_t nbits, uint64_t* dev_out2,
                      xg_stream_t stream) {
    if (!dev_words || !dev_out2 || (reinterpret_cast<uintptr_t>(dev_out2) % 8) != 0) return XG_EINVAL;
    if (nbits == 0) return XG_OK;
    int dev;
    int rc = ptr_device(dev_words, &dev);
    if (rc) return rc;
    DeviceGuard dg(dev);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t nwords = (nbits + 31) / 32;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((nwords + 255) / 256, 148 * 16));
    ones_runs_kernel<<<grid, 256, 0, s>>>(dev_words, nbits,
                                          reinterpret_cast<unsigned long long*>(dev_out2));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

int xg_birthday_duplicates(const uint32_t* dev_words, uint32_t n_draws, uint32_t rounds,
                           unsigned t_bits, uint64_t* dev_dup, xg_stream_t stream) {
    if (!dev_words || !dev_dup || (reinterpret_cast<uintptr_t>(dev_dup) % 8) != 0) return XG_EINVAL;
    if (t_bits == 0 || t_bits > 32 || n_draws < 2 ||
        n_draws > static_cast<uint32_t>(kBdThreads * kBdItems))
        return XG_EINVAL;
    if (rounds == 0) return XG_OK;
    int dev;
    int rc = ptr_device(dev_words, &dev);
    if (rc) return rc;
    DeviceGuard dg(dev);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    birthday_kernel<<<rounds, kBdThreads, 0, s>>>(dev_words, n_draws, 32u - t_bits,
                                                   reinterpret_cast<unsigned long long*>(dev_dup));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

int xg_digest_u32(const uint32_t* dev_words, uint64_t rows, uint64_t per_row, uint32_t* dev_xor,
                  uint64_t* dev_sum, uint64_t* dev_wsum, xg_stream_t stream) {
    if (rows == 0) return XG_OK;
    if (!dev_words || !dev_xor || !dev_sum || !dev_wsum || rows > 0x7fffffffull) return XG_EINVAL;
    if ((reinterpret_cast<uintptr_t>(dev_sum) | reinterpret_cast<uintptr_t>(dev_wsum)) % 8 != 0)
        return XG_EINVAL;
    uint64_t total;
    if (mul_overflows(rows, per_row, &total)) return XG_EINVAL;
    int dev;
    int rc = ptr_device(dev_xor, &dev);
    if (!rc && per_row) rc = ptr_device(dev_words, &dev);
    if (rc) return rc;
    DeviceGuard dg(dev);
    if (!dg.ok) return XG_ECUDA;
    digest_kernel<<<static_cast<unsigned>(rows), kDigestThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        dev_words, per_row, dev_xor, reinterpret_cast<unsigned long long*>(dev_sum),
        reinterpret_cast<unsigned long long*>(dev_wsum));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

int xg_skip(xg_ensemble_t h, uint64_t words, xg_stream_t stream) {
    if (!h) return XG_EINVAL;
    if (words == 0) return XG_OK;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    return launch_fill<kSkip>(h, 0, h->num_streams, words, nullptr, nullptr, s);
}

}  // extern "C"

namespace {

// BlockEnsemble::generate into host memory, element T (uint32 words or the
// reference's uint64 container), produced by kernel mode MODE.
template <int MODE, class T>
int generate_host_impl(xg_ensemble_t h, uint64_t per_stream, T* host_out, xg_stream_t stream) {
    if (!h) return XG_EINVAL;
    uint64_t total;
    if (mul_overflows(per_stream, h->num_streams, &total)) return XG_EINVAL;
    if (per_stream == 0) return XG_OK;
    if (!host_out) return XG_EINVAL;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    // Two staging slots of up to 64 Mi words.  The (streams x words) output is
    // cut into tiles: groups of whole streams when a stream fits a slot,
    // otherwise groups of 2048 streams advanced in word chunks (each stream's
    // chunks in order, so the continuation is exact).  Tile i is generated on
    // `s` while tile i-1 is copied (2D, into the block-major host layout) on a
    // second stream.
    constexpr uint64_t kSlotWords = (1ull << 28) / sizeof(T);  // 256 MiB per staging slot
    constexpr uint64_t kGroup = 2048;
    uint64_t cnt_max, m_max;
    if (per_stream <= kSlotWords) {
        m_max = per_stream;
        cnt_max = std::min<uint64_t>(std::max<uint64_t>(1, kSlotWords / per_stream), h->num_streams);
    } else {
        cnt_max = std::min<uint64_t>(kGroup, h->num_streams);
        m_max = (kSlotWords / cnt_max) & ~uint64_t{127};
    }
    const uint64_t slot_words = cnt_max * m_max;
    if (h->stage_words < 2 * slot_words * sizeof(T)) {
        cudaFree(h->d_stage);
        h->d_stage = nullptr;
        h->stage_words = 0;
        rc = cuda_rc(cudaMalloc(&h->d_stage, 2 * slot_words * sizeof(T)));
        if (rc) return rc;
        h->stage_words = 2 * slot_words * sizeof(T);
    }
    cudaStream_t cs;
    rc = cuda_rc(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    if (rc) return rc;
    cudaEvent_t gen_done[2], copy_done[2];
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&gen_done[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&copy_done[i], cudaEventDisableTiming);
        cudaEventRecord(copy_done[i], cs);
    }
    int slot = 0;
    for (uint64_t g0 = 0; g0 < h->num_streams && !rc; g0 += cnt_max) {
        const uint32_t cnt = static_cast<uint32_t>(std::min<uint64_t>(cnt_max, h->num_streams - g0));
        for (uint64_t k0 = 0; k0 < per_stream && !rc; k0 += m_max) {
            const uint64_t m = std::min<uint64_t>(m_max, per_stream - k0);
            T* d = reinterpret_cast<T*>(h->d_stage) + slot * slot_words;
            cudaStreamWaitEvent(s, copy_done[slot], 0);
            rc = launch_fill<MODE>(h, static_cast<uint32_t>(g0), cnt, (MODE == kF64 ? 2 : 1) * m, d,
                                   nullptr, s);
            if (rc) break;
            cudaEventRecord(gen_done[slot], s);
            cudaStreamWaitEvent(cs, gen_done[slot], 0);
            rc = cuda_rc(cudaMemcpy2DAsync(host_out + g0 * per_stream + k0, per_stream * sizeof(T), d,
                                           m * sizeof(T), m * sizeof(T), cnt,
                                           cudaMemcpyDeviceToHost, cs));
            cudaEventRecord(copy_done[slot], cs);
            slot ^= 1;
        }
    }
    const int rc2 = cuda_rc(cudaStreamSynchronize(cs));
    const int rc3 = cuda_rc(cudaStreamSynchronize(s));
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(gen_done[i]);
        cudaEventDestroy(copy_done[i]);
    }
    cudaStreamDestroy(cs);
    return rc ? rc : (rc2 ? rc2 : rc3);
}

// BlockEnsemble::generate through host tiles: tiles of streams x words are
// generated on `s` as u32 (w <= 32; 4 PCIe bytes per word instead of 8),
// copied to pinned staging on a second stream, and handed to `consume` on
// nthr host threads (consume(g0, k0, streams, words, tile, id, nthr)) while
// the device already produces and copies the next tile.  Tiles of one stream
// arrive in word order.
template <int MODE, class T, class Consume>
int generate_tiles_impl(xg_ensemble_t h, uint64_t per_stream, unsigned nthr, Consume consume,
                        cudaStream_t s) {
    constexpr uint64_t kSlotWords = (1ull << 28) / sizeof(T);  // 256 MiB per staging slot
    constexpr uint64_t kGroup = 2048;
    uint64_t cnt_max, m_max;
    if (per_stream <= kSlotWords) {
        m_max = per_stream;
        cnt_max = std::min<uint64_t>(std::max<uint64_t>(1, kSlotWords / per_stream), h->num_streams);
    } else {
        cnt_max = std::min<uint64_t>(kGroup, h->num_streams);
        m_max = (kSlotWords / cnt_max) & ~uint64_t{127};
    }
    const uint64_t slot_words = cnt_max * m_max;
    const size_t slot_bytes = slot_words * sizeof(T);
    int rc = XG_OK;
    if (h->stage_words < 2 * slot_bytes) {
        cudaFree(h->d_stage);
        h->d_stage = nullptr;
        h->stage_words = 0;
        rc = cuda_rc(cudaMalloc(&h->d_stage, 2 * slot_bytes));
        if (rc) return rc;
        h->stage_words = 2 * slot_bytes;
    }
    if (h->h_stage_bytes < 2 * slot_bytes) {
        cudaFreeHost(h->h_stage);
        h->h_stage = nullptr;
        h->h_stage_bytes = 0;
        rc = cuda_rc(cudaMallocHost(&h->h_stage, 2 * slot_bytes));
        if (rc) return rc;
        h->h_stage_bytes = 2 * slot_bytes;
    }
    struct Tile {
        uint64_t g0, k0, cnt, m;
    };
    std::vector<Tile> tiles;
    for (uint64_t g0 = 0; g0 < h->num_streams; g0 += cnt_max) {
        const uint64_t cnt = std::min<uint64_t>(cnt_max, h->num_streams - g0);
        for (uint64_t k0 = 0; k0 < per_stream; k0 += m_max)
            tiles.push_back({g0, k0, cnt, std::min<uint64_t>(m_max, per_stream - k0)});
    }
    cudaStream_t cs;
    rc = cuda_rc(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    if (rc) return rc;
    cudaEvent_t gen_done[2], copy_done[2];
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&gen_done[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&copy_done[i], cudaEventDisableTiming);
    }
    auto enqueue = [&](size_t t) {
        const Tile& tl = tiles[t];
        const int slot = static_cast<int>(t & 1);
        T* d = static_cast<T*>(h->d_stage) + slot * slot_words;
        T* hs = static_cast<T*>(h->h_stage) + slot * slot_words;
        int e = launch_fill<MODE>(h, static_cast<uint32_t>(tl.g0), static_cast<uint32_t>(tl.cnt), tl.m, d,
                                  nullptr, s);
        if (!e) e = cuda_rc(cudaEventRecord(gen_done[slot], s));
        if (!e) e = cuda_rc(cudaStreamWaitEvent(cs, gen_done[slot], 0));
        if (!e) e = cuda_rc(cudaMemcpyAsync(hs, d, tl.cnt * tl.m * sizeof(T), cudaMemcpyDeviceToHost, cs));
        if (!e) e = cuda_rc(cudaEventRecord(copy_done[slot], cs));
        return e;
    };
    if (!tiles.empty()) rc = enqueue(0);
    for (size_t t = 0; t < tiles.size() && !rc; ++t) {
        // Tile t+1 goes into the slot tile t-1 used, whose rows were written
        // in the previous iteration.
        if (t + 1 < tiles.size()) rc = enqueue(t + 1);
        if (!rc) rc = cuda_rc(cudaEventSynchronize(copy_done[t & 1]));
        if (rc) break;
        const Tile tl = tiles[t];
        const T* hs = static_cast<const T*>(h->h_stage) + (t & 1) * slot_words;
        auto widen = [&, tl, hs](unsigned id) {
            consume(tl.g0, tl.k0, tl.cnt, tl.m, hs, id, nthr);
        };
        std::vector<std::thread> pool;
        pool.reserve(nthr - 1);
        for (unsigned id = 1; id < nthr; ++id) pool.emplace_back(widen, id);
        widen(0);
        for (auto& th : pool) th.join();
    }
    const int rc2 = cuda_rc(cudaStreamSynchronize(cs));
    const int rc3 = cuda_rc(cudaStreamSynchronize(s));
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(gen_done[i]);
        cudaEventDestroy(copy_done[i]);
    }
    cudaStreamDestroy(cs);
    return rc ? rc : (rc2 ? rc2 : rc3);
}

}  // namespace

extern "C" {

int xg_generate_host_rows(xg_ensemble_t h, uint64_t per_stream, uint64_t* const* rows,
                          xg_stream_t stream) {
    if (!h) return XG_EINVAL;
    uint64_t total;
    if (mul_overflows(per_stream, h->num_streams, &total)) return XG_EINVAL;
    if (per_stream == 0) return XG_OK;
    if (!rows) return XG_EINVAL;
    for (uint32_t g = 0; g < h->num_streams; ++g)
        if (!rows[g]) return XG_EINVAL;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    const unsigned nthr = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    // rows split between threads; one long row split by words
    auto copy = [rows](uint64_t g0, uint64_t kb, uint64_t cnt, uint64_t m, const auto* hs, unsigned id,
                       unsigned nt) {
        const uint64_t parts = cnt >= nt ? cnt : nt;
        for (uint64_t q = id; q < parts; q += nt) {
            uint64_t i, k0, k1;
            if (cnt >= nt) {
                i = q; k0 = 0; k1 = m;
            } else {
                const uint64_t per_row = nt / cnt;  // threads per row (>= 1)
                i = q / per_row;
                const uint64_t sub = q % per_row;
                if (i >= cnt) continue;
                k0 = m * sub / per_row; k1 = m * (sub + 1) / per_row;
            }
            uint64_t* dst = rows[g0 + i] + kb;
            const auto* src = hs + i * m;
            for (uint64_t k = k0; k < k1; ++k) dst[k] = src[k];
        }
    };
    if (h->params.w <= 32) return generate_tiles_impl<kU32, uint32_t>(h, per_stream, nthr, copy, s);
    return generate_tiles_impl<kWide, uint64_t>(h, per_stream, nthr, copy, s);
}

int xg_generate_host_tiles(xg_ensemble_t h, uint64_t per_stream, xg_tile_fn fn, void* ctx,
                           unsigned threads, xg_stream_t stream) {
    if (!h || !fn) return XG_EINVAL;
    uint64_t total;
    if (mul_overflows(per_stream, h->num_streams, &total)) return XG_EINVAL;
    if (per_stream == 0) return XG_OK;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = settle_next(h, s);
    if (rc) return rc;
    const unsigned nthr = threads ? std::min(threads, 256u)
                                  : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    auto call = [fn, ctx](uint64_t g0, uint64_t kb, uint64_t cnt, uint64_t m, const auto* hs, unsigned id,
                          unsigned nt) {
        fn(ctx, g0, kb, cnt, m, hs, static_cast<unsigned>(sizeof(*hs)), id, nt);
    };
    if (h->params.w <= 32) return generate_tiles_impl<kU32, uint32_t>(h, per_stream, nthr, call, s);
    return generate_tiles_impl<kWide, uint64_t>(h, per_stream, nthr, call, s);
}

int xg_generate_host(xg_ensemble_t h, uint64_t per_stream, uint32_t* host_out,
                     xg_stream_t stream) {
    if (h && h->params.w > 32) return XG_EUNSUPPORTED;  // xg_generate_host_words for w = 64
    return generate_host_impl<kU32>(h, per_stream, host_out, stream);
}

int xg_generate_host_words(xg_ensemble_t h, uint64_t per_stream, uint64_t* host_out,
                           xg_stream_t stream) {
    return generate_host_impl<kWide>(h, per_stream, host_out, stream);
}

int xg_generate_host_f32(xg_ensemble_t h, uint64_t per_stream, float* host_out, xg_stream_t stream) {
    if (h && h->kind == kGeneric) return XG_EUNSUPPORTED;
    return generate_host_impl<kF32>(h, per_stream, host_out, stream);
}

int xg_generate_host_f64(xg_ensemble_t h, uint64_t per_stream, double* host_out, xg_stream_t stream) {
    if (h && h->kind == kGeneric) return XG_EUNSUPPORTED;
    uint64_t words;
    if (mul_overflows(per_stream, 2, &words)) return XG_EINVAL;
    return generate_host_impl<kF64>(h, per_stream, host_out, stream);
}

}  // extern "C"

namespace {

// One refill of ring slot i on the ring's stream: save the state, generate
// kNextBuf words of the (single) stream in the reference's uint64 container
// (so the host's next_word is one load, whatever w), copy them to the pinned
// slot.
int ring_refill(xg_ensemble* h, int i) {
    auto& r = h->nr;
    int rc = copy_state(h, r.snap[i], /*to_snapshot=*/true, r.st);
    if (!rc)
        rc = launch_fill<kWide>(h, 0, 1, kNextBuf, r.dev[i], nullptr, r.st);
    if (!rc) rc = cuda_rc(cudaMemcpyAsync(r.host[i], r.dev[i], kNextBuf * sizeof(uint64_t), cudaMemcpyDeviceToHost, r.st));
    if (!rc) rc = cuda_rc(cudaEventRecord(r.ev[i], r.st));
    return rc;
}

// Make slot `cur` hold unserved words: the first call (or the first after
// a settle) orders after all device work, then queues both slots; later
// calls wait for the slot generated in the background and queue the next
// refill into the slot just consumed, so generation and the PCIe copy of
// slot i+1 overlap the host's consumption of slot i.
int ring_next(xg_ensemble* h) {
    auto& r = h->nr;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    int rc = XG_OK;
    if (!r.st) {
        size_t wb;
        const size_t sb = state_bytes(h, &wb);
        rc = cuda_rc(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking));
        for (int i = 0; i < 2 && !rc; ++i) {
            rc = cuda_rc(cudaMallocHost(&r.host[i], kNextBuf * sizeof(uint64_t)));
            if (!rc) rc = cuda_rc(cudaMalloc(&r.dev[i], kNextBuf * sizeof(uint64_t)));
            if (!rc) rc = cuda_rc(cudaMalloc(&r.snap[i], sb));
            if (!rc) rc = cuda_rc(cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming));
        }
        if (rc) return rc;
    }
    if (!r.active) {
        // Host-synchronous start: order after any work queued on any stream.
        rc = cuda_rc(cudaDeviceSynchronize());
        if (!rc) rc = ring_refill(h, 0);
        if (!rc) rc = ring_refill(h, 1);
        if (!rc) rc = cuda_rc(cudaEventSynchronize(r.ev[0]));
        if (rc) return rc;
        r.cur = 0;
    } else {
        const int nxt = r.cur ^ 1;
        rc = cuda_rc(cudaEventSynchronize(r.ev[nxt]));
        if (!rc) rc = ring_refill(h, r.cur);
        if (rc) return rc;
        r.cur = nxt;
    }
    r.pos = 0;
    r.active = true;
    return XG_OK;
}

}  // namespace

extern "C" {

// XorgensState::next_word (proj/include/xg/xorgens.hpp:58-62): the w-bit
// word in a uint64, served from device-generated refills of kNextBuf words.
int xg_next_word(xg_ensemble_t h, uint64_t* out) {
    if (!h || !out) return XG_EINVAL;
    auto& r = h->nr;
    if (r.active && r.pos < kNextBuf) {
        *out = static_cast<const uint64_t*>(r.host[r.cur])[r.pos++];
        return XG_OK;
    }
    if (h->num_streams != 1) return XG_EINVAL;
    int rc = ring_next(h);
    if (rc) return rc;
    *out = static_cast<const uint64_t*>(r.host[r.cur])[r.pos++];
    return XG_OK;
}

int xg_next_view(xg_ensemble_t h, const uint64_t** words, uint64_t* count) {
    if (!h || !words || !count) return XG_EINVAL;
    if (h->num_streams != 1) return XG_EINVAL;
    auto& r = h->nr;
    if (!r.active || r.pos >= kNextBuf) {
        int rc = ring_next(h);
        if (rc) return rc;
    }
    *words = static_cast<const uint64_t*>(r.host[r.cur]) + r.pos;
    *count = kNextBuf - r.pos;
    r.pos = kNextBuf;  // served, until xg_next_return gives some back
    return XG_OK;
}

int xg_next_return(xg_ensemble_t h, uint64_t unread) {
    if (!h) return XG_EINVAL;
    auto& r = h->nr;
    if (unread == 0) return XG_OK;
    if (!r.active || unread > r.pos) return XG_ERANGE;
    r.pos -= unread;
    return XG_OK;
}

int xg_next_u32(xg_ensemble_t h, uint32_t* out) {
    if (!h || !out) return XG_EINVAL;
    if (h->params.w > 32) return XG_EUNSUPPORTED;
    uint64_t v;
    int rc = xg_next_word(h, &v);
    if (!rc) *out = static_cast<uint32_t>(v);
    return rc;
}

int xg_next_u64(xg_ensemble_t h, uint64_t* out) {
    if (!h || !out) return XG_EINVAL;
    if (h->params.w == 64) return xg_next_word(h, out);
    if (h->params.w != 32) return XG_EUNSUPPORTED;
    uint64_t lo, hi;
    int rc = xg_next_word(h, &lo);
    if (rc) return rc;
    rc = xg_next_word(h, &hi);
    if (rc) return rc;
    *out = lo | (hi << 32);
    return XG_OK;
}

int xg_state_export(xg_ensemble_t h, uint32_t index, uint64_t* buffer, uint64_t* weyl) {
    if (!h || !buffer || !weyl) return XG_EINVAL;
    if (index >= h->num_streams) return XG_ERANGE;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    int rc = cuda_rc(cudaDeviceSynchronize());
    if (!rc) rc = settle_next(h, nullptr);
    if (rc) return rc;
    if (h->kind == kGeneric) {
        const unsigned r = h->params.r;
        rc = cuda_rc(cudaMemcpy(buffer, h->d_win64 + static_cast<size_t>(index) * r, r * 8,
                                cudaMemcpyDeviceToHost));
        if (!rc) rc = cuda_rc(cudaMemcpy(weyl, h->d_weyl64 + index, 8, cudaMemcpyDeviceToHost));
        return rc;
    }
    uint32_t win[kR], wy;
    rc = cuda_rc(cudaMemcpy(win, h->d_win + static_cast<size_t>(index) * kR, sizeof win,
                            cudaMemcpyDeviceToHost));
    if (!rc) rc = cuda_rc(cudaMemcpy(&wy, h->d_weyl + index, 4, cudaMemcpyDeviceToHost));
    if (rc) return rc;
    for (unsigned i = 0; i < kR; ++i) buffer[i] = win[i];
    *weyl = wy;
    return XG_OK;
}

int xg_state_import(xg_ensemble_t h, uint32_t index, const uint64_t* buffer, uint64_t weyl) {
    if (!h || !buffer) return XG_EINVAL;
    if (index >= h->num_streams) return XG_ERANGE;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    int rc = cuda_rc(cudaDeviceSynchronize());
    if (!rc) rc = settle_next(h, nullptr);
    if (rc) return rc;
    if (h->kind == kGeneric) {
        const unsigned r = h->params.r;
        const uint64_t mask = h->params.w >= 64 ? ~0ull : ((1ull << h->params.w) - 1);
        std::vector<uint64_t> win(buffer, buffer + r);
        for (auto& v : win) v &= mask;
        const uint64_t wy = weyl & mask;
        rc = cuda_rc(cudaMemcpy(h->d_win64 + static_cast<size_t>(index) * r, win.data(), r * 8,
                                cudaMemcpyHostToDevice));
        if (!rc) rc = cuda_rc(cudaMemcpy(h->d_weyl64 + index, &wy, 8, cudaMemcpyHostToDevice));
        return rc;
    }
    uint32_t win[kR];
    for (unsigned i = 0; i < kR; ++i) win[i] = static_cast<uint32_t>(buffer[i] & kMask32);
    const uint32_t wy = static_cast<uint32_t>(weyl & kMask32);
    rc = cuda_rc(cudaMemcpy(h->d_win + static_cast<size_t>(index) * kR, win, sizeof win,
                            cudaMemcpyHostToDevice));
    if (!rc) rc = cuda_rc(cudaMemcpy(h->d_weyl + index, &wy, 4, cudaMemcpyHostToDevice));
    return rc;
}

int xg_state_export_all(xg_ensemble_t h, uint32_t* host_window, uint32_t* host_weyl) {
    if (!h || !host_window || !host_weyl) return XG_EINVAL;
    if (h->kind == kGeneric) return XG_EUNSUPPORTED;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    int rc = cuda_rc(cudaDeviceSynchronize());
    if (!rc) rc = settle_next(h, nullptr);
    const size_t n = h->num_streams;
    if (!rc) rc = cuda_rc(cudaMemcpy(host_window, h->d_win, n * kR * 4, cudaMemcpyDeviceToHost));
    if (!rc) rc = cuda_rc(cudaMemcpy(host_weyl, h->d_weyl, n * 4, cudaMemcpyDeviceToHost));
    return rc;
}

int xg_state_import_all(xg_ensemble_t h, const uint32_t* host_window, const uint32_t* host_weyl) {
    if (!h || !host_window || !host_weyl) return XG_EINVAL;
    if (h->kind == kGeneric) return XG_EUNSUPPORTED;
    DeviceGuard dg(h->device);
    if (!dg.ok) return XG_ECUDA;
    int rc = cuda_rc(cudaDeviceSynchronize());
    if (!rc) rc = settle_next(h, nullptr);
    const size_t n = h->num_streams;
    if (!rc) rc = cuda_rc(cudaMemcpy(h->d_win, host_window, n * kR * 4, cudaMemcpyHostToDevice));
    if (!rc) rc = cuda_rc(cudaMemcpy(h->d_weyl, host_weyl, n * 4, cudaMemcpyHostToDevice));
    return rc;
}

int xg_jump_minpoly(const xg_params_t* p, uint64_t* coeffs64) {
    if (!p || !coeffs64) return XG_EINVAL;
    Kind kind;
    int e = classify(p, &kind);
    if (e) return e;
    if (kind == kGeneric) return XG_EUNSUPPORTED;
    std::vector<uint64_t> m;
    bool ok = false;
    auto raw = [p](const std::vector<uint32_t>& window, size_t n, uint32_t* out) {
        host_raw_words(*p, window, n, out);
        return XG_OK;
    };
    e = minpoly_of(raw, m, &ok);
    if (e) return e;
    if (!ok) return XG_EUNSUPPORTED;
    std::memcpy(coeffs64, m.data(), kPolyWords * sizeof(uint64_t));
    return XG_OK;
}

int xg_partition(uint64_t total_streams, uint32_t world, uint32_t rank, uint64_t* first,
                 uint32_t* count) {
    if (!first || !count || world == 0) return XG_EINVAL;
    if (rank >= world) return XG_ERANGE;
    const unsigned __int128 t = total_streams;
    const uint64_t lo = static_cast<uint64_t>(t * rank / world);
    const uint64_t hi = static_cast<uint64_t>(t * (rank + 1) / world);
    if (hi - lo > 0xffffffffull) return XG_ERANGE;
    *first = lo;
    *count = static_cast<uint32_t>(hi - lo);
    return XG_OK;
}

uint64_t xg_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* xg_build_info(void) {
    return "libxg_gpu: xorgensGP warp-per-stream register-window kernels, sm_100a";
}

}  // extern "C"

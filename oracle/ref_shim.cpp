// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C entry layer over the UNMODIFIED reference sources
// (proj/src/{params,xorgens,parallel}.cpp, compiled where they lie by
// oracle/Makefile into oracle/_ref/libxgref.so).  Used (1) to pin the C
// restatement in oracle/xg_oracle.c and to generate tests/golden fixtures, and
// (2) as bench.py's reference arm / cpu_baseline (cpu_baseline.kind
// "reference").  Nothing here re-implements generator arithmetic: every value
// comes out of xg::XorgensState / xg::batch_step / xg::BlockEnsemble.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <ctime>
#include <exception>
#include <stdexcept>
#include <vector>

#include "xg/baselines.hpp"
#include "xg/params.hpp"
#include "xg/parallel.hpp"
#include "xg/xorgens.hpp"

namespace {

xg::GeneratorParams to_params(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma) {
    xg::GeneratorParams p;
    p.r = rsabcdw[0];
    p.s = rsabcdw[1];
    p.a = rsabcdw[2];
    p.b = rsabcdw[3];
    p.c = rsabcdw[4];
    p.d = rsabcdw[5];
    p.w = rsabcdw[6];
    p.omega = omega;
    p.gamma = gamma;
    return p;
}

double thread_cpu_seconds() {
    timespec ts;
    clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
    return static_cast<double>(ts.tv_sec) + static_cast<double>(ts.tv_nsec) * 1e-9;
}

} // namespace

extern "C" {

// check_params: 0 or 1 + ParamError ordinal.
int xgref_check_params(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma) {
    auto e = xg::check_params(to_params(rsabcdw, omega, gamma));
    return e ? 1 + static_cast<int>(*e) : 0;
}

// XorgensState(params, seed).next_word() x n.
int xgref_stream(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                 std::uint64_t seed, std::uint64_t n, std::uint64_t* out) {
    try {
        xg::XorgensState st(to_params(rsabcdw, omega, gamma), seed);
        for (std::uint64_t k = 0; k < n; ++k)
            out[k] = st.next_word();
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// RawXorgens(params, seed).next() x n (proj/include/xg/baselines.hpp:60-71).
int xgref_raw_stream(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                     std::uint64_t seed, std::uint64_t n, std::uint64_t* out) {
    try {
        xg::RawXorgens g(to_params(rsabcdw, omega, gamma), seed);
        for (std::uint64_t k = 0; k < n; ++k)
            out[k] = g.next();
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Low bit of every word of RawXorgens(params, seed) (raw = 1) or
// XorgensState(params, seed) (raw = 0) over `words` words: the first `window`
// bits and the last `window` bits, as collect_low_bits does
// (proj/tests/test_long_linearity.cpp:30-52).
int xgref_low_bit_windows(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                          std::uint64_t seed, int raw, std::uint64_t words, std::uint64_t window,
                          std::uint8_t* first, std::uint8_t* last) {
    try {
        const auto p = to_params(rsabcdw, omega, gamma);
        xg::RawXorgens rg(p, seed);
        xg::XorgensState st(p, seed);
        std::vector<std::uint8_t> ring(window, 0);
        std::uint64_t pos = 0;
        for (std::uint64_t i = 0; i < words; ++i) {
            const auto bit = static_cast<std::uint8_t>((raw ? rg.next() : st.next_word()) & 1);
            if (i < window) first[i] = bit;
            ring[pos] = bit;
            if (++pos == window) pos = 0;
        }
        for (std::uint64_t i = 0; i < window; ++i) last[i] = ring[(pos + i) % window];
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// State right after seeding: logical buffer (oldest first) + weyl.
int xgref_seeded_state(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                       std::uint64_t seed, std::uint64_t* buffer, std::uint64_t* weyl) {
    try {
        xg::XorgensState st(to_params(rsabcdw, omega, gamma), seed);
        auto lb = st.logical_buffer();
        std::memcpy(buffer, lb.data(), lb.size() * sizeof(std::uint64_t));
        *weyl = st.weyl_value();
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// from_raw(params, buffer, weyl).next_word() x n.
int xgref_from_raw_stream(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                          const std::uint64_t* buffer, std::uint64_t weyl, std::uint64_t n,
                          std::uint64_t* out) {
    try {
        auto p = to_params(rsabcdw, omega, gamma);
        std::vector<std::uint64_t> buf(buffer, buffer + p.r);
        auto st = xg::XorgensState::from_raw(p, buf, weyl);
        for (std::uint64_t k = 0; k < n; ++k)
            out[k] = st.next_word();
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// ---- BlockEnsemble handle (proj/src/parallel.cpp:84-135) -----------------

void* xgref_ensemble_create(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                            std::uint64_t base_seed, unsigned num_blocks, unsigned lanes) {
    try {
        return new xg::BlockEnsemble(to_params(rsabcdw, omega, gamma), base_seed, num_blocks,
                                     lanes);
    } catch (const std::exception&) {
        return nullptr;
    }
}

void xgref_ensemble_destroy(void* h) { delete static_cast<xg::BlockEnsemble*>(h); }

// generate(per_block, workers); the wall time of generate() alone is
// returned in *seconds (measure_ensemble_throughput, proj/src/bench.cpp:95-112).
// If out != nullptr the block-major words are copied out as uint32.
int xgref_ensemble_generate(void* h, std::uint64_t per_block, unsigned workers,
                            std::uint32_t* out, double* seconds, std::uint64_t* xor_sink) {
    try {
        auto* e = static_cast<xg::BlockEnsemble*>(h);
        auto t0 = std::chrono::steady_clock::now();
        auto blocks = e->generate(per_block, workers);
        std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
        if (seconds) *seconds = dt.count();
        std::uint64_t sink = 0;
        std::size_t pos = 0;
        for (const auto& b : blocks)
            for (std::uint64_t w : b) {
                sink ^= w;
                if (out) out[pos] = static_cast<std::uint32_t>(w);
                ++pos;
            }
        if (xor_sink) *xor_sink = sink;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Digests of streams [first, first + count) of BlockEnsemble(params,
// base_seed, ...) -- stream g is XorgensState(params, base_seed + g)
// (proj/src/parallel.cpp:84-95) -- for the full-size parity goldens.  Per
// stream and per output, three numbers over the row's elements e_k (k = 0..):
// xor (u32), sum e_k and sum e_k * (k + 1) (uint64 wrap).  Outputs (each
// [count]-long, nullptr = skip):
//   u32: the first n_u32 words;  f32: the bit patterns of (w >> 8) * 2^-24 of
//   the same words;  f64: the n_f64 doubles (u64 >> 11) * 2^-53 with u64 = the
//   word pair (w[2m], w[2m+1]) lo first, digested as 2 * n_f64 u32 elements
//   (the little-endian halves);  mc: hits of the first n_mc samples (pair m,
//   signed coordinates, hit iff x^2 + y^2 < 2^62).  The conversions are the
//   DESIGN.md section 3 conventions applied to reference words (the reference
//   has none of its own); every generated word comes from next_word().
struct Digest3 {
    std::uint32_t x = 0;
    std::uint64_t s = 0, ws = 0, k = 0;
    void add(std::uint32_t v) {
        x ^= v;
        s += v;
        ws += static_cast<std::uint64_t>(v) * ++k;
    }
};

int xgref_stream_digests(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                         std::uint64_t base_seed, std::uint64_t first, std::uint64_t count,
                         std::uint64_t n_u32, std::uint64_t n_f64, std::uint64_t n_mc,
                         std::uint32_t* u32_x, std::uint64_t* u32_s, std::uint64_t* u32_ws,
                         std::uint32_t* f32_x, std::uint64_t* f32_s, std::uint64_t* f32_ws,
                         std::uint32_t* f64_x, std::uint64_t* f64_s, std::uint64_t* f64_ws,
                         std::uint32_t* mc_hits) {
    try {
        const auto p = to_params(rsabcdw, omega, gamma);
        std::uint64_t n = n_u32;
        if (2 * n_f64 > n) n = 2 * n_f64;
        if (2 * n_mc > n) n = 2 * n_mc;
        for (std::uint64_t i = 0; i < count; ++i) {
            xg::XorgensState st(p, base_seed + first + i);
            Digest3 du, df, dd;
            std::uint32_t hits = 0, lo = 0;
            for (std::uint64_t k = 0; k < n; ++k) {
                const auto w = static_cast<std::uint32_t>(st.next_word());
                if (k < n_u32) {
                    du.add(w);
                    const float f = static_cast<float>(w >> 8) * 0x1p-24f;
                    std::uint32_t fb;
                    std::memcpy(&fb, &f, 4);
                    df.add(fb);
                }
                if ((k & 1) == 0) {
                    lo = w;
                    continue;
                }
                const std::uint64_t m = k >> 1;
                if (m < n_f64) {
                    const std::uint64_t u = lo | (static_cast<std::uint64_t>(w) << 32);
                    const double d = static_cast<double>(u >> 11) * 0x1p-53;
                    std::uint64_t db;
                    std::memcpy(&db, &d, 8);
                    dd.add(static_cast<std::uint32_t>(db));
                    dd.add(static_cast<std::uint32_t>(db >> 32));
                }
                if (m < n_mc) {
                    const std::int64_t x = static_cast<std::int32_t>(lo), y = static_cast<std::int32_t>(w);
                    hits += static_cast<std::uint64_t>(x * x) + static_cast<std::uint64_t>(y * y) <
                            (1ull << 62);
                }
            }
            if (u32_x) { u32_x[i] = du.x; u32_s[i] = du.s; u32_ws[i] = du.ws; }
            if (f32_x) { f32_x[i] = df.x; f32_s[i] = df.s; f32_ws[i] = df.ws; }
            if (f64_x) { f64_x[i] = dd.x; f64_s[i] = dd.s; f64_ws[i] = dd.ws; }
            if (mc_hits) mc_hits[i] = hits;
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Streams [first, first + count) of BlockEnsemble(params, base_seed, ...) as
// independent XorgensState loops, n words each, every word folded into a
// per-stream xor (the CPU baseline of the 2^34-word disjoint-stream fill:
// per-stream states on all cores; generate() would need 128 GiB).
int xgref_streams_xor(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                      std::uint64_t base_seed, std::uint64_t first, std::uint64_t count,
                      std::uint64_t n, std::uint32_t* xor_out) {
    try {
        const auto p = to_params(rsabcdw, omega, gamma);
        for (std::uint64_t i = 0; i < count; ++i) {
            xg::XorgensState st(p, base_seed + first + i);
            std::uint64_t x = 0;
            for (std::uint64_t k = 0; k < n; ++k) x ^= st.next_word();
            xor_out[i] = static_cast<std::uint32_t>(x);
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// The CPU equivalent of the fused conversion fills for the bench baseline:
// streams [first, first + count) as XorgensState loops, n values each,
// mode 0 = f32 (w >> 8) * 2^-24 of one word, 1 = f64 (u64 >> 11) * 2^-53 of
// the word pair (lo first) -- the DESIGN.md section 3 conventions applied to
// reference words; the value bits fold into a per-stream xor sink.
int xgref_streams_convert(const unsigned* rsabcdw, std::uint64_t omega, unsigned gamma,
                          std::uint64_t base_seed, std::uint64_t first, std::uint64_t count,
                          std::uint64_t n, int mode, std::uint64_t* sink_out) {
    try {
        const auto p = to_params(rsabcdw, omega, gamma);
        for (std::uint64_t i = 0; i < count; ++i) {
            xg::XorgensState st(p, base_seed + first + i);
            std::uint64_t sink = 0;
            for (std::uint64_t k = 0; k < n; ++k) {
                if (mode == 0) {
                    const float f = static_cast<float>(static_cast<std::uint32_t>(st.next_word()) >> 8) * 0x1p-24f;
                    std::uint32_t b;
                    std::memcpy(&b, &f, 4);
                    sink ^= b;
                } else {
                    const std::uint64_t lo = st.next_word(), hi = st.next_word();
                    const double d = static_cast<double>((lo | (hi << 32)) >> 11) * 0x1p-53;
                    std::uint64_t b;
                    std::memcpy(&b, &d, 8);
                    sink ^= b;
                }
            }
            sink_out[i] = sink;
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Serial next_word throughput, the measure_throughput method
// (proj/src/bench.cpp:67-93): best chunk rate on thread CPU time.
double xgref_serial_rate(std::uint64_t seed, std::uint64_t count, unsigned chunks,
                         std::uint64_t* sink_out) {
    xg::XorgensState st(xg::xorgensgp32_params(), seed);
    std::uint64_t sink = 0, produced = 0;
    const std::uint64_t chunk = count / chunks;
    double best = 0.0;
    for (unsigned c = 0; c < chunks; ++c) {
        const std::uint64_t n = (c == chunks - 1) ? count - produced : chunk;
        const double t0 = thread_cpu_seconds();
        for (std::uint64_t i = 0; i < n; ++i)
            sink ^= st.next_word();
        const double dt = thread_cpu_seconds() - t0;
        produced += n;
        if (dt > 0.0 && static_cast<double>(n) / dt > best) best = static_cast<double>(n) / dt;
    }
    if (sink_out) *sink_out = sink;
    return best;
}

} // extern "C"

// dropin_test.cpp -- TEST: the reference C++ API next to its GPU drop-in.
//
// Compiled (oracle/Makefile target `dropin`) against the reference headers,
// linked with oracle/_ref/libxgref.so (the reference sources) and
// libxg_gpu.so.  Every check compares xg:: (reference, CPU) with xg::gpu::
// (this framework, B200) on the same inputs, through the same calls a C++
// user of the reference makes.  Exit 0 = all equal.
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "xg/gpu.hpp"
#include "xg/parallel.hpp"
#include "xg/params.hpp"
#include "xg/stream.hpp"
#include "xg/xorgens.hpp"

static int failures = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                            \
        }                                                          \
    } while (0)

int main() {
    const xg::GeneratorParams p = xg::xorgensgp32_params();

    // BlockEnsemble::generate, twice (continuation), awkward sizes.
    for (std::size_t per : {1ul, 17ul, 1000ul, 4097ul}) {
        xg::BlockEnsemble ref(p, 7, 5, 63);
        xg::gpu::BlockEnsemble gpu(p, 7, 5, 63);
        for (int call = 0; call < 2; ++call) CHECK(ref.generate(per) == gpu.generate(per));
    }
    // Serial stream, batch_step, state hooks.
    xg::XorgensState rs(p, 42);
    xg::gpu::XorgensState gs(p, 42);
    for (int i = 0; i < 5000; ++i) CHECK(rs.next_word() == gs.next_word());
    CHECK(xg::batch_step(rs, 63) == xg::gpu::batch_step(gs, 63));
    CHECK(rs.logical_buffer() == gs.logical_buffer());
    CHECK(rs.weyl_value() == gs.weyl_value());
    auto rr = xg::XorgensState::from_raw(p, rs.logical_buffer(), rs.weyl_value());
    auto gr = xg::gpu::XorgensState::from_raw(p, rs.logical_buffer(), rs.weyl_value());
    for (int i = 0; i < 3000; ++i) CHECK(rr.next_word() == gr.next_word());
    // WordSource adapter (stream.hpp:25-35) behind the reference's virtual base.
    {
        xg::XorgensSource rsrc(p, 77);
        xg::gpu::XorgensSource<xg::WordSource> gsrc(p, 77);
        xg::WordSource& as_base = gsrc;
        CHECK(as_base.word_bits() == rsrc.word_bits());
        for (int i = 0; i < 300000; ++i) CHECK(rsrc.next() == as_base.next());  // > 4 refill slots
    }
    // next_word across refill slots, interleaved with generate(): the unread
    // words of the inline cache are handed back first, so the stream continues
    // exactly after the last word the caller saw.
    {
        xg::XorgensState r2(p, 2024);
        xg::gpu::XorgensState g2(p, 2024);
        for (int round = 0; round < 3; ++round) {
            for (int i = 0; i < 70001; ++i) CHECK(r2.next_word() == g2.next_word());
            const auto blk = g2.generate(1001);
            for (std::uint64_t w : blk[0]) CHECK(r2.next_word() == w);
        }
        CHECK(r2.logical_buffer() == g2.logical_buffer());
        CHECK(r2.weyl_value() == g2.weyl_value());
        for (int i = 0; i < 10; ++i) CHECK(r2.next_word() == g2.next_word());
    }
    // Checkpoint / resume continues every block exactly.
    {
        xg::gpu::BlockEnsemble a(p, 11, 4, 63);
        a.generate(1000);
        std::vector<std::uint32_t> win, wy;
        a.export_state(win, wy);
        auto next_a = a.generate(500);
        xg::gpu::BlockEnsemble b(p, 0, 4, 63);
        b.import_state(win, wy);
        CHECK(b.generate(500) == next_a);
        xg::BlockEnsemble ref(p, 11, 4, 63);
        ref.generate(1000);
        CHECK(ref.generate(500) == next_a);
    }
    // Non-production parameter sets (general-parameter kernels): the tiny
    // verification sets of params.hpp:89-91 and the w = 64 set.
    {
        xg::GeneratorParams w64 = p;
        w64.r = 64; w64.s = 53; w64.a = 33; w64.b = 26; w64.c = 27; w64.d = 29; w64.w = 64;
        w64.gamma = 32; w64.omega = 0x9E3779B97F4A7C15ull;
        const xg::GeneratorParams sets[] = {xg::tiny_r2w8_params(), xg::tiny_r2w16_params(),
                                            xg::tiny_r4w16_params(), w64};
        for (const auto& q : sets) {
            const unsigned lanes = xg::lane_bound(q) < 4 ? xg::lane_bound(q) : 4;
            xg::BlockEnsemble ref(q, 3, 3, lanes);
            xg::gpu::BlockEnsemble gpu(q, 3, 3, lanes);
            for (int call = 0; call < 2; ++call) CHECK(ref.generate(333) == gpu.generate(333));
            xg::XorgensState rq(q, 9);
            xg::gpu::XorgensState gq(q, 9);
            for (int i = 0; i < 2000; ++i) CHECK(rq.next_word() == gq.next_word());
        }
    }
    // Same exception classes.
    bool threw = false;
    try { xg::gpu::BlockEnsemble bad(p, 0, 1, 64); } catch (const std::out_of_range&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { xg::gpu::BlockEnsemble bad(p, 0, 0, 1); } catch (const std::out_of_range&) { threw = true; }
    CHECK(threw);
    threw = false;
    xg::GeneratorParams q = p;
    q.s = 64;
    try { xg::gpu::BlockEnsemble bad(q, 0, 1, 1); } catch (const std::invalid_argument& e) { threw = true; }
    CHECK(threw);
    std::printf("dropin_test: %s (%d failures)\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}

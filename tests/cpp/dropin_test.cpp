// dropin_test.cpp -- TEST: the reference C++ API next to its GPU drop-in.
//
// Compiled (oracle/Makefile target `dropin`) against the reference headers,
// linked with oracle/_ref/libxgref.so (the reference sources) and
// libxg_gpu.so.  Every check compares xg:: (reference, CPU) with xg::gpu::
// (this framework, B200) on the same inputs, through the same calls a C++
// user of the reference makes.  Exit 0 = all equal.
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "xg/gpu.hpp"
#include "xg/parallel.hpp"
#include "xg/params.hpp"
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

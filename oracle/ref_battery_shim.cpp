// ref_battery_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Runs the reference's own statistical battery (proj/src/stattests/*, via
// xg::stats::run_battery, proj/src/stattests/battery.cpp:72-112) over a
// caller-supplied buffer of 32-bit words -- e.g. words the GPU generated --
// through the reference's CallbackSource (proj/include/xg/stream.hpp:67-78).
// Built into oracle/_ref/libxgref_battery.so by oracle/Makefile.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "xg/stattests/battery.hpp"
#include "xg/stattests/gf2.hpp"
#include "xg/stattests/tests.hpp"
#include "xg/stream.hpp"

extern "C" {

// Returns the overall verdict (0 pass, 1 suspect, 2 fail, 3 n/a) or -1 when
// the buffer ran out / the run failed; the JSON report is copied to json_out.
int xgref_battery_on_words(const std::uint32_t* words, std::uint64_t n, int quick,
                           const char* label, char* json_out, std::uint64_t cap) {
    std::uint64_t pos = 0;
    xg::CallbackSource src(
        [&]() -> std::uint64_t {
            if (pos >= n) throw std::runtime_error("word buffer exhausted");
            return words[pos++];
        },
        32);
    try {
        auto cfg = quick ? xg::stats::BatteryConfig::quick() : xg::stats::BatteryConfig::defaults();
        auto report = xg::stats::run_battery(src, cfg, label, "GPU-generated words", 0);
        std::string js = xg::stats::to_json(report);
        if (json_out && cap) {
            std::strncpy(json_out, js.c_str(), cap - 1);
            json_out[cap - 1] = 0;
        }
        return static_cast<int>(report.overall);
    } catch (const std::exception& e) {
        if (json_out && cap) {
            std::strncpy(json_out, e.what(), cap - 1);
            json_out[cap - 1] = 0;
        }
        return -1;
    }
}

// run_battery over `bits`-wide words (bits = 8, 16, 32, 64: each buffer
// element holds one word) with a BatteryConfig parsed from `config_text`
// (BatteryConfig::parse, battery.cpp:38-70; empty = defaults); the report's
// generator / params / seed fields are the caller's.  Returns the overall
// verdict as xgref_battery_on_words does (-1: exhausted / threw, message in
// json_out).
int xgref_battery_config_on_words(const std::uint64_t* words, std::uint64_t n, unsigned bits,
                                  const char* config_text, const char* generator, const char* params,
                                  std::uint64_t seed, char* json_out, std::uint64_t cap) {
    std::uint64_t pos = 0;
    xg::CallbackSource src(
        [&]() -> std::uint64_t {
            if (pos >= n) throw std::runtime_error("word buffer exhausted");
            return words[pos++];
        },
        bits);
    try {
        std::istringstream in(config_text ? config_text : "");
        auto cfg = xg::stats::BatteryConfig::parse(in);
        auto report = xg::stats::run_battery(src, cfg, generator, params, seed);
        std::string js = xg::stats::to_json(report);
        if (json_out && cap) {
            std::strncpy(json_out, js.c_str(), cap - 1);
            json_out[cap - 1] = 0;
        }
        return static_cast<int>(report.overall);
    } catch (const std::exception& e) {
        if (json_out && cap) {
            std::strncpy(json_out, e.what(), cap - 1);
            json_out[cap - 1] = 0;
        }
        return -1;
    }
}

// The reference's own rank (proj/src/stattests/gf2.cpp:37-45, single-word
// rows) of one 32 x 32 matrix.
unsigned xgref_gf2_rank32(const std::uint32_t* rows32) {
    std::vector<std::uint64_t> rows(rows32, rows32 + 32);
    return xg::stats::gf2_rank(rows, 32);
}

// The reference's matrix_rank_test (proj/src/stattests/tests.cpp:81-126)
// over a word buffer through CallbackSource + BitSource; returns 0, or -1
// when the buffer ran out / the test threw.
int xgref_matrix_rank_on_words(const std::uint32_t* words, std::uint64_t n,
                               std::uint64_t num_matrices, double* statistic, double* p_value) {
    std::uint64_t pos = 0;
    xg::CallbackSource src(
        [&]() -> std::uint64_t {
            if (pos >= n) throw std::runtime_error("word buffer exhausted");
            return words[pos++];
        },
        32);
    try {
        xg::BitSource bits(src);
        auto r = xg::stats::matrix_rank_test(bits, num_matrices, 32);
        *statistic = r.statistic;
        *p_value = r.p_value;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// The reference's Berlekamp-Massey (proj/src/stattests/gf2.cpp:62-110) of n
// bits (one byte per bit).
std::uint64_t xgref_berlekamp_massey(const std::uint8_t* bits, std::uint64_t n) {
    std::vector<std::uint8_t> v(bits, bits + n);
    return xg::stats::berlekamp_massey(v);
}

// The reference's linear_complexity_test (proj/src/stattests/tests.cpp:128-178)
// over a word buffer; returns 0, or -1 when the buffer ran out / it threw.
int xgref_linear_complexity_on_words(const std::uint32_t* words, std::uint64_t n,
                                     unsigned block_length, std::uint64_t num_blocks,
                                     double* statistic, double* p_value) {
    std::uint64_t pos = 0;
    xg::CallbackSource src(
        [&]() -> std::uint64_t {
            if (pos >= n) throw std::runtime_error("word buffer exhausted");
            return words[pos++];
        },
        32);
    try {
        xg::BitSource bits(src);
        auto r = xg::stats::linear_complexity_test(bits, block_length, num_blocks);
        *statistic = r.statistic;
        *p_value = r.p_value;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
